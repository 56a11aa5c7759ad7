"""Packet detection by normalised sliding correlation against the PN preamble,
on the device.

Mirrors the reference ``ofdmrx.sync`` (sync.py:1-44): ``DetectionResult``,
``DEFAULT_THRESHOLD`` and ``detect_packet(capture, pn, threshold)`` keep
their names, argument meaning and errors (InputError when a stream is
shorter than the PN).  The offset decision is taken on antenna 0; every
antenna's (peak index, peak metric) is reported.  The arithmetic runs in the
library's sm_100a kernels (``ofdmrx_detect`` / ``ofdmrx_corr_metrics``):
fp32 correlation over every window, fp64 re-scoring of the windows within the
fp32 error bound of each row's maximum.

``detect_frames`` is the batched device-resident form over F captures
[F, N, S]; its result feeds ``frames.receive_frames(symbol0_offset=...)``.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, device
from .errors import ContractError, InputError

DEFAULT_THRESHOLD = 0.6  # sync.py:14


@dataclass(frozen=True)
class DetectionResult:
    """sync.py:17-23."""

    detected: bool
    frame_start: int          # index of the first PN chip
    symbol0_offset: int       # index of the first OFDM symbol
    peak_metric: float        # normalized correlation magnitude in [0, 1]
    per_antenna_peaks: tuple  # (peak_index, peak_metric) per antenna


@dataclass
class FrameDetections:
    """Batched detection results (CUDA tensors)."""

    peak_index: torch.Tensor   # [F, N] int32, first argmax per (frame, antenna)
    peak_metric: torch.Tensor  # [F, N] float64
    n_chips: int
    threshold: float

    @property
    def detected(self):
        """[F] bool: antenna 0's peak >= threshold (sync.py:40)."""
        return self.peak_metric[:, 0] >= self.threshold

    @property
    def frame_start(self):
        return self.peak_index[:, 0]

    @property
    def symbol0_offset(self):
        return self.peak_index[:, 0].to(torch.int64) + self.n_chips

    def result(self, f=0):
        """DetectionResult of frame f (host copy)."""
        idx = self.peak_index[f].cpu().numpy()
        met = self.peak_metric[f].cpu().numpy()
        peaks = tuple((int(i), float(m)) for i, m in zip(idx, met))
        start, peak = peaks[0]
        return DetectionResult(detected=peak >= self.threshold, frame_start=start,
                               symbol0_offset=start + self.n_chips, peak_metric=peak, per_antenna_peaks=peaks)


class _ChipCache:
    def __init__(self):
        self._c = {}

    def get(self, chips, dev):
        a = np.ascontiguousarray(np.asarray(chips, dtype=np.float64).ravel())
        key = (str(dev), a.tobytes())
        t = self._c.get(key)
        if t is None:
            t = torch.from_numpy(a.astype(np.float32)).to(dev)
            self._c[key] = t
        return t


_CHIPS = _ChipCache()


def _chips_of(pn):
    chips = getattr(pn, "chips", pn)
    if isinstance(chips, torch.Tensor):
        chips = chips.detach().cpu().numpy()
    chips = np.asarray(chips)
    if chips.ndim != 1 or chips.size == 0:
        raise ContractError(f"PN chips must be a non-empty 1-D array, got shape {chips.shape}")
    if np.iscomplexobj(chips):
        raise ContractError("PN chips must be real (bipolar m-sequence, waveform.py:77-117)")
    return chips


def _rows(rx, dev):
    x = device.as_c64(rx, dev)
    if x.dim() == 1:
        x = x[None, None]
    elif x.dim() == 2:
        x = x[None]
    if x.dim() != 3:
        raise ContractError(f"streams must be [S], [N, S] or [F, N, S], got {tuple(x.shape)}")
    return x


def detect_frames(rx, pn, threshold=DEFAULT_THRESHOLD, *, antennas="all", scratch=None, stream=None):
    """Detect the PN preamble in the antenna streams of F captures.

    rx: complex64 CUDA tensor [F, N, S] (or [N, S]; numpy is copied H2D).
    pn: PnSequence-like (``.chips``) or a real chip array.
    antennas: "all" (every antenna's peak, DetectionResult.per_antenna_peaks)
    or "first" (antenna 0 only: the decision input of sync.py:37-42, 1/N of
    the work; peak arrays are then [F, 1]).
    Returns FrameDetections (no host sync)."""
    if antennas not in ("all", "first"):
        raise ContractError('antennas must be "all" or "first"')
    dev = device.require_cuda(rx.device if isinstance(rx, torch.Tensor) and rx.is_cuda else None)
    chips = _chips_of(pn)
    x = _rows(rx, dev)
    f, n, s = x.shape
    if s < chips.size:
        raise InputError(f"stream length {s} shorter than PN length {chips.size}")  # sync.py:28-31
    n_rows = n if antennas == "all" else 1  # antenna 0 only: rows f*N*S, one per frame
    lib = _lib.load()
    need = int(lib.ofdmrx_detect_scratch_bytes(f, n_rows, s, int(chips.size)))
    if need < 0:
        raise ContractError("invalid detection sizes")
    c = _CHIPS.get(chips, dev)
    with device.on_stream(stream):  # scratch and outputs belong to the launch stream
        if scratch is None or scratch.numel() < need:
            scratch = torch.empty((max(need, 8),), dtype=torch.uint8, device=dev)
        elif stream is not None:
            scratch.record_stream(stream)
        idx = torch.empty((f, n_rows), dtype=torch.int32, device=dev)
        met = torch.empty((f, n_rows), dtype=torch.float64, device=dev)
        _lib.call("ofdmrx_detect", device.ptr(x), f, n_rows, s, s, n * s, device.ptr(c), int(chips.size),
                  device.ptr(scratch), device.ptr(idx), device.ptr(met), device.stream_handle(stream))
    return FrameDetections(peak_index=idx, peak_metric=met, n_chips=int(chips.size), threshold=float(threshold))


def detect_packet(capture, pn, threshold=DEFAULT_THRESHOLD):
    """sync.detect_packet (sync.py:26-44) on the device.

    capture: RxCapture-like (``.streams`` [N, S]) or the streams array."""
    streams = getattr(capture, "streams", capture)
    if isinstance(streams, np.ndarray):
        streams = np.atleast_2d(streams)
    chips = _chips_of(pn)
    if streams.shape[-1] < chips.size:
        raise InputError(f"stream length {streams.shape[-1]} shorter than PN length {chips.size}")
    det = detect_frames(streams, chips, threshold)
    return det.result(0)


def corr_metrics(stream, chips, stream_=None):
    """kernels.corr_metrics (kernels/__init__.py:45-48) on the device:
    metric per window of a 1-D stream (or per row of [R, S]).  numpy in ->
    numpy float64 out; CUDA tensor in -> float32 CUDA tensor out."""
    host = not isinstance(stream, torch.Tensor)
    dev = device.require_cuda(stream.device if not host and stream.is_cuda else None)
    ch = _chips_of(chips)
    x = device.as_c64(stream, dev)
    single = x.dim() == 1
    if single:
        x = x[None]
    if x.dim() != 2:
        raise ContractError(f"stream must be [S] or [R, S], got {tuple(x.shape)}")
    r, s = x.shape
    if s < ch.size:
        raise InputError(f"stream length {s} shorter than PN length {ch.size}")
    out = torch.empty((r, s - ch.size + 1), dtype=torch.float32, device=dev)
    c = _CHIPS.get(ch, dev)
    _lib.call("ofdmrx_corr_metrics", device.ptr(x), 1, r, s, s, r * s, device.ptr(c), int(ch.size),
              device.ptr(out), device.stream_handle(stream_))
    if single:
        out = out[0]
    return out.cpu().numpy().astype(np.float64) if host else out
