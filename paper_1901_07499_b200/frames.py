"""Batched, device-resident receive: the throughput entry point.

``receive_frames`` runs the fused sm_100a kernel over F captures at once:
CP drop + FFT + fftshift, LS estimate on the pilot symbol, MRC over the
antennas, divide, hard demap — one pass over HBM.  It is the batched form of
the reference's per-frame chain extract_slots -> run_ring_pipeline ->
process_symbol (receiver.py:238-348); the per-symbol API in receiver.py is
compatibility sugar over it.

Input layout: ``rx`` is a complex64 tensor [F, N, S] (or [N, S] for one frame)
holding each antenna's sample stream; the pilot symbol (with its CP) starts
at ``symbol0_offset`` (DetectionResult.symbol0_offset, sync.py:21) and is
followed by ``n_data`` data symbols of fft_len + cp_len samples.  This is the
interleaved cf32 layout of the reference's .cf32 files (io_formats.py:18-30).
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, device
from .errors import ContractError, InputError
from .waveform import OfdmConfig, PilotDefinition, as_config, make_pilot


@dataclass
class FrameBatch:
    """Outputs of one receive_frames call (CUDA tensors unless copied)."""

    H: torch.Tensor        # [F, N, M] complex64  ChannelEstimate.gains
    s_hat: torch.Tensor    # [F, D, M] complex64  CombinedSymbol.equalized
    weights: torch.Tensor  # [F, M]    float32    CombinedSymbol.weight_norm
    bits: torch.Tensor     # [F, D*M*b] uint8     PipelineResult.bits
    flags: torch.Tensor    # [F]       int32      OR of FLAG_NONFINITE / FLAG_ERASED
    zf: torch.Tensor = None  # [F, D, N, M] per-antenna ZF output (optional)
    # [F, 5] int64 SM cycles per stage (pilot FFT, LS, data FFT, MRC, combine+demap),
    # only with receive_frames(profile=True) (ofdmrx_rx_frames_profiled)
    stage_cycles: torch.Tensor = None

    def stage_shares(self):
        """Fraction of the fused kernel's lane time per stage, summed over the
        batch: (pilot_fft, ls, data_fft, mrc, combine_demap)."""
        if self.stage_cycles is None:
            raise ContractError("receive_frames(profile=True) records the stage cycles")
        tot = self.stage_cycles.sum(0).double()
        return (tot / max(float(tot.sum()), 1.0)).tolist()

    @property
    def erased(self):
        """CombinedSymbol.erased per frame/subcarrier (receiver.py:234)."""
        return self.weights < device.MRC_WEIGHT_FLOOR


def _pilot_values(pilot, fft_len):
    if pilot is None:
        pilot = make_pilot(fft_len)
    # a PilotDefinition (ours or the reference's, waveform.py:204-211) or the values
    vals = pilot.values if isinstance(pilot, PilotDefinition) or hasattr(pilot, "values") else pilot
    vals = np.asarray(vals.cpu() if isinstance(vals, torch.Tensor) else vals)
    if vals.shape != (fft_len,):
        raise ContractError(f"pilot has {vals.shape} values, config needs ({fft_len},)")
    if not np.allclose(np.abs(vals), 1.0, atol=1e-12):
        from .errors import ConfigurationError

        raise ConfigurationError("pilot values must have unit modulus")
    return vals


_DEFAULT_PILOT_INFO = {}  # fft_len -> (values, options) of the default pilot, validated once


def _pilot_info(pilot, fft_len):
    """(values, OFDMRX pilot options, cache key) of a pilot.  The default pilot
    (pilot=None, waveform.py:214-220) is built and validated once per FFT
    length -- it dominated the host cost of a receive call; a caller's table
    is validated on every call (it may have been modified in between)."""
    if pilot is None:
        hit = _DEFAULT_PILOT_INFO.get(fft_len)
        if hit is None:
            vals = _pilot_values(None, fft_len)
            hit = _DEFAULT_PILOT_INFO[fft_len] = (vals, device.pilot_options(vals), ("default", fft_len))
        return hit
    vals = _pilot_values(pilot, fft_len)
    return vals, device.pilot_options(vals), None


class PilotCache:
    """Device copies of pilot tables, keyed by (device, values) -- or by
    (device, key) for the default pilots of _pilot_info."""

    def __init__(self):
        self._cache = {}

    def get(self, vals, dev, key=None):
        key = (str(dev), key) if key is not None else (
            str(dev), vals.shape[0], hash(np.asarray(vals, dtype=np.complex64).tobytes()))
        t = self._cache.get(key)
        if t is None:
            t = torch.from_numpy(np.ascontiguousarray(vals, dtype=np.complex64)).to(dev)
            self._cache[key] = t
        return t


_PILOTS = PilotCache()


def allocate_outputs(n_frames, n_antennas, fft_len, n_data, qam_order, dev, want_h=True, zf=False):
    qb = device.qam_bits(qam_order)
    return FrameBatch(
        H=torch.empty((n_frames, n_antennas, fft_len), dtype=torch.complex64, device=dev) if want_h else None,
        s_hat=torch.empty((n_frames, n_data, fft_len), dtype=torch.complex64, device=dev),
        weights=torch.empty((n_frames, fft_len), dtype=torch.float32, device=dev),
        bits=torch.empty((n_frames, n_data * fft_len * qb), dtype=torch.uint8, device=dev),
        flags=torch.zeros((n_frames,), dtype=torch.int32, device=dev),
        zf=torch.empty((n_frames, n_data, n_antennas, fft_len), dtype=torch.complex64, device=dev) if zf else None,
    )


def receive_frames(rx, cfg, pilot=None, *, symbol0_offset=0, n_data=None, eps=device.MRC_WEIGHT_FLOOR,
                   out=None, want_h=True, zf=False, check=False, stream=None, shards=None, profile=False,
                   latency=False):
    """Fused receive of a batch of captures on the current CUDA device.

    rx: complex64 CUDA tensor [F, N, S] or [N, S] (numpy is copied H2D).
    Returns a FrameBatch.  With check=True, raises NumericInputError when a
    frame fed non-finite samples to the FFT (forces a device sync).  Results
    do not depend on the batch (F) a frame is received in; `shards` is
    accepted for compatibility and ignored.  profile=True also records the
    per-stage SM cycles of the fused kernel (FrameBatch.stage_cycles; same
    results, an instrumented build of the kernel).  latency=True selects the
    single-frame latency plan (OFDMRX_OPT_LATENCY: each frame over a whole
    thread-block cluster; its own fixed antenna-sum order)."""
    cfg = as_config(cfg)
    dev = device.require_cuda(rx.device if isinstance(rx, torch.Tensor) and rx.is_cuda else None)
    x = device.as_c64(rx, dev)
    if x.dim() == 2:
        x = x[None]
    if x.dim() != 3:
        raise ContractError(f"rx must be [F, N, S] or [N, S], got shape {tuple(x.shape)}")
    f, n, s = x.shape
    if n != cfg.n_antennas:
        raise ContractError(f"rx has {n} antenna rows, config has {cfg.n_antennas}")
    sym_len = cfg.symbol_len
    if n_data is None:
        n_data = (s - symbol0_offset) // sym_len - 1
    if n_data < 0 or symbol0_offset < 0:
        raise InputError(f"capture of {s} samples holds no pilot symbol at offset {symbol0_offset}")
    desc_args = (f, n, cfg.fft_len, cfg.cp_len, n_data, cfg.qam_order, symbol0_offset, s, n * s, eps)
    return _launch_rx(desc_args, x, cfg, pilot, out, want_h, zf, check, stream, profile=profile, latency=latency)


def _launch_rx(desc_args, x, cfg, pilot, out, want_h, zf, check, stream, profile=False, latency=False):
    f, n, _, _, n_data = desc_args[:5]
    pvals, popts, pkey = _pilot_info(pilot, cfg.fft_len)
    opts = popts | (_lib.OPT_LATENCY if latency else 0)
    desc = device.make_desc(*desc_args, options=opts, rx_samples=x.numel())
    device.check_desc(desc)
    pv = _PILOTS.get(pvals, x.device, pkey)
    with device.on_stream(stream):  # outputs allocated / zeroed on the launch stream
        if out is None:
            out = allocate_outputs(f, n, cfg.fft_len, n_data, cfg.qam_order, x.device, want_h=want_h, zf=zf)
        else:
            out.flags.zero_()
        if profile:
            out.stage_cycles = torch.zeros((f, 5), dtype=torch.int64, device=x.device)
            _lib.call("ofdmrx_rx_frames_profiled", ctypes.byref(desc), device.ptr(x), device.ptr(pv),
                      device.ptr(out.H), device.ptr(out.s_hat), device.ptr(out.weights), device.ptr(out.bits),
                      device.ptr(out.zf), device.ptr(out.flags), device.ptr(out.stage_cycles),
                      device.stream_handle(stream))
        else:
            _lib.call("ofdmrx_rx_frames", ctypes.byref(desc), device.ptr(x), device.ptr(pv), device.ptr(out.H),
                      device.ptr(out.s_hat), device.ptr(out.weights), device.ptr(out.bits), device.ptr(out.zf),
                      device.ptr(out.flags), device.stream_handle(stream))
    if check:
        device.raise_on_flags(out.flags)
    return out


def stage_symbols(src, cfg, *, symbol0_offset=0, n_data, dst=None, stream=None):
    """Ingest: copy only the symbol payloads (CP dropped) of captures `src`
    [F, N, S] complex64 (pinned host or CUDA) into a dense CUDA tensor
    [F, N, 1+D, M] with strided copy-engine transfers (ofdmrx_stage_symbols).
    This is extract_slots + cp_drop (receiver.py:274-291,186-193) applied
    before the bytes cross PCIe."""
    if src.dim() == 2:
        src = src[None]
    if src.dtype != torch.complex64 or not src.is_contiguous():
        raise ContractError("stage_symbols needs a contiguous complex64 [F, N, S] tensor")
    f, n, s = src.shape
    dev = device.require_cuda(None if not src.is_cuda else src.device)
    if dst is None:
        dst = torch.empty((f, n, 1 + n_data, cfg.fft_len), dtype=torch.complex64, device=dev)
    if tuple(dst.shape) != (f, n, 1 + n_data, cfg.fft_len) or not dst.is_contiguous():
        raise ContractError(f"dst must be contiguous [{f}, {n}, {1 + n_data}, {cfg.fft_len}]")
    desc = device.make_desc(f, n, cfg.fft_len, cfg.cp_len, n_data, cfg.qam_order, symbol0_offset, s, n * s,
                            rx_samples=f * n * s)
    device.check_desc(desc)
    _lib.call("ofdmrx_stage_symbols", ctypes.byref(desc), device.ctypes_void(src.data_ptr()), device.ptr(dst),
              device.stream_handle(stream))
    return dst


def receive_staged(x, cfg, pilot=None, *, eps=device.MRC_WEIGHT_FLOOR, out=None, want_h=True, zf=False,
                   check=False, stream=None):
    """receive_frames on the dense [F, N, 1+D, M] layout stage_symbols writes
    (cp_len 0, symbols back to back)."""
    if x.dim() != 4 or x.dtype != torch.complex64 or not x.is_cuda:
        raise ContractError("receive_staged needs a complex64 CUDA tensor [F, N, 1+D, M]")
    f, n, sy, m = x.shape
    if m != cfg.fft_len or n != cfg.n_antennas:
        raise ContractError(f"staged batch {tuple(x.shape)} does not match the config")
    desc_args = (f, n, m, 0, sy - 1, cfg.qam_order, 0, sy * m, n * sy * m, eps)
    return _launch_rx(desc_args, x, cfg, pilot, out, want_h, zf, check, stream)


def receive_partials(rx, cfg, pilot=None, *, symbol0_offset=0, n_data=None, eps=device.MRC_WEIGHT_FLOOR,
                     want_h=True, stream=None):
    """Antenna-shard half of the fused pass: returns (H, num [F,D,M] c64,
    den [F,M] f32, flags) — the un-normalised MRC accumulators over this
    shard's antennas (mrc_seq, numba_backend.py:146-151)."""
    dev = device.require_cuda(rx.device if isinstance(rx, torch.Tensor) and rx.is_cuda else None)
    x = device.as_c64(rx, dev)
    if x.dim() == 2:
        x = x[None]
    f, n, s = x.shape
    if n_data is None:
        n_data = (s - symbol0_offset) // cfg.symbol_len - 1
    pvals = _pilot_values(pilot, cfg.fft_len)
    desc = device.make_desc(f, n, cfg.fft_len, cfg.cp_len, n_data, cfg.qam_order, symbol0_offset, s, n * s, eps,
                            options=device.pilot_options(pvals), rx_samples=x.numel())
    device.check_desc(desc)
    pv = _PILOTS.get(pvals, dev)
    with device.on_stream(stream):
        H = torch.empty((f, n, cfg.fft_len), dtype=torch.complex64, device=dev) if want_h else None
        num = torch.empty((f, n_data, cfg.fft_len), dtype=torch.complex64, device=dev)
        den = torch.empty((f, cfg.fft_len), dtype=torch.float32, device=dev)
        flags = torch.zeros((f,), dtype=torch.int32, device=dev)
        _lib.call("ofdmrx_rx_partials", ctypes.byref(desc), device.ptr(x), device.ptr(pv), device.ptr(H),
                  device.ptr(num), device.ptr(den), device.ptr(flags), device.stream_handle(stream))
    return H, num, den, flags


def finish_partials(num_parts, den_parts, qam_order, eps=device.MRC_WEIGHT_FLOOR, stream=None):
    """Sum gathered partials [G, F, D, M] / [G, F, M] over G in the reference
    pairwise-tree order, floor, divide and demap.  Returns (s_hat, weights,
    bits, flags)."""
    g, f, d, m = num_parts.shape
    if tuple(den_parts.shape) != (g, f, m):
        raise ContractError(f"den partials {tuple(den_parts.shape)} do not match num {tuple(num_parts.shape)}")
    dev = num_parts.device
    qb = device.qam_bits(qam_order)
    with device.on_stream(stream):
        nump, denp = num_parts.contiguous(), den_parts.contiguous()
        s_hat = torch.empty((f, d, m), dtype=torch.complex64, device=dev)
        weights = torch.empty((f, m), dtype=torch.float32, device=dev)
        bits = torch.empty((f, d * m * qb), dtype=torch.uint8, device=dev)
        flags = torch.zeros((f,), dtype=torch.int32, device=dev)
        _lib.call("ofdmrx_mrc_finish", f, d, m, int(qam_order), g, device.ptr(nump), device.ptr(denp), float(eps),
                  device.ptr(s_hat), device.ptr(weights), device.ptr(bits), device.ptr(flags),
                  device.stream_handle(stream))
    return s_hat, weights, bits, flags


def fft_symbols(rx, cfg, *, symbol0_offset=0, n_data=None, first_symbol=0, n_symbols=None, stream=None):
    """Staged stage 1 over a batch: Y [F, S, N, M] (CP dropped, FFT, fftshift)."""
    dev = device.require_cuda(rx.device if isinstance(rx, torch.Tensor) and rx.is_cuda else None)
    x = device.as_c64(rx, dev)
    if x.dim() == 2:
        x = x[None]
    f, n, s = x.shape
    if n_data is None:
        n_data = (s - symbol0_offset) // cfg.symbol_len - 1
    if n_symbols is None:
        n_symbols = 1 + n_data - first_symbol
    desc = device.make_desc(f, n, cfg.fft_len, cfg.cp_len, n_data, cfg.qam_order, symbol0_offset, s, n * s,
                            rx_samples=x.numel())
    device.check_desc(desc)
    y = torch.empty((f, n_symbols, n, cfg.fft_len), dtype=torch.complex64, device=dev)
    _lib.call("ofdmrx_fft_shift", ctypes.byref(desc), int(first_symbol), int(n_symbols), device.ptr(x),
              device.ptr(y), device.stream_handle(stream))
    return y


class StreamingReceiver:
    """Pipelined host-to-host receive through the public API (SURVEY.md §8(f)
    #2: the paper's bottleneck was the CPU<->GPU transfer).

    Frames stream from pinned host memory in chunks: chunk i+1's H2D copy (copy
    stream) overlaps chunk i's fused kernel (compute stream) and chunk i-1's
    D2H of bits (+ optionally s_hat) on a third stream.  Double-buffered device
    staging; `run` blocks until every result is back in host memory."""

    def __init__(self, cfg, chunk_frames, n_data, symbol0_offset=0, samples_per_row=None, pilot=None,
                 copy_s_hat=False, device_index=None):
        self.cfg = cfg
        self.fc = int(chunk_frames)
        self.n_data = int(n_data)
        self.s0 = int(symbol0_offset)
        self.samples = int(samples_per_row or symbol0_offset + (1 + n_data) * cfg.symbol_len)
        self.pilot = pilot
        self.copy_s_hat = copy_s_hat
        self.dev = device.require_cuda(None if device_index is None else f"cuda:{device_index}")
        shape = (self.fc, cfg.n_antennas, 1 + self.n_data, cfg.fft_len)  # CP never crosses PCIe
        self.x = [torch.empty(shape, dtype=torch.complex64, device=self.dev) for _ in range(2)]
        self.out = [allocate_outputs(self.fc, cfg.n_antennas, cfg.fft_len, self.n_data, cfg.qam_order, self.dev,
                                     want_h=False) for _ in range(2)]
        self.s_h2d = torch.cuda.Stream(self.dev)
        self.s_comp = torch.cuda.Stream(self.dev)
        self.s_d2h = torch.cuda.Stream(self.dev)
        self.ev_in = [torch.cuda.Event() for _ in range(2)]
        self.ev_done = [torch.cuda.Event() for _ in range(2)]
        self.ev_out = [torch.cuda.Event() for _ in range(2)]

    def run(self, host_rx, host_bits, host_s_hat=None):
        """host_rx: pinned complex64 [F, N, S]; host_bits: pinned uint8 [F, D*M*b]."""
        F = host_rx.shape[0]
        n_chunks = (F + self.fc - 1) // self.fc
        for c in range(n_chunks):
            b = c & 1
            lo, hi = c * self.fc, min(F, (c + 1) * self.fc)
            n = hi - lo
            with torch.cuda.stream(self.s_h2d):
                if c >= 2:
                    self.s_h2d.wait_event(self.ev_done[b])  # kernel of chunk c-2 done with x[b]
                stage_symbols(host_rx[lo:hi], self.cfg, symbol0_offset=self.s0, n_data=self.n_data,
                              dst=self.x[b][:n], stream=self.s_h2d)
                self.ev_in[b].record(self.s_h2d)
            with torch.cuda.stream(self.s_comp):
                self.s_comp.wait_event(self.ev_in[b])
                if c >= 2:
                    self.s_comp.wait_event(self.ev_out[b])  # D2H of chunk c-2 done with out[b]
                receive_staged(self.x[b][:n], self.cfg, self.pilot, out=_slice_batch(self.out[b], n),
                               stream=self.s_comp)
                self.ev_done[b].record(self.s_comp)
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(self.ev_done[b])
                host_bits[lo:hi].copy_(self.out[b].bits[:n], non_blocking=True)
                if host_s_hat is not None:
                    host_s_hat[lo:hi].copy_(self.out[b].s_hat[:n], non_blocking=True)
                self.ev_out[b].record(self.s_d2h)
        self.s_d2h.synchronize()


def _slice_batch(out, n):
    return FrameBatch(H=None, s_hat=out.s_hat[:n], weights=out.weights[:n], bits=out.bits[:n], flags=out.flags[:n])


def receive_captures(rx, cfg, n_data, pn=None, pilot=None, *, threshold=None, eps=device.MRC_WEIGHT_FLOOR,
                     want_h=True, zf=False, shards=None, antennas="first", stream=None):
    """Raw captures -> bits with the packet timing found on the device.

    The reference's detect_packet -> extract_slots -> run_ring_pipeline chain
    (cli.py:306-321; sync.py:26-44, receiver.py:274-348) for F captures
    [F, N, S] in two launches and no host round trip: sync.detect_frames, then
    the fused receive with each frame's symbol0 = its antenna-0 peak + PN
    length.  Frames whose peak is below `threshold` get FLAG_NOT_DETECTED,
    frames too short for 1 + n_data symbols after the peak FLAG_OUT_OF_RANGE;
    both are skipped.  The decision only needs antenna 0 (sync.py:37-42), so
    by default only antenna 0 is correlated (antennas="all" also reports every
    antenna's peak).  Returns (FrameBatch, FrameDetections)."""
    from . import sync
    from .synth import generate_pn_chips

    cfg = as_config(cfg)
    dev = device.require_cuda(rx.device if isinstance(rx, torch.Tensor) and rx.is_cuda else None)
    x = device.as_c64(rx, dev)
    if x.dim() == 2:
        x = x[None]
    f, n, s = x.shape
    if n != cfg.n_antennas:
        raise ContractError(f"rx has {n} antenna rows, config has {cfg.n_antennas}")
    chips = generate_pn_chips(length=cfg.pn_len) if pn is None else pn
    thr = sync.DEFAULT_THRESHOLD if threshold is None else float(threshold)
    det = sync.detect_frames(x, chips, thr, antennas=antennas, stream=stream)
    pvals = _pilot_values(pilot, cfg.fft_len)
    desc = device.make_desc(f, n, cfg.fft_len, cfg.cp_len, n_data, cfg.qam_order, 0, s, n * s, eps,
                            options=device.pilot_options(pvals), rx_samples=x.numel())
    pv = _PILOTS.get(pvals, dev)
    with device.on_stream(stream):  # outputs zeroed on the stream the detection + receive run on
        out = allocate_outputs(f, n, cfg.fft_len, n_data, cfg.qam_order, dev, want_h=want_h, zf=zf)
        _lib.call("ofdmrx_rx_frames_detected", ctypes.byref(desc), s, device.ptr(det.peak_index),
                  device.ptr(det.peak_metric), det.peak_index.shape[1], det.n_chips, thr, device.ptr(x),
                  device.ptr(pv), device.ptr(out.H), device.ptr(out.s_hat), device.ptr(out.weights),
                  device.ptr(out.bits), device.ptr(out.zf), device.ptr(out.flags), device.stream_handle(stream))
    return out, det
