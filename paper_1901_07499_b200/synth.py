"""Synthetic uplink captures for benchmarks and examples.

Restates the reference transmitter and channel simulator — build_frame
(waveform.py:260-286), ofdm_modulate (248-257), generate_pn (77-117) and
apply_channel (channel.py:72-108) — consuming the same random streams
(payload default_rng(seed), per-antenna default_rng([seed, antenna])), so a
capture equals the reference's up to the IFFT rounding (np.fft here, the
reference's radix-2 loop there; ~1e-16 relative).  Out of the hot path:
inputs are generated on the host once and tiled on the device.
"""

import math
from dataclasses import dataclass

import numpy as np

from .waveform import OfdmConfig, make_pilot, qam_map

DEFAULT_PN_TAPS = (8, 6, 5, 4)


def generate_pn_chips(taps=DEFAULT_PN_TAPS, seed=1, length=255):
    """Bipolar m-sequence (waveform.py:77-117)."""
    taps = tuple(sorted(set(int(t) for t in taps), reverse=True))
    degree = taps[0]
    state = seed
    bits = np.empty(length, dtype=np.uint8)
    for n in range(length):
        bits[n] = (state >> (degree - 1)) & 1
        fb = 0
        for t in taps:
            fb ^= (state >> (t - 1)) & 1
        state = ((state << 1) & ((1 << degree) - 1)) | fb
    return np.where(bits == 1, 1.0, -1.0)


def ofdm_modulate(rows, cp_len):
    """waveform.py:248-257 with np.fft for the inverse transform."""
    rows = np.atleast_2d(np.asarray(rows, dtype=np.complex128))
    m = rows.shape[1]
    half = m // 2
    shifted = np.concatenate([rows[:, half:], rows[:, :half]], axis=1)
    t = np.fft.ifft(shifted, axis=1) * math.sqrt(m)
    return np.hstack([t[:, m - cp_len:], t]) if cp_len else t


@dataclass
class Capture:
    streams: np.ndarray   # [N, S] complex128
    tx_bits: np.ndarray   # payload bits
    symbol0_offset: int   # first OFDM symbol (after the PN preamble)
    gains: np.ndarray     # per-antenna flat gains (truth)


def synth_capture(cfg: OfdmConfig, n_data, seed, snr_db=10.0, mode="flat_rayleigh", pilot=None):
    """One capture: PN | pilot | n_data data symbols through the channel."""
    b = cfg.bits_per_qam_symbol
    bits = np.random.default_rng(seed).integers(0, 2, size=n_data * cfg.fft_len * b, dtype=np.uint8)
    pilot = make_pilot(cfg.fft_len) if pilot is None else pilot
    grid = qam_map(bits, cfg.qam_order).reshape(n_data, cfg.fft_len)
    pn = generate_pn_chips(length=cfg.pn_len) if cfg.pn_len == 255 else generate_pn_chips(length=cfg.pn_len)
    tx = np.concatenate([pn.astype(np.complex128), ofdm_modulate(pilot.values, cfg.cp_len)[0],
                         ofdm_modulate(grid, cfg.cp_len).ravel()])
    n = tx.shape[0]
    streams = np.empty((cfg.n_antennas, n), dtype=np.complex128)
    gains = np.empty(cfg.n_antennas, dtype=np.complex128)
    for a in range(cfg.n_antennas):
        rng = np.random.default_rng([int(seed), int(a)])
        if mode == "flat_rayleigh":
            g = (rng.standard_normal() + 1j * rng.standard_normal()) / math.sqrt(2.0)
        else:
            g = 1.0 + 0j
        gains[a] = g
        sig = g * tx
        if snr_db is None:
            streams[a] = sig
            continue
        p_sig = float(np.mean(np.abs(sig) ** 2))
        scale = math.sqrt(p_sig / (10.0 ** (snr_db / 10.0)) / 2.0)
        streams[a] = sig + scale * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
    return Capture(streams=streams, tx_bits=bits, symbol0_offset=pn.shape[0], gains=gains)


def synth_batch(cfg: OfdmConfig, n_data, seeds, snr_db=10.0, mode="flat_rayleigh", strip_preamble=True):
    """Stack captures into a complex64 [K, N, L] array (L = (1+D)*(M+C) when
    the preamble is stripped, so symbol0_offset = 0).  Returns (rx, bits[K])."""
    caps = [synth_capture(cfg, n_data, int(s), snr_db, mode) for s in seeds]
    off = caps[0].symbol0_offset if strip_preamble else 0
    L = (1 + n_data) * cfg.symbol_len
    rx = np.stack([c.streams[:, off: off + L] if strip_preamble else c.streams for c in caps])
    return rx.astype(np.complex64), np.stack([c.tx_bits for c in caps]), (0 if strip_preamble else caps[0].symbol0_offset)


# ---------------------------------------------------------------------------
# Device synthesizer: build_frame + apply_channel as
# sm_100a kernels (csrc/synth.cu) behind ofdmrx_synth_frames.
# ---------------------------------------------------------------------------

CHANNEL_MODES = ("identity", "fixed_gains", "flat_rayleigh", "multipath")  # channel.py:13


@dataclass
class DeviceFrames:
    """A synthesised batch on the GPU."""

    rx: "object"             # torch complex64 [F, N, S]
    bits: "object"           # torch uint8 [F, D*M*b] payload (PipelineResult truth)
    response: "object"       # torch complex64 [F or 1, N, T] channel response used
    symbol0_offset: int      # timing_offset + PN length
    frame_start: int         # timing_offset


def synth_frames(cfg: OfdmConfig, n_data, n_frames, *, seed=0, snr_db=10.0, mode="flat_rayleigh",
                 timing_offset=0, bits=None, gains=None, taps=None, pilot=None, pn=None, n_samples=None,
                 stream=None):
    """Synthesize F captures on the current CUDA device.

    Mirrors waveform.build_frame (payload bits exactly filling ``n_data``
    symbols) + channel.apply_channel with ChannelModel(mode, gains, taps,
    snr_db, timing_offset): ``gains`` [N] for fixed_gains, ``taps`` [N, T]
    for multipath, flat_rayleigh draws CN(0,1) per (frame, antenna).
    ``bits`` (uint8 [F, D*M*b], numpy or torch) default to device-drawn fair
    bits.  snr_db=None is noiseless.  Returns DeviceFrames."""
    import ctypes

    import torch

    from . import _lib, device
    from .errors import ConfigurationError, ContractError

    if mode not in CHANNEL_MODES:
        raise ConfigurationError(f"channel mode must be one of {CHANNEL_MODES}")
    if timing_offset < 0:
        raise ConfigurationError("timing_offset must be >= 0")
    dev = device.require_cuda()
    f, n, m = int(n_frames), cfg.n_antennas, cfg.fft_len
    nb = n_data * m * cfg.bits_per_qam_symbol
    st = device.stream_handle(stream)
    if bits is None:
        bits_t = torch.empty((f, nb), dtype=torch.uint8, device=dev)
        _lib.call("ofdmrx_synth_bits", device.ptr(bits_t), f, nb, int(seed), st)
    else:
        bits_t = torch.as_tensor(np.asarray(bits.cpu() if isinstance(bits, torch.Tensor) else bits,
                                            dtype=np.uint8)).reshape(f, nb).to(dev).contiguous()
    if mode == "identity":
        resp = torch.ones((1, n, 1), dtype=torch.complex64, device=dev)
    elif mode == "fixed_gains":
        if gains is None or len(gains) != n:
            raise ConfigurationError("fixed_gains needs one gain per antenna")
        resp = torch.from_numpy(np.asarray(gains, dtype=np.complex64).reshape(1, n, 1)).to(dev)
    elif mode == "flat_rayleigh":
        resp = torch.empty((f, n, 1), dtype=torch.complex64, device=dev)
        _lib.call("ofdmrx_synth_rayleigh", device.ptr(resp), f * n, int(seed), st)
    else:
        t = np.asarray(taps, dtype=np.complex64)
        if t.ndim != 2 or t.shape[0] != n:
            raise ConfigurationError("multipath needs taps [n_antennas, T]")
        resp = torch.from_numpy(np.ascontiguousarray(t)[None]).to(dev)
    pv = pilot.values if pilot is not None and hasattr(pilot, "values") else pilot
    pv = make_pilot(m).values if pv is None else np.asarray(pv)
    if pv.shape != (m,):
        raise ContractError(f"pilot has {pv.shape} values, config needs ({m},)")
    chips = generate_pn_chips(length=cfg.pn_len) if pn is None else np.asarray(getattr(pn, "chips", pn), float)
    from .frames import _PILOTS
    from .sync import _CHIPS

    pilot_t = _PILOTS.get(pv, dev)   # cached device copies: no H2D inside a graph capture
    chips_t = _CHIPS.get(chips, dev)
    frame_len = chips.size + (1 + n_data) * cfg.symbol_len
    s = int(n_samples) if n_samples is not None else timing_offset + frame_len
    rx = torch.empty((f, n, s), dtype=torch.complex64, device=dev)
    desc = _lib.SynthDesc(f, n, m, cfg.cp_len, int(n_data), cfg.qam_order, int(chips.size), int(resp.shape[2]),
                          int(resp.shape[0] > 1 or mode == "flat_rayleigh"), int(snr_db is not None),
                          float(snr_db if snr_db is not None else 0.0), int(timing_offset), s, int(seed))
    _lib.call("ofdmrx_synth_frames", ctypes.byref(desc), device.ptr(pilot_t), device.ptr(chips_t),
              device.ptr(bits_t), device.ptr(resp), device.ptr(rx), st)
    return DeviceFrames(rx=rx, bits=bits_t, response=resp, symbol0_offset=int(timing_offset + chips.size),
                        frame_start=int(timing_offset))
