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
