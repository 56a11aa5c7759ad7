"""Numerology, pilot and QAM tables of the receive path, mirroring the
reference's waveform.py (waveform.py:15-59,124-220).  ``qam_demap`` runs on
the device (ofdmrx_demap); everything else here is host-side configuration.
The TX-side helpers (qam_map, ofdm_modulate) only feed the synthetic frame
generator in synth.py."""

import math
from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError, FramingError

DEFAULT_PILOT_SEED = 20519          # waveform.py:15
CANONICAL_CP = {64: 16, 1024: 72}    # waveform.py:18
QAM_ORDERS = (4, 16, 64)             # waveform.py:20
MAX_FFT_LEN = 4096                   # device-path limit (ofdmrx_fft.cuh plans)


def is_power_of_two(n):
    """numerics.py:16-17."""
    return n >= 1 and (n & (n - 1)) == 0


@dataclass(frozen=True)
class OfdmConfig:
    """waveform.py:23-54 (same fields, validation and derived properties)."""

    fft_len: int
    cp_len: int
    n_antennas: int
    qam_order: int = 4
    pn_len: int = 255
    sample_rate_hz: float = 10e6

    def __post_init__(self):
        if not is_power_of_two(self.fft_len) or self.fft_len < 2:
            raise ConfigurationError(f"fft_len must be a power of two, got {self.fft_len}")
        if not 0 <= self.cp_len < self.fft_len:
            raise ConfigurationError(
                f"cp_len must satisfy 0 <= cp_len < fft_len, got {self.cp_len}")
        if self.n_antennas < 1:
            raise ConfigurationError(f"n_antennas must be >= 1, got {self.n_antennas}")
        if self.qam_order not in QAM_ORDERS:
            raise ConfigurationError(f"qam_order must be one of {QAM_ORDERS}")
        if self.pn_len < 7 or not is_power_of_two(self.pn_len + 1):
            raise ConfigurationError(f"pn_len must be 2^r - 1 with r >= 3, got {self.pn_len}")

    @property
    def symbol_len(self):
        return self.fft_len + self.cp_len

    @property
    def bits_per_qam_symbol(self):
        return int(math.log2(self.qam_order))


def as_config(cfg):
    """Accept this package's OfdmConfig or any object with the reference
    OfdmConfig's fields (e.g. ofdmrx.waveform.OfdmConfig, waveform.py:23-54),
    so reference-built configs drive the device path unchanged."""
    if isinstance(cfg, OfdmConfig):
        return cfg
    try:
        return OfdmConfig(int(cfg.fft_len), int(cfg.cp_len), int(cfg.n_antennas), qam_order=int(cfg.qam_order),
                          pn_len=int(getattr(cfg, "pn_len", 255)),
                          sample_rate_hz=float(getattr(cfg, "sample_rate_hz", 10e6)))
    except AttributeError as e:
        from .errors import ContractError
        raise ContractError(f"cfg must be an OfdmConfig (missing field: {e})") from None


def default_cp(fft_len):
    """waveform.py:57-59."""
    return CANONICAL_CP.get(fft_len, max(1, fft_len // 8))


def _gray_decode(g):
    i = g
    g >>= 1
    while g:
        i ^= g
        g >>= 1
    return i


def _build_constellation(order):
    """waveform.py:138-151 -> (table, scale, axis_bits, levels)."""
    bits_per = int(math.log2(order))
    axis_bits = bits_per // 2
    levels = 1 << axis_bits
    mean_axis_power = np.mean([(levels - 1 - 2 * i) ** 2 for i in range(levels)])
    scale = 1.0 / math.sqrt(2.0 * mean_axis_power)
    table = np.empty(order, dtype=np.complex128)
    for value in range(order):
        i_bits, q_bits = value >> axis_bits, value & (levels - 1)
        table[value] = complex((levels - 1) - 2 * _gray_decode(i_bits),
                               (levels - 1) - 2 * _gray_decode(q_bits)) * scale
    return table, scale, axis_bits, levels


_CONSTELLATIONS = {order: _build_constellation(order) for order in QAM_ORDERS}


def qam_constellation(order):
    if order not in _CONSTELLATIONS:
        raise ConfigurationError(f"qam order must be one of {QAM_ORDERS}, got {order}")
    return _CONSTELLATIONS[order][0]


def qam_map(bits, order):
    """Gray QAM mapping (waveform.py:164-176); TX side, used by synth.py."""
    table = qam_constellation(order)
    bits = np.asarray(bits, dtype=np.uint8).ravel()
    bits_per = int(math.log2(order))
    if bits.size % bits_per != 0:
        raise FramingError(f"bit count {bits.size} is not a multiple of {bits_per} (order {order})")
    groups = bits.reshape(-1, bits_per)
    return table[groups @ (1 << np.arange(bits_per - 1, -1, -1))]


def qam_demap(symbols, order):
    """Hard decision to bits on the B200 (waveform.py:179-197 semantics):
    numpy in, numpy uint8 0/1 out; torch CUDA tensors in, CUDA tensor out."""
    if order not in _CONSTELLATIONS:
        raise ConfigurationError(f"qam order must be one of {QAM_ORDERS}, got {order}")
    from . import device

    return device.demap(symbols, order)


@dataclass(frozen=True)
class PilotDefinition:
    """waveform.py:204-211."""

    values: np.ndarray

    def __post_init__(self):
        if not np.allclose(np.abs(self.values), 1.0, atol=1e-12):
            raise ConfigurationError("pilot values must all have unit modulus")


def make_pilot(fft_len, seed=DEFAULT_PILOT_SEED):
    """Fixed-seed BPSK pilot (waveform.py:214-220)."""
    rng = np.random.default_rng(seed)
    values = np.where(rng.integers(0, 2, size=fft_len) == 1, 1.0, -1.0).astype(np.complex128)
    return PilotDefinition(values=values)
