"""CPU oracle for the uplink OFDM receive hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference receiver
(``ofdmrx``, /root/reference/pkg/src/ofdmrx) for the path the B200 build
replaces.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it,
and only as the checker / the CPU baseline — never as a product code path.
The product (``paper_1901_07499_b200``) fails loudly when its CUDA library
is missing instead of falling back to anything in here.

Parity is pinned: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by the reference itself
(``tests/golden/make_golden.py``, run in the build container where
/root/reference is importable with ``OFDMRX_BACKEND=numpy``).  The oracle
follows the reference's numpy backend operation-for-operation, so on the same
complex128 inputs it reproduces the reference outputs bit-for-bit.

Every function cites the reference file:line it restates (paths relative to
/root/reference/pkg/src/ofdmrx).
"""

import math

import numpy as np

MRC_WEIGHT_FLOOR = 1e-12          # receiver.py:33
QAM_ORDERS = (4, 16, 64)          # waveform.py:20
CANONICAL_CP = {64: 16, 1024: 72}  # waveform.py:18
DEFAULT_PILOT_SEED = 20519        # waveform.py:15
DEFAULT_PN_TAPS = (8, 6, 5, 4)    # waveform.py:13
DEFAULT_PN_SEED = 1               # waveform.py:14


def default_cp(fft_len):
    """waveform.py:57-59."""
    return CANONICAL_CP.get(fft_len, max(1, fft_len // 8))


# ---------------------------------------------------------------------------
# FFT core (kernels/numpy_backend.py:14-45, numerics.py:57-64)
# ---------------------------------------------------------------------------

def _bit_reverse_indices(n):
    """kernels/numpy_backend.py:14-20."""
    bits = n.bit_length() - 1
    idx = np.arange(n, dtype=np.int64)
    rev = np.zeros(n, dtype=np.int64)
    for b in range(bits):
        rev |= ((idx >> b) & 1) << (bits - 1 - b)
    return rev


def fft_rows(mat, inverse=False):
    """Radix-2 DIT transform of every row (kernels/numpy_backend.py:23-45).

    Forward is unnormalized (sign -1), inverse carries 1/n."""
    mat = np.ascontiguousarray(mat, dtype=np.complex128)
    rows, n = mat.shape
    out = mat[:, _bit_reverse_indices(n)].copy()
    sign = 1.0 if inverse else -1.0
    size = 2
    while size <= n:
        half = size // 2
        tw = np.exp(sign * 2j * np.pi * np.arange(half) / size)
        work = out.reshape(rows, n // size, size)
        upper = work[:, :, :half].copy()
        lower = work[:, :, half:] * tw
        work[:, :, :half] = upper + lower
        work[:, :, half:] = upper - lower
        size *= 2
    if inverse:
        out /= n
    return out


def fftshift(x):
    """Swap the halves of the last axis (numerics.py:57-64)."""
    x = np.asarray(x)
    half = x.shape[-1] // 2
    return np.concatenate([x[..., half:], x[..., :half]], axis=-1)


def dft_direct(x):
    """O(n^2) forward DFT (numerics.py:67-73)."""
    x = np.ascontiguousarray(x, dtype=np.complex128)
    n = x.shape[0]
    k = np.arange(n)
    return np.exp(-2j * np.pi * np.outer(k, k) / n) @ x


# ---------------------------------------------------------------------------
# Receive stages (receiver.py:92-99,186-235; kernels/numpy_backend.py:73-107)
# ---------------------------------------------------------------------------

def cp_drop(payload, fft_len, cp_len):
    """receiver.py:186-193 (view of columns cp_len: of each antenna row)."""
    payload = np.atleast_2d(payload)
    assert payload.shape[1] == fft_len + cp_len
    return payload[:, cp_len:]


def freq_transform(time_matrix):
    """SequentialEngine.freq_transform (receiver.py:92-93): fft then shift."""
    return fftshift(fft_rows(time_matrix))


def ls_divide(freq_matrix, pilot_values):
    """SequentialEngine.ls_divide (receiver.py:95-96)."""
    return freq_matrix / pilot_values[None, :]


def tree_reduce_rows(mat):
    """Pairwise tree over axis 0, odd row carried (numpy_backend.py:73-83)."""
    acc = np.asarray(mat, dtype=np.complex128)
    while acc.shape[0] > 1:
        cnt = acc.shape[0]
        half = cnt // 2
        merged = acc[0 : 2 * half : 2] + acc[1 : 2 * half : 2]
        if cnt % 2:
            merged = np.concatenate([merged, acc[-1:]], axis=0)
        acc = merged
    return acc[0]


def mrc_tree(ymat, hmat, eps=MRC_WEIGHT_FLOOR):
    """MRC with the pairwise antenna tree (numpy_backend.py:86-94)."""
    ymat = np.asarray(ymat, dtype=np.complex128)
    hmat = np.asarray(hmat, dtype=np.complex128)
    num = np.conj(hmat) * ymat
    den = hmat.real**2 + hmat.imag**2
    num_sum = tree_reduce_rows(num)
    den_sum = tree_reduce_rows(den).real
    weights = den_sum.copy()
    np.maximum(den_sum, eps, out=den_sum)
    return num_sum / den_sum, weights


def mrc_seq(ymat, hmat, eps=MRC_WEIGHT_FLOOR):
    """MRC accumulating antennas in index order (numpy_backend.py:97-107)."""
    ymat = np.asarray(ymat, dtype=np.complex128)
    hmat = np.asarray(hmat, dtype=np.complex128)
    nant, ncar = ymat.shape
    num = np.zeros(ncar, dtype=np.complex128)
    den = np.zeros(ncar, dtype=np.float64)
    for n in range(nant):
        num += np.conj(hmat[n]) * ymat[n]
        den += hmat[n].real ** 2 + hmat[n].imag ** 2
    weights = den.copy()
    np.maximum(den, eps, out=den)
    return num / den, weights


def zf_per_antenna(ymat, hmat, eps=MRC_WEIGHT_FLOOR):
    """Per-antenna ZF output.  The reference has no ZF; for a
    single-user SIMO link ZF on one antenna is mrc_combine on a 1-row slice
    (receiver.py:221-235), which is what this restates."""
    ymat = np.asarray(ymat, dtype=np.complex128)
    hmat = np.asarray(hmat, dtype=np.complex128)
    out = np.empty_like(ymat)
    for n in range(ymat.shape[0]):
        out[n] = mrc_seq(ymat[n : n + 1], hmat[n : n + 1], eps)[0]
    return out


# ---------------------------------------------------------------------------
# QAM (waveform.py:124-197)
# ---------------------------------------------------------------------------

def _gray_decode(g):
    """waveform.py:124-130."""
    i = g
    g >>= 1
    while g:
        i ^= g
        g >>= 1
    return i


def build_constellation(order):
    """waveform.py:133-151 -> (table, scale, axis_bits, levels)."""
    bits_per = int(math.log2(order))
    axis_bits = bits_per // 2
    levels = 1 << axis_bits
    mean_axis_power = np.mean([(levels - 1 - 2 * i) ** 2 for i in range(levels)])
    scale = 1.0 / math.sqrt(2.0 * mean_axis_power)
    table = np.empty(order, dtype=np.complex128)
    for value in range(order):
        i_bits = value >> axis_bits
        q_bits = value & (levels - 1)
        table[value] = complex(
            (levels - 1) - 2 * _gray_decode(i_bits),
            (levels - 1) - 2 * _gray_decode(q_bits),
        ) * scale
    return table, scale, axis_bits, levels


_CONST = {order: build_constellation(order) for order in QAM_ORDERS}


def qam_map(bits, order):
    """waveform.py:164-176."""
    table = _CONST[order][0]
    bits = np.asarray(bits, dtype=np.uint8).ravel()
    bits_per = int(math.log2(order))
    assert bits.size % bits_per == 0
    groups = bits.reshape(-1, bits_per)
    weights = 1 << np.arange(bits_per - 1, -1, -1)
    return table[groups @ weights]


def qam_demap(symbols, order):
    """Per-axis slicer with Gray code (waveform.py:179-197)."""
    _, scale, axis_bits, levels = _CONST[order]
    symbols = np.asarray(symbols, dtype=np.complex128).ravel() / scale
    ranks_i = np.clip(np.round(((levels - 1) - symbols.real) / 2), 0, levels - 1)
    ranks_q = np.clip(np.round(((levels - 1) - symbols.imag) / 2), 0, levels - 1)
    ranks_i = ranks_i.astype(np.int64)
    ranks_q = ranks_q.astype(np.int64)
    code_i = ranks_i ^ (ranks_i >> 1)
    code_q = ranks_q ^ (ranks_q >> 1)
    out = np.empty((symbols.size, 2 * axis_bits), dtype=np.uint8)
    for b in range(axis_bits):
        shift = axis_bits - 1 - b
        out[:, b] = (code_i >> shift) & 1
        out[:, axis_bits + b] = (code_q >> shift) & 1
    return out.ravel()


# ---------------------------------------------------------------------------
# Pilot, PN and TX synthesis (input generation for the tests)
# waveform.py:77-117,214-220,248-286; channel.py:42-108
# ---------------------------------------------------------------------------

def make_pilot(fft_len, seed=DEFAULT_PILOT_SEED):
    """waveform.py:214-220 (BPSK +-1, complex128)."""
    rng = np.random.default_rng(seed)
    return np.where(rng.integers(0, 2, size=fft_len) == 1, 1.0, -1.0).astype(np.complex128)


def generate_pn(taps=DEFAULT_PN_TAPS, seed=DEFAULT_PN_SEED, length=255):
    """Fibonacci LFSR m-sequence, bipolar (waveform.py:77-117)."""
    taps = tuple(sorted(set(int(t) for t in taps), reverse=True))
    degree = taps[0]
    state = seed
    bits = np.empty(length, dtype=np.uint8)
    for n in range(length):
        bits[n] = (state >> (degree - 1)) & 1
        feedback = 0
        for t in taps:
            feedback ^= (state >> (t - 1)) & 1
        state = ((state << 1) & ((1 << degree) - 1)) | feedback
    return np.where(bits == 1, 1.0, -1.0)


def ofdm_modulate(subcarrier_rows, cp_len):
    """waveform.py:248-257: un-shift, inverse radix-2 FFT, x sqrt(M), prepend CP."""
    rows = np.atleast_2d(np.asarray(subcarrier_rows, dtype=np.complex128))
    fft_len = rows.shape[1]
    time = fft_rows(fftshift(rows), inverse=True)
    time *= math.sqrt(fft_len)
    return np.hstack([time[:, fft_len - cp_len :], time]) if cp_len else time


def build_frame_samples(fft_len, cp_len, qam_order, pilot, payload_bits, pn_chips):
    """waveform.py:260-286 -> (samples, tx_qam, n_data)."""
    payload_bits = np.asarray(payload_bits, dtype=np.uint8).ravel()
    tx_qam = qam_map(payload_bits, qam_order)
    n_data = -(-tx_qam.size // fft_len)
    pad = n_data * fft_len - tx_qam.size
    grid = np.concatenate([tx_qam, np.zeros(pad, dtype=np.complex128)]).reshape(n_data, fft_len)
    samples = np.concatenate([
        pn_chips.astype(np.complex128),
        ofdm_modulate(pilot, cp_len)[0],
        ofdm_modulate(grid, cp_len).ravel(),
    ])
    return samples, tx_qam, n_data


def apply_channel(tx, n_antennas, mode="identity", snr_db=None, timing_offset=0,
                  rng_seed=0, gains=None, taps=None):
    """channel.py:72-108 (per-antenna rng default_rng([seed, antenna]))."""
    n_samples = tx.shape[0] + timing_offset
    streams = np.empty((n_antennas, n_samples), dtype=np.complex128)
    truth = []
    for antenna in range(n_antennas):
        rng = np.random.default_rng([int(rng_seed), int(antenna)])
        if mode == "identity":
            response = np.ones(1, dtype=np.complex128)
        elif mode == "fixed_gains":
            response = np.array([gains[antenna]], dtype=np.complex128)
        elif mode == "flat_rayleigh":
            g = (rng.standard_normal() + 1j * rng.standard_normal()) / math.sqrt(2.0)
            response = np.array([g], dtype=np.complex128)
        else:
            response = np.asarray(taps[antenna], dtype=np.complex128)
        if response.size == 1:
            signal = response[0] * tx
        else:
            signal = np.convolve(tx, response)[: tx.shape[0]]
        truth.append(response.copy())
        if snr_db is None:
            noise_scale = 0.0
        else:
            signal_power = float(np.mean(np.abs(signal) ** 2))
            noise_power = signal_power / (10.0 ** (snr_db / 10.0))
            noise_scale = math.sqrt(noise_power / 2.0)
        if noise_scale > 0.0:
            noise = noise_scale * (
                rng.standard_normal(n_samples) + 1j * rng.standard_normal(n_samples)
            )
        else:
            noise = np.zeros(n_samples, dtype=np.complex128)
        streams[antenna, :timing_offset] = noise[:timing_offset]
        streams[antenna, timing_offset:] = signal + noise[timing_offset:]
    return streams, truth


def synth_capture(fft_len, cp_len, n_antennas, qam_order, n_data, frame_seed,
                  snr_db=10.0, mode="flat_rayleigh"):
    """One capture per SURVEY.md §8(d): payload default_rng(seed) exactly
    filling n_data symbols, make_pilot, generate_pn, build_frame, apply_channel
    with rng_seed=seed.  Returns (streams [N, S] c128, payload bits, symbol0)."""
    bits_per = int(math.log2(qam_order))
    bits = np.random.default_rng(frame_seed).integers(
        0, 2, size=n_data * fft_len * bits_per, dtype=np.uint8)
    pn = generate_pn()
    samples, _, nd = build_frame_samples(fft_len, cp_len, qam_order,
                                         make_pilot(fft_len), bits, pn)
    assert nd == n_data
    streams, _ = apply_channel(samples, n_antennas, mode=mode, snr_db=snr_db,
                               timing_offset=0, rng_seed=frame_seed)
    return streams, bits, pn.shape[0]


# ---------------------------------------------------------------------------
# Whole-frame pipeline (receiver.py:238-267,274-291,308-348)
# ---------------------------------------------------------------------------

def receive_frame(streams, symbol0, fft_len, cp_len, n_data, qam_order,
                  pilot=None, order="seq"):
    """One frame through extract_slots -> process_symbol for 1 pilot + n_data
    data symbols.  Returns (H [N,M], s_hat [D,M], weights [M], bits [D*M*b])."""
    pilot = make_pilot(fft_len) if pilot is None else pilot
    sym_len = fft_len + cp_len
    mrc = mrc_seq if order == "seq" else mrc_tree
    H = None
    s_hat = []
    weights = None
    bits = []
    for s in range(1 + n_data):
        lo = symbol0 + s * sym_len
        payload = streams[:, lo : lo + sym_len]
        freq = freq_transform(np.ascontiguousarray(cp_drop(payload, fft_len, cp_len)))
        if s == 0:
            H = ls_divide(freq, pilot)
        else:
            eq, w = mrc(freq, H)
            s_hat.append(eq)
            weights = w
            bits.append(qam_demap(eq, qam_order))
    s_hat = np.array(s_hat).reshape(n_data, fft_len)
    bits = np.concatenate(bits) if bits else np.empty(0, dtype=np.uint8)
    if weights is None:
        weights = np.sum(H.real**2 + H.imag**2, axis=0)
    return H, s_hat, weights, bits


# ---------------------------------------------------------------------------
# PN packet detection (sync.py:26-44; kernels/numpy_backend.py:48-70)
# ---------------------------------------------------------------------------

DEFAULT_THRESHOLD = 0.6  # sync.py:14


def corr_metrics(stream, chips):
    """Normalised sliding correlation |sum chips*conj(window)| / (|chips| |window|)
    per window position (kernels/numpy_backend.py:48-70, np.correlate + cumsum
    energy; windows with denom <= 1e-30 score 0)."""
    stream = np.ascontiguousarray(stream, dtype=np.complex128)
    chips = np.asarray(chips, dtype=np.float64)
    n, p = stream.shape[0], chips.shape[0]
    raw = np.correlate(stream, chips.astype(np.complex128), mode="valid")
    power = np.empty(n + 1, dtype=np.float64)
    power[0] = 0.0
    np.cumsum(stream.real**2 + stream.imag**2, out=power[1:])
    win = power[p:] - power[: n - p + 1]
    np.maximum(win, 0.0, out=win)
    denom = np.sqrt(np.sum(chips**2)) * np.sqrt(win)
    out = np.zeros(n - p + 1, dtype=np.float64)
    ok = denom > 1e-30
    out[ok] = np.abs(raw[ok]) / denom[ok]
    return out


def detect_packet(streams, chips, threshold=DEFAULT_THRESHOLD):
    """sync.detect_packet (sync.py:26-44): per-antenna argmax of corr_metrics;
    the decision uses antenna 0.  Returns (detected, frame_start,
    symbol0_offset, peak_metric, per_antenna_peaks)."""
    streams = np.atleast_2d(streams)
    chips = np.asarray(chips, dtype=np.float64)
    if streams.shape[1] < chips.shape[0]:
        raise ValueError("stream shorter than PN")  # InputError in the reference
    peaks = []
    for a in range(streams.shape[0]):
        m = corr_metrics(streams[a], chips)
        i = int(np.argmax(m))
        peaks.append((i, float(m[i])))
    start, peak = peaks[0]
    return peak >= threshold, start, start + chips.shape[0], peak, tuple(peaks)


# cases of tests/golden/make_golden.py SYNC_CASES (the reference's
# tests/test_sync.py small frame through apply_channel with a timing offset)
SYNC_CASES = [
    ("clean_1000", 1, "identity", None, 1000, 0),
    ("rayleigh20_50_4ant", 4, "flat_rayleigh", 20.0, 50, 1),
    ("zero_db_a", 1, "flat_rayleigh", 0.0, 17, 3),
    ("zero_db_b", 2, "flat_rayleigh", 0.0, 211, 4),
    ("minus6db_8ant", 8, "flat_rayleigh", -6.0, 77, 5),
    ("c3_like_64ant", 64, "flat_rayleigh", 10.0, 0, 6),
]


def sync_capture(n_antennas, mode, snr_db, timing_offset, rng_seed):
    """tests/test_sync.py:10-14 small frame (64/16 QPSK, 4 data symbols from
    default_rng(3)) through channel.apply_channel (channel.py:72-108)."""
    bits = np.random.default_rng(3).integers(0, 2, size=4 * 64 * 2, dtype=np.uint8)
    samples, _, _ = build_frame_samples(64, 16, 4, make_pilot(64), bits, generate_pn())
    streams, _ = apply_channel(samples, n_antennas, mode=mode, snr_db=snr_db,
                               timing_offset=timing_offset, rng_seed=rng_seed)
    return streams
