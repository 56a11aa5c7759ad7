"""CPU model of the device FFT decomposition (ofdmrx_fft.cuh): the same plans,
Stockham index formulas, padded exchange, bit-reversed DIT register order and
register->subcarrier mapping, checked against the oracle DFT.  This pins the
kernel's indexing design without a GPU; the CUDA kernels are checked against
the oracle in the -m gpu tests."""

import math
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "paper_1901_07499_b200", "csrc"))
from gen_twiddles import PLANS, store_table, table  # noqa: E402

from oracle import ofdm_oracle as orc  # noqa: E402


def brev(x, bits):
    r = 0
    for _ in range(bits):
        r = (r << 1) | (x & 1)
        x >>= 1
    return r


def dit(v):
    r = len(v)
    v = list(v)
    span = 1
    while span < r:
        for blk in range(0, r, 2 * span):
            for j in range(span):
                w = np.exp(-2j * np.pi * j / (2 * span))
                a, b = v[blk + j], v[blk + j + span] * w
                v[blk + j], v[blk + j + span] = a + b, a - b
        span *= 2
    return v


def model_fft(x, m):
    p, g, radices = PLANS[m]
    tw = np.array([complex(c, s) for c, s in table(m)])
    tws = np.array([complex(c, s) for c, s in store_table(m)])
    regs = [[0j] * p for _ in range(g)]
    buf = {}
    span, tw_off, prev_r = 1, 0, None
    for pi, r in enumerate(radices):
        nb = p // r
        logr = int(math.log2(r))
        last = pi == len(radices) - 1
        for t in range(g):
            for vv in range(nb):
                b = t + vv * g
                for q in range(r):
                    idx = b + q * (m // r)
                    if pi == 0:
                        val = x[idx]
                    else:
                        val = buf[idx + 2 * (idx >> int(math.log2(prev_r)))]
                    regs[t][vv * r + brev(q, logr)] = val
        if pi >= 2:
            for t in range(g):
                for vv in range(nb):
                    k = (t + vv * g) & (span - 1)
                    for q in range(1, r):
                        regs[t][vv * r + brev(q, logr)] *= tw[(q - 1) * span + k]
        for t in range(g):
            for vv in range(nb):
                regs[t][vv * r:(vv + 1) * r] = dit(regs[t][vv * r:(vv + 1) * r])
        if pi == 0 and not last:
            for t in range(g):
                for rr in range(r):
                    regs[t][rr] *= tws[((rr // 2) * g + t) * 2 + (rr % 2)]
        if not last:
            buf = {}
            for t in range(g):
                for vv in range(nb):
                    b = t + vv * g
                    base = (b // span) * span * r + (b & (span - 1))
                    for rr in range(r):
                        o = base + rr * span
                        buf[o + 2 * (o >> logr)] = regs[t][vv * r + rr]
            assert len(buf) == m
        prev_r = r
        span *= r
    out = np.empty(m, dtype=complex)
    r_last = radices[-1]
    for t in range(g):
        for i in range(p):
            k = t + (i // r_last) * g + (i % r_last) * (m // r_last)
            out[(k + m // 2) % m] = regs[t][i]
    return out


@pytest.mark.parametrize("m", sorted(PLANS))
def test_plan_model_matches_shifted_dft(m):
    rng = np.random.default_rng(m)
    x = rng.standard_normal(m) + 1j * rng.standard_normal(m)
    ref = orc.fftshift(orc.dft_direct(x))
    got = model_fft(x, m)
    assert np.max(np.abs(got - ref)) < 1e-9 * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("m", sorted(PLANS))
def test_exchange_pad_is_bank_friendly(m):
    """Pass-0 128-bit stores of (r, r+1) pairs: each quarter-warp phase (8 lane
    threads) covers 32 distinct banks, and the pairs are 16-B aligned."""
    p, g, radices = PLANS[m]
    if len(radices) == 1:
        return
    r = radices[0]
    logr = int(math.log2(r))
    for rr in range(0, r, 2):
        for phase in range(0, min(g, 32), 8):
            banks = []
            for t in range(phase, min(phase + 8, g)):
                o = t * r + rr
                e = o + 2 * (o >> logr)
                assert e % 2 == 0
                banks += [(2 * e + w) % 32 for w in range(4)]
            assert len(banks) == len(set(banks))
