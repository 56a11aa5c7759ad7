"""Randomised parity sweep of ofdmrx_rx_frames against the oracle: FFT sizes
2..4096, 1..70 antennas, 0..14 data symbols, every QAM order, random CP,
symbol0 offsets (odd sample offsets included), padded rows, ZF on/off and
the throughput / single-frame latency plans, so every kernel path
(rx_balanced at any cluster mapping, rx_fused, the row-parallel latency
path) meets the same bar: bits exact, H / s_hat / weights within 1e-4
relative.  Fixed seed: the same 60 configurations every run."""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import ofdm_oracle as orc  # noqa: E402

REL_TOL = 1e-4


def rel(a, b):
    a = np.asarray(a, np.complex128)
    b = np.asarray(b, np.complex128)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _configs(n=60, seed=20261017):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        m = int(2 ** rng.integers(1, 13))
        n_ant = int(rng.integers(1, 71))
        d = int(rng.integers(0, 15))
        qam = int(rng.choice([4, 16, 64]))
        cp = int(rng.integers(0, max(1, m // 4) + 1)) if m > 2 else int(rng.integers(0, 2))
        cp = min(cp, m - 1)
        nf = int(rng.integers(1, 6))
        if m * n_ant * (d + 1) * nf > 3_000_000:
            continue
        out.append((m, n_ant, d, qam, cp, nf, int(rng.integers(0, 8)), int(rng.integers(0, 5)),
                    bool(rng.integers(0, 2)), bool(rng.integers(0, 2)), int(rng.integers(0, 1 << 30))))
    return out


@pytest.mark.parametrize("cfg", _configs(),
                         ids=lambda c: f"M{c[0]}N{c[1]}D{c[2]}q{c[3]}cp{c[4]}F{c[5]}{'lat' if c[9] else ''}")
def test_fuzz_fused_vs_oracle(cfg):
    import paper_1901_07499_b200 as P

    m, n_ant, d, qam, cp, nf, off, pad, zf, latency, seed = cfg
    rng = np.random.default_rng(seed)
    b = int(math.log2(qam))
    pilot = orc.make_pilot(m)
    pn = orc.generate_pn()
    s_len = off + 255 + (1 + d) * (m + cp) + pad
    streams = np.zeros((nf, n_ant, s_len), dtype=np.complex128)
    for f in range(nf):
        bits = rng.integers(0, 2, size=max(d, 1) * m * b, dtype=np.uint8)
        tx, _, nd = orc.build_frame_samples(m, cp, qam, pilot, bits, pn)
        tx = tx[: 255 + (1 + d) * (m + cp)]
        st, _ = orc.apply_channel(tx, n_ant, mode="flat_rayleigh", snr_db=float(rng.uniform(10, 25)),
                                  rng_seed=seed + f)
        streams[f, :, off:off + st.shape[1]] = st
    cfgp = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    x = torch.from_numpy(streams.astype(np.complex64)).cuda()
    out = P.receive_frames(x, cfgp, symbol0_offset=off + 255, n_data=d, zf=zf, latency=latency)
    torch.cuda.synchronize()
    assert int((out.flags & 1).sum()) == 0
    for f in range(nf):
        xf = streams[f].astype(np.complex64).astype(np.complex128)  # the device reads cf32
        H, s_hat, w, bits = orc.receive_frame(xf, off + 255, m, cp, d, qam)
        assert rel(out.H[f].cpu().numpy(), H) < REL_TOL
        if d > 0:
            assert np.array_equal(out.bits[f].cpu().numpy(), bits)
            assert rel(out.s_hat[f].cpu().numpy(), s_hat) < REL_TOL
            assert rel(out.weights[f].cpu().numpy(), w) < REL_TOL
        if zf and d > 0:
            Y = [orc.freq_transform(np.ascontiguousarray(orc.cp_drop(
                xf[:, off + 255 + (1 + j) * (m + cp): off + 255 + (2 + j) * (m + cp)], m, cp))) for j in range(d)]
            zref = np.stack([orc.zf_per_antenna(Yj, H) for Yj in Y])
            assert rel(out.zf[f].cpu().numpy(), zref) < REL_TOL
