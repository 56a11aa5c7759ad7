"""The receive epilogue's full-division redo (ofdmrx_fft.cuh finish_points_qb:
a thread whose num / den or s_hat / scale operands leave the fast path's
guard redoes its points with IEEE division) gives the oracle's results:

* an all-zero capture (num = den = 0 exactly, s_hat = 0 / eps = 0: the
  demap division of every point takes the redo);
* captures scaled by 1e12 (num and den far above 2^40: every thread of the
  s_hat division takes the redo);
* subcarriers whose pilot carries no energy on any antenna (den < eps), the
  reference's erasure case (test_receiver.py:216-223): the other
  subcarriers must be unaffected (the erased ones hold num / eps of fp32
  rounding noise, as in the reference, and are only checked finite).

Each shape runs on the kernel its plan picks (rx_balanced for M = 1024 /
2048, rx_fused for M = 64 / 256); bits must equal the oracle's, s_hat and
weights within 1e-4."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import ofdm_oracle as orc  # noqa: E402

REL_TOL = 1e-4

SHAPES = [  # (N, M, CP, qam, D)
    (64, 1024, 72, 16, 10),   # rx_balanced (C3 shape)
    (16, 2048, 256, 64, 4),   # rx_balanced, M = 2048 lanes
    (16, 256, 32, 16, 10),    # rx_fused, 192-thread CTAs (C2 shape)
    (8, 64, 16, 4, 10),       # rx_fused (C1 shape)
]


def rel(a, b):
    a = np.asarray(a, np.complex128)
    b = np.asarray(b, np.complex128)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def erased_capture(n_ant, m, cp, qam, d, seed):
    """Pilot with zero energy on every 7th subcarrier, random QAM data, identity channel."""
    rng = np.random.default_rng(seed)
    X = np.tile(orc.make_pilot(m), (n_ant, 1))
    X[:, ::7] = 0.0
    rows = [orc.ofdm_modulate(X, cp)]
    qb = int(np.log2(qam))
    for _ in range(d):
        bits = rng.integers(0, 2, size=m * qb).astype(np.uint8)  # one transmitter: same symbols on every antenna
        rows.append(orc.ofdm_modulate(np.tile(orc.qam_map(bits, qam), (n_ant, 1)), cp))
    return np.concatenate(rows, axis=1)


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"N{s[0]}xM{s[1]}q{s[3]}")
def test_epilogue_redo_matches_oracle(shape):
    import paper_1901_07499_b200 as P

    n_ant, m, cp, qam, d = shape
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    cap, _, s0 = orc.synth_capture(m, cp, n_ant, qam, d, 77, snr_db=10.0)
    erased = erased_capture(n_ant, m, cp, qam, d, 5)
    zero = np.zeros_like(cap).astype(np.complex64)
    cases = [(zero, s0, "zero"), ((cap * 1e12).astype(np.complex64), s0, "scaled 1e12"),
             (erased.astype(np.complex64), 0, "erased")]
    qb = int(np.log2(qam))
    keep = np.arange(m) % 7 != 0
    for x, sym0, what in cases:
        out = P.receive_frames(torch.from_numpy(x[None]).cuda(), cfg, symbol0_offset=sym0, n_data=d)
        torch.cuda.synchronize()
        H, s_hat, w, bits = orc.receive_frame(x.astype(np.complex128), sym0, m, cp, d, qam)
        got_bits = out.bits[0].cpu().numpy().reshape(d, m, qb)
        got_s = out.s_hat[0].cpu().numpy()
        sel = keep if what == "erased" else np.ones(m, bool)
        assert np.array_equal(got_bits[:, sel], bits.reshape(d, m, qb)[:, sel]), what
        assert rel(got_s[:, sel], s_hat[:, sel]) < REL_TOL, what
        assert np.all(np.isfinite(got_s)), what
        if what == "zero":
            assert np.all(got_s == 0) and int(out.flags[0]) & 2, what
        if what == "erased":
            assert int(out.flags[0]) & 2, what
