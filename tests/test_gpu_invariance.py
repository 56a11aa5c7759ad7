"""Batch invariance of the fused receive (include/ofdmrx_b200.h: "Results
never depend on the batch").

A frame's bits, s_hat, H and weights must be bit-identical whether it is
received alone (F = 1: each frame spread over a thread-block cluster of
several SMs), next to other frames, or inside a throughput-sized batch (one
CTA per frame).  The antenna-sum order is fixed by the frame shape only
(ofdmrx_rx_plan "workers"); the tests also assert that the CTA mapping really
changes across the batch sizes, so the equality is not vacuous.  The distinct
frames are checked against the CPU oracle as well (bits exact, 1e-4)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import ofdm_oracle as orc  # noqa: E402

REL_TOL = 1e-4

SHAPES = [
    # (N, M, CP, qam, D, distinct frames, batch sizes)
    (64, 1024, 72, 16, 10, 3, (1, 2, 5, 64, 1024)),   # C3: balanced kernel, 12 workers
    (256, 2048, 256, 64, 10, 2, (1, 2, 16, 64)),      # C4: balanced kernel, M = 2048 lanes of 64 threads
    (8, 64, 16, 4, 10, 3, (1, 2, 64, 4096)),          # C1: fused kernel
    (16, 256, 32, 16, 10, 3, (1, 2, 64, 1000)),       # C2: fused kernel
    (4, 4096, 512, 16, 3, 2, (1, 3, 100)),             # M = 4096: lanes of 128 threads
    (2, 1024, 72, 4, 5, 2, (1, 7, 300)),              # N < workers: lanes without rows
]


def rel(a, b):
    a = np.asarray(a, np.complex128)
    b = np.asarray(b, np.complex128)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"N{s[0]}xM{s[1]}q{s[3]}D{s[4]}")
def test_outputs_independent_of_batch(shape):
    import paper_1901_07499_b200 as P
    from paper_1901_07499_b200 import device

    n_ant, m, cp, qam, d, k, batches = shape
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    caps = [orc.synth_capture(m, cp, n_ant, qam, d, 300 + i, snr_db=10.0) for i in range(k)]
    s0 = caps[0][2]
    host = np.stack([c[0] for c in caps]).astype(np.complex64)
    distinct = torch.from_numpy(host).cuda()
    # reference per frame: each frame received alone (F = 1)
    alone = [P.receive_frames(distinct[i:i + 1], cfg, symbol0_offset=s0, n_data=d) for i in range(k)]
    torch.cuda.synchronize()
    for i in range(k):  # and the alone-results are the oracle's
        H, s_hat, w, bits = orc.receive_frame(host[i].astype(np.complex128), s0, m, cp, d, qam)
        assert np.array_equal(alone[i].bits[0].cpu().numpy(), bits)
        assert rel(alone[i].s_hat[0].cpu().numpy(), s_hat) < REL_TOL
        assert rel(alone[i].H[0].cpu().numpy(), H) < REL_TOL
        assert rel(alone[i].weights[0].cpu().numpy(), w) < REL_TOL
    plans = set()
    for F in batches:
        reps = (F + k - 1) // k
        x = distinct.repeat(reps, 1, 1)[:F].contiguous()
        desc = device.make_desc(F, n_ant, m, cp, d, qam, s0, x.shape[2], n_ant * x.shape[2],
                                options=device.pilot_options(orc.make_pilot(m)), rx_samples=x.numel())
        plan = device.rx_plan(desc)
        plans.add((plan["kernel"], plan["workers"], plan["cluster"], plan["lanes_per_cta"]))
        out = P.receive_frames(x, cfg, symbol0_offset=s0, n_data=d)
        torch.cuda.synchronize()
        assert int(out.flags.abs().sum()) == 0
        for j in range(F):
            ref = alone[j % k]
            assert torch.equal(out.bits[j], ref.bits[0]), f"F={F} frame {j}: bits depend on the batch"
            assert torch.equal(out.s_hat[j], ref.s_hat[0]), f"F={F} frame {j}: s_hat depends on the batch"
            assert torch.equal(out.H[j], ref.H[0]), f"F={F} frame {j}: H depends on the batch"
            assert torch.equal(out.weights[j], ref.weights[0]), f"F={F} frame {j}: weights depend on the batch"
        del x, out
    kernels = {p[0] for p in plans}
    workers = {(p[0], p[1]) for p in plans}
    assert len(kernels) == 1 and len(workers) == 1, f"arithmetic plan changed with the batch: {plans}"
    lanes_max = {1024: 12, 2048: 6, 4096: 3}.get(m, 0)
    if 1 in kernels and next(iter(workers))[1] < 8 * lanes_max:
        # balanced with room for more than one cluster size: the CTA mapping
        # must actually differ across the batch sizes
        assert len({p[2] for p in plans}) > 1, plans


@pytest.mark.parametrize("n_ant,m,cp,qam,d", [(64, 1024, 72, 16, 10), (16, 256, 32, 16, 6), (32, 2048, 256, 64, 4)])
def test_zf_output_does_not_change_s_hat(n_ant, m, cp, qam, d):
    """The per-antenna ZF output is an extra store, not a different kernel:
    s_hat / bits are identical with and without it."""
    import paper_1901_07499_b200 as P

    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    caps = [orc.synth_capture(m, cp, n_ant, qam, d, 400 + i, snr_db=10.0) for i in range(2)]
    s0 = caps[0][2]
    host = np.stack([c[0] for c in caps])
    x = torch.from_numpy(host.astype(np.complex64)).cuda()
    a = P.receive_frames(x, cfg, symbol0_offset=s0, n_data=d)
    b = P.receive_frames(x, cfg, symbol0_offset=s0, n_data=d, zf=True)
    torch.cuda.synchronize()
    assert torch.equal(a.bits, b.bits) and torch.equal(a.s_hat, b.s_hat) and torch.equal(a.H, b.H)
    for f in range(2):
        H = orc.receive_frame(host[f].astype(np.complex64).astype(np.complex128), s0, m, cp, d, qam)[0]
        zf = b.zf[f].cpu().numpy()
        for j in range(d):
            lo = s0 + (j + 1) * (m + cp) + cp
            Y = orc.freq_transform(host[f][:, lo:lo + m].astype(np.complex64).astype(np.complex128))
            assert rel(zf[j], orc.zf_per_antenna(Y, H)) < REL_TOL


def test_partials_independent_of_batch():
    """ofdmrx_rx_partials (the antenna-sharded half) is batch-invariant too."""
    import paper_1901_07499_b200 as P

    n_ant, m, cp, qam, d = 32, 2048, 256, 64, 10
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    caps = [orc.synth_capture(m, cp, n_ant, qam, d, 500 + i, snr_db=10.0) for i in range(2)]
    s0 = caps[0][2]
    x = torch.from_numpy(np.stack([c[0] for c in caps]).astype(np.complex64)).cuda()
    ref = [P.receive_partials(x[i:i + 1], cfg, symbol0_offset=s0, n_data=d) for i in range(2)]
    big = x.repeat(40, 1, 1).contiguous()
    H, num, den, fl = P.receive_partials(big, cfg, symbol0_offset=s0, n_data=d)
    torch.cuda.synchronize()
    for j in range(80):
        r = ref[j % 2]
        assert torch.equal(num[j], r[1][0]) and torch.equal(den[j], r[2][0]) and torch.equal(H[j], r[0][0])


@pytest.mark.parametrize("shape", [(64, 1024, 72, 16, 10), (16, 4096, 512, 16, 3), (256, 2048, 256, 64, 10)],
                         ids=["C3", "M4096", "C4"])
def test_latency_plan(shape):
    """OFDMRX_OPT_LATENCY (receive_frames(latency=True)): the row-parallel
    path (every FFT row its own lane, antenna sums ascending); bits exact vs
    the oracle, H / s_hat / weights within 1e-4; batch-invariant within the
    plan (F = 1, 3, 40); the ZF output and the stage attribution work."""
    import paper_1901_07499_b200 as P
    from paper_1901_07499_b200 import _lib, device

    n_ant, m, cp, qam, d = shape
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    caps = [orc.synth_capture(m, cp, n_ant, qam, d, 700 + i, snr_db=10.0) for i in range(2)]
    s0 = caps[0][2]
    host = np.stack([c[0] for c in caps]).astype(np.complex64)
    x = torch.from_numpy(host).cuda()
    opts = device.pilot_options(orc.make_pilot(m))
    mk = lambda F, o: device.make_desc(F, n_ant, m, cp, d, qam, s0, x.shape[2], n_ant * x.shape[2],  # noqa: E731
                                       options=o, rx_samples=F * n_ant * x.shape[2])
    lat, thr = device.rx_plan(mk(1, opts | _lib.OPT_LATENCY)), device.rx_plan(mk(1, opts))
    assert lat["kernel"] == _lib.KERNEL_ROWS and lat["workers"] == n_ant, lat
    # the partial-sum entry point takes the balanced kernel's widest plan instead
    lat1 = device.rx_plan(mk(1, opts | _lib.OPT_LATENCY), mode=1)
    assert lat1["kernel"] == _lib.KERNEL_BALANCED and lat1["workers"] > thr["workers"], (lat1, thr)
    alone = [P.receive_frames(x[i:i + 1], cfg, symbol0_offset=s0, n_data=d, latency=True) for i in range(2)]
    torch.cuda.synchronize()
    for i in range(2):
        H, s_hat, w, bits = orc.receive_frame(host[i].astype(np.complex128), s0, m, cp, d, qam)
        assert np.array_equal(alone[i].bits[0].cpu().numpy(), bits)
        assert rel(alone[i].s_hat[0].cpu().numpy(), s_hat) < REL_TOL
        assert rel(alone[i].H[0].cpu().numpy(), H) < REL_TOL
        assert rel(alone[i].weights[0].cpu().numpy(), w) < REL_TOL
    for F in (3, 40):
        xb = x.repeat((F + 1) // 2, 1, 1)[:F].contiguous()
        out = P.receive_frames(xb, cfg, symbol0_offset=s0, n_data=d, latency=True)
        torch.cuda.synchronize()
        assert int(out.flags.abs().sum()) == 0
        for j in range(F):
            assert torch.equal(out.bits[j], alone[j % 2].bits[0])
            assert torch.equal(out.s_hat[j], alone[j % 2].s_hat[0])
            assert torch.equal(out.H[j], alone[j % 2].H[0])
    z = P.receive_frames(x, cfg, symbol0_offset=s0, n_data=d, latency=True, zf=True, profile=True)
    torch.cuda.synchronize()
    assert torch.equal(z.bits[0], alone[0].bits[0]) and (z.stage_cycles.cpu().numpy() > 0).all()
    Hh = orc.receive_frame(host[0].astype(np.complex128), s0, m, cp, d, qam)[0]
    for j in range(d):
        lo = s0 + (j + 1) * (m + cp) + cp
        Y = orc.freq_transform(host[0][:, lo:lo + m].astype(np.complex128))
        assert rel(z.zf[0, j].cpu().numpy(), orc.zf_per_antenna(Y, Hh)) < REL_TOL
