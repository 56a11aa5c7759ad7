"""Parity of the sm_100a kernels (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star): demodulated bits bit-exact; H estimates and
equalised symbols within 1e-4 relative (normwise per frame) in fp32.
"""

import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import ofdm_oracle as orc  # noqa: E402

REL_TOL = 1e-4  # north_star: H and s_hat within 1e-4 relative in fp32


def rel(a, b):
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def P():
    import paper_1901_07499_b200 as P
    from paper_1901_07499_b200 import device

    device.require_cuda()
    return P


def make_batch(m, cp, n_ant, qam, d, seeds, snr=10.0):
    caps = [orc.synth_capture(m, cp, n_ant, qam, d, s, snr_db=snr) for s in seeds]
    streams = np.stack([c[0] for c in caps])
    return streams, [c[1] for c in caps], caps[0][2]


def oracle_frames(streams, s0, m, cp, d, qam, order="seq"):
    return [orc.receive_frame(x, s0, m, cp, d, qam, order=order) for x in streams]


CASES = [
    # (N, M, CP, qam, D, seeds)
    (8, 64, 16, 4, 10, (0, 1, 2, 3)),       # C1
    (16, 256, 32, 16, 10, (0, 1)),          # C2
    (64, 1024, 72, 16, 10, (0, 1)),         # C3
    (4, 2, 1, 4, 3, (5,)),
    (3, 8, 1, 4, 4, (6,)),
    (5, 16, 2, 16, 7, (7,)),
    (2, 32, 4, 64, 5, (8,)),
    (7, 128, 16, 64, 12, (9,)),
    (9, 512, 64, 16, 20, (10,)),
    (8, 2048, 256, 64, 6, (11,)),
    (4, 4096, 512, 16, 3, (12,)),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"N{c[0]}xM{c[1]}q{c[3]}D{c[4]}")
def test_fused_vs_oracle(P, case):
    n_ant, m, cp, qam, d, seeds = case
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    streams, tx_bits, s0 = make_batch(m, cp, n_ant, qam, d, seeds)
    out = P.receive_frames(torch.from_numpy(streams.astype(np.complex64)).cuda(), cfg,
                           symbol0_offset=s0, n_data=d, check=True)
    torch.cuda.synchronize()
    for i, (H, s_hat, w, bits) in enumerate(oracle_frames(streams, s0, m, cp, d, qam)):
        assert np.array_equal(out.bits[i].cpu().numpy(), bits), f"frame {i}: bits differ"
        assert rel(out.H[i].cpu().numpy(), H) < REL_TOL
        assert rel(out.s_hat[i].cpu().numpy(), s_hat) < REL_TOL
        assert rel(out.weights[i].cpu().numpy(), w) < REL_TOL
    assert int(out.flags.abs().sum()) == 0


GOLDEN_SETS = ["C1", "C1_0dB", "C2", "C3", "C3_0dB", "C4", "C4_0dB"]


@pytest.mark.parametrize("tile", [1, 160, "latency"], ids=["alone", "batch160", "latency_path"])
@pytest.mark.parametrize("name", GOLDEN_SETS)
def test_fused_vs_reference_golden(P, golden_dir, name, tile):
    """Directly against vectors produced by the reference itself, with the
    frame received alone (F = 1, spread over a cluster for M >= 1024),
    tiled into a 160-frame batch (one CTA per frame: the benched mapping),
    and alone through the row-parallel latency path (OFDMRX_OPT_LATENCY)."""
    latency = tile == "latency"
    tile = 1 if latency else tile
    g = dict(np.load(os.path.join(golden_dir, f"frames_{name}.npz")))
    n_ant, m, cp, qam, d = (int(v) for v in g["spec"])
    if tile > 1 and n_ant * m > 64 * 1024:
        tile = 40  # C4: 40 x 52 MB
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    for f in g["seeds"]:
        tag = f"f{int(f)}"
        streams, _, s0 = orc.synth_capture(m, cp, n_ant, qam, d, int(f), snr_db=float(g["snr_db"]))
        x = torch.from_numpy(streams.astype(np.complex64)).cuda()[None].repeat(tile, 1, 1).contiguous()
        out = P.receive_frames(x, cfg, symbol0_offset=s0, n_data=d, latency=latency)
        torch.cuda.synchronize()
        if tile > 1:  # every copy identical, then check copy `tile - 1` below
            assert torch.equal(out.bits, out.bits[:1].expand_as(out.bits))
            assert torch.equal(out.s_hat, out.s_hat[:1].expand_as(out.s_hat))
            out = type(out)(H=out.H[tile - 1:], s_hat=out.s_hat[tile - 1:], weights=out.weights[tile - 1:],
                            bits=out.bits[tile - 1:], flags=out.flags[tile - 1:])
        ref_bits = np.unpackbits(g[f"{tag}_bits"])[: d * m * cfg.bits_per_qam_symbol]
        assert np.array_equal(out.bits[0].cpu().numpy(), ref_bits)
        assert rel(out.s_hat[0].cpu().numpy(), g[f"{tag}_s_hat"]) < REL_TOL
        assert rel(out.weights[0].cpu().numpy(), g[f"{tag}_weights"]) < REL_TOL
        H = out.H[0].cpu().numpy()
        if f"{tag}_H" in g:
            assert rel(H, g[f"{tag}_H"]) < REL_TOL
        else:
            assert rel(H[g[f"{tag}_H_rows"]], g[f"{tag}_H_sub"]) < REL_TOL
        assert np.allclose(np.linalg.norm(H, axis=1), g[f"{tag}_H_norm"], rtol=REL_TOL)


def test_fused_odd_offsets_and_strides(P):
    """Misaligned rows exercise the 8-byte TMA shift path: odd symbol0 offset,
    odd CP, odd row stride (rows padded by one sample)."""
    m, cp, n_ant, qam, d = 64, 7, 5, 16, 6
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    streams, _, s0 = make_batch(m, cp, n_ant, qam, d, (21, 22, 23))
    for extra in (0, 1, 3):
        pad = np.zeros(streams.shape[:2] + (extra,), dtype=streams.dtype)
        x = np.concatenate([pad, streams, pad[..., :1]], axis=2)
        out = P.receive_frames(torch.from_numpy(x.astype(np.complex64)).cuda(), cfg,
                               symbol0_offset=s0 + extra, n_data=d)
        for i, (H, s_hat, w, bits) in enumerate(oracle_frames(streams, s0, m, cp, d, qam)):
            assert np.array_equal(out.bits[i].cpu().numpy(), bits)
            assert rel(out.H[i].cpu().numpy(), H) < REL_TOL


def test_fused_pilot_only_and_many_chunks(P):
    m, cp, n_ant, qam = 256, 32, 4, 4
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    streams, _, s0 = make_batch(m, cp, n_ant, qam, 37, (31, 32))
    out = P.receive_frames(torch.from_numpy(streams.astype(np.complex64)).cuda(), cfg,
                           symbol0_offset=s0, n_data=37)
    for i, (H, s_hat, w, bits) in enumerate(oracle_frames(streams, s0, m, cp, 37, qam)):
        assert np.array_equal(out.bits[i].cpu().numpy(), bits)
        assert rel(out.s_hat[i].cpu().numpy(), s_hat) < REL_TOL
    out0 = P.receive_frames(torch.from_numpy(streams.astype(np.complex64)).cuda(), cfg,
                            symbol0_offset=s0, n_data=0)
    assert out0.bits.shape == (2, 0)
    H_ref = oracle_frames(streams, s0, m, cp, 0, qam)[0][0]
    assert rel(out0.H[0].cpu().numpy(), H_ref) < REL_TOL


def test_fused_zf_option(P):
    m, cp, n_ant, qam, d = 128, 16, 6, 16, 4
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    streams, _, s0 = make_batch(m, cp, n_ant, qam, d, (41,))
    out = P.receive_frames(torch.from_numpy(streams.astype(np.complex64)).cuda(), cfg,
                           symbol0_offset=s0, n_data=d, zf=True)
    H = oracle_frames(streams, s0, m, cp, d, qam)[0][0]
    zf = out.zf[0].cpu().numpy()
    for k in range(d):
        lo = s0 + (k + 1) * (m + cp)
        Y = orc.freq_transform(streams[0][:, lo + cp: lo + cp + m])
        assert rel(zf[k], orc.zf_per_antenna(Y, H)) < REL_TOL


def test_nonfinite_input_flagged(P):
    from paper_1901_07499_b200 import NumericInputError

    m, cp, n_ant, qam, d = 64, 16, 3, 4, 2
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    streams, _, s0 = make_batch(m, cp, n_ant, qam, d, (51, 52))
    streams[1, 2, s0 + (m + cp) + cp + 5] = np.nan
    out = P.receive_frames(torch.from_numpy(streams.astype(np.complex64)).cuda(), cfg,
                           symbol0_offset=s0, n_data=d)
    fl = out.flags.cpu().numpy()
    assert fl[0] == 0 and fl[1] & 1
    with pytest.raises(NumericInputError):
        P.receive_frames(torch.from_numpy(streams.astype(np.complex64)).cuda(), cfg,
                         symbol0_offset=s0, n_data=d, check=True)
    # a NaN inside the cyclic prefix is never read (cp_drop)
    streams[1, 2, s0 + (m + cp) + cp + 5] = 0
    streams[1, 2, s0 + (m + cp) + 3] = np.nan
    out = P.receive_frames(torch.from_numpy(streams.astype(np.complex64)).cuda(), cfg,
                           symbol0_offset=s0, n_data=d, check=True)


def test_erased_subcarrier_flag(P):
    """A pilot with zero energy on one subcarrier -> weight 0 -> erased, finite output
    (reference test_receiver.py:216-223)."""
    m, cp, n_ant, qam = 64, 16, 2, 4
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    pilot = orc.make_pilot(m)
    X = np.tile(pilot, (n_ant, 1))
    X[:, 3] = 0.0
    data = np.ones((n_ant, m), dtype=complex)
    rows = [orc.ofdm_modulate(X, cp), orc.ofdm_modulate(data, cp)]
    x = np.concatenate(rows, axis=1)[None]
    out = P.receive_frames(torch.from_numpy(x.astype(np.complex64)).cuda(), cfg, n_data=1)
    w = out.weights[0].cpu().numpy()
    assert out.erased[0, 3] and not out.erased[0, 2]
    assert w[3] < 1e-6
    assert np.all(np.isfinite(out.s_hat.cpu().numpy()))
    assert int(out.flags[0]) & 2


@pytest.mark.parametrize("m", [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096])
def test_staged_fft_vs_oracle(P, m):
    from paper_1901_07499_b200 import device

    rng = np.random.default_rng(m)
    x = rng.standard_normal((5, m)) + 1j * rng.standard_normal((5, m))
    y = device.fft_shift_rows(x).cpu().numpy()
    ref = orc.freq_transform(x)
    assert rel(y, ref) < 1e-5
    for r in range(5):  # reference test_receiver.py:102-108, relative form for fp32
        assert np.max(np.abs(y[r] - orc.fftshift(orc.dft_direct(x[r])))) < 1e-5 * np.max(np.abs(ref[r]))


def test_staged_fft_impulse_and_zero(P):
    from paper_1901_07499_b200 import device

    mat = np.zeros((3, 64), dtype=complex)
    assert np.array_equal(device.fft_shift_rows(mat).cpu().numpy(), mat)
    mat[:, 0] = 1.0
    assert np.allclose(device.fft_shift_rows(mat).cpu().numpy(), 1.0, atol=1e-6)


@pytest.mark.parametrize("tree", [False, True])
@pytest.mark.parametrize("n_ant", [1, 3, 16, 64, 97])
def test_staged_mrc_vs_oracle(P, n_ant, tree):
    from paper_1901_07499_b200 import device

    rng = np.random.default_rng(n_ant)
    y = rng.standard_normal((n_ant, 256)) + 1j * rng.standard_normal((n_ant, 256))
    h = rng.standard_normal((n_ant, 256)) + 1j * rng.standard_normal((n_ant, 256))
    s, w = device.mrc(y, h, tree=tree)
    s_ref, w_ref = (orc.mrc_tree if tree else orc.mrc_seq)(y, h)
    assert rel(s.cpu().numpy(), s_ref) < REL_TOL
    assert rel(w.cpu().numpy(), w_ref) < REL_TOL


def test_staged_ls_and_demap(P, golden_dir):
    from paper_1901_07499_b200 import device

    u = dict(np.load(os.path.join(golden_dir, "unit_vectors.npz")))
    for order in (4, 16, 64):
        assert np.array_equal(device.demap(u["demap_in"], order), u[f"demap_out_{order}"])
    pilot = orc.make_pilot(64)
    gains = np.array([2 - 1j, 0.3 + 0.4j, -1.5 + 0j])
    received = gains[:, None] * pilot[None, :]
    H = device.ls(received, pilot).cpu().numpy()
    assert np.allclose(H, np.tile(gains[:, None], (1, 64)), atol=1e-6)


def test_antenna_sharded_partials_match_full(P):
    """C4-style antenna sharding on one device: split 32 antennas into G=4
    shards, partial sums per shard, tree-combine over shards, finish."""
    m, cp, n_ant, qam, d, G = 2048, 256, 32, 64, 4, 4
    cfg_full = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    streams, _, s0 = make_batch(m, cp, n_ant, qam, d, (61,))
    x = torch.from_numpy(streams.astype(np.complex64)).cuda()
    full = P.receive_frames(x, cfg_full, symbol0_offset=s0, n_data=d)
    cfg_sh = P.OfdmConfig(m, cp, n_ant // G, qam_order=qam)
    nums, dens = [], []
    for g in range(G):
        xs = x[:, g * (n_ant // G):(g + 1) * (n_ant // G)].contiguous()
        _, num, den, _ = P.receive_partials(xs, cfg_sh, symbol0_offset=s0, n_data=d)
        nums.append(num)
        dens.append(den)
    s_hat, w, bits, flags = P.finish_partials(torch.stack(nums), torch.stack(dens), qam)
    H, s_ref, w_ref, b_ref = oracle_frames(streams, s0, m, cp, d, qam)[0]
    assert np.array_equal(bits[0].cpu().numpy(), b_ref)
    assert np.array_equal(bits.cpu().numpy(), full.bits.cpu().numpy())
    assert rel(s_hat[0].cpu().numpy(), s_ref) < REL_TOL
    assert rel(w[0].cpu().numpy(), w_ref) < REL_TOL


def test_large_batch_properties(P):
    """C3 at a throughput-sized batch: 8 distinct frames tiled to F=256.
    Size-independent properties: tiled frames give identical outputs, bits
    equal the oracle on the distinct frames, BER vs the transmitted payload is
    small at 10 dB with 64-antenna array gain."""
    m, cp, n_ant, qam, d = 1024, 72, 64, 16, 10
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    streams, tx_bits, s0 = make_batch(m, cp, n_ant, qam, d, range(8))
    base = torch.from_numpy(streams.astype(np.complex64)).cuda()
    x = base.repeat(32, 1, 1)
    out = P.receive_frames(x, cfg, symbol0_offset=s0, n_data=d, check=True)
    bits = out.bits.cpu().numpy()
    for i, ref in enumerate(oracle_frames(streams[:2], s0, m, cp, d, qam)):
        assert np.array_equal(bits[i], ref[3])
    assert np.array_equal(bits.reshape(32, 8, -1), np.broadcast_to(bits[:8], (32,) + bits[:8].shape))
    ber = np.mean(bits[:8] != np.stack(tx_bits))
    assert ber < 1e-3


@pytest.mark.parametrize("mode", ["gather", "allreduce", "scatter"])
def test_antenna_sharded_receiver_world1(P, mode):
    """AntennaShardedReceiver through torch.distributed (NCCL, world size 1)."""
    import socket

    import torch.distributed as dist

    from paper_1901_07499_b200 import sharding

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        m, cp, n_ant, qam, d = 512, 64, 16, 64, 5
        cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
        streams, _, s0 = make_batch(m, cp, n_ant, qam, d, (71, 72))
        x = torch.from_numpy(streams.astype(np.complex64)).cuda()
        rx = sharding.AntennaShardedReceiver(cfg, d, symbol0_offset=s0, mode=mode)
        s_hat, w, bits, fl, _ = rx.receive(x)
        for i, (H, s_ref, w_ref, b_ref) in enumerate(oracle_frames(streams, s0, m, cp, d, qam)):
            assert np.array_equal(bits[i].cpu().numpy(), b_ref)
            assert rel(s_hat[i].cpu().numpy(), s_ref) < REL_TOL
        assert int(fl.abs().sum()) == 0
    finally:
        dist.destroy_process_group()


def test_streaming_receiver_matches_batch(P):
    from paper_1901_07499_b200 import frames

    m, cp, n_ant, qam, d = 256, 32, 16, 16, 10
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    streams, _, s0 = make_batch(m, cp, n_ant, qam, d, range(5))
    host = torch.from_numpy(streams.astype(np.complex64)).pin_memory()
    bits = torch.empty((5, d * m * 4), dtype=torch.uint8).pin_memory()
    s_hat = torch.empty((5, d, m), dtype=torch.complex64).pin_memory()
    rx = frames.StreamingReceiver(cfg, 2, d, symbol0_offset=s0, samples_per_row=streams.shape[2])
    rx.run(host, bits, s_hat)
    for i, (H, s_ref, w_ref, b_ref) in enumerate(oracle_frames(streams, s0, m, cp, d, qam)):
        assert np.array_equal(bits[i].numpy(), b_ref)
        assert rel(s_hat[i].numpy(), s_ref) < REL_TOL


@pytest.mark.parametrize("layout", ["uniform", "frame_gap", "one_antenna", "one_frame"])
def test_stage_symbols_drops_cp_and_matches_full_receive(P, layout):
    """ofdmrx_stage_symbols copies exactly the FFT windows (CP dropped) for
    every frame/antenna/symbol; receive_staged on the dense copy equals
    receive_frames on the capture (same kernel, same bits/values)."""
    from paper_1901_07499_b200 import frames

    m, cp, qam, d = 128, 16, 16, 5
    n_ant = 1 if layout == "one_antenna" else 6
    nf = 1 if layout == "one_frame" else 4
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    streams, _, s0 = make_batch(m, cp, n_ant, qam, d, range(nf))
    s0 += 3  # odd offset inside the capture
    pad = np.zeros(streams.shape[:2] + (3,), dtype=streams.dtype)
    streams = np.concatenate([pad, streams], axis=2)
    host = torch.from_numpy(streams.astype(np.complex64))
    if layout == "frame_gap":  # frames that are not N*row_stride apart
        big = torch.zeros((nf, n_ant + 1, streams.shape[2]), dtype=torch.complex64)
        big[:, :n_ant] = host
        host = big[:, :n_ant]
    src = host.contiguous().pin_memory() if layout != "frame_gap" else host
    if layout == "frame_gap":
        # a non-contiguous view cannot go through the tensor wrapper; call the
        # C ABI with the parent's strides directly
        import ctypes

        from paper_1901_07499_b200 import _lib, device

        base = big.pin_memory()
        dst = torch.empty((nf, n_ant, 1 + d, m), dtype=torch.complex64, device="cuda")
        desc = device.make_desc(nf, n_ant, m, cp, d, qam, s0, streams.shape[2], (n_ant + 1) * streams.shape[2],
                                rx_samples=base.numel())
        _lib.call("ofdmrx_stage_symbols", ctypes.byref(desc), device.ctypes_void(base.data_ptr()), device.ptr(dst),
                  device.stream_handle())
    else:
        dst = frames.stage_symbols(src, cfg, symbol0_offset=s0, n_data=d)
    torch.cuda.synchronize()
    ref = host.numpy()
    for f in range(nf):
        for n in range(n_ant):
            for s in range(1 + d):
                a = s0 + s * (m + cp) + cp
                assert np.array_equal(dst[f, n, s].cpu().numpy(), ref[f, n, a:a + m])
    got = frames.receive_staged(dst, cfg)
    full = frames.receive_frames(torch.from_numpy(ref.copy()).cuda(), cfg, symbol0_offset=s0, n_data=d)
    torch.cuda.synchronize()
    assert torch.equal(got.bits, full.bits)
    assert torch.equal(got.s_hat, full.s_hat)
    assert torch.equal(got.H, full.H)


@pytest.mark.parametrize("n_ant,m,cp,qam,d,nf", [(8, 64, 16, 16, 6, 3), (64, 1024, 72, 16, 10, 2), (16, 256, 32, 64, 4, 2)])
def test_fused_complex_unit_pilot(P, n_ant, m, cp, qam, d, nf):
    """Any unit-modulus pilot (not only make_pilot's BPSK): the fused kernel's
    general H = Y conj(P) path (ls_divide, receiver.py:95-96), including the
    on-device antenna-shard path at 64 antennas x 2 frames."""
    rng = np.random.default_rng(m + n_ant)
    pilot = np.exp(2j * np.pi * rng.random(m))
    caps = []
    for f in range(nf):
        bits = np.random.default_rng(100 + f).integers(0, 2, size=d * m * int(math.log2(qam)), dtype=np.uint8)
        tx, _, _ = orc.build_frame_samples(m, cp, qam, pilot, bits, orc.generate_pn())
        st, _ = orc.apply_channel(tx, n_ant, mode="flat_rayleigh", snr_db=12.0, rng_seed=f)
        caps.append(st)
    streams = np.stack(caps)
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    out = P.receive_frames(torch.from_numpy(streams.astype(np.complex64)).cuda(), cfg, pilot,
                           symbol0_offset=255, n_data=d)
    torch.cuda.synchronize()
    for f in range(nf):
        H, s_hat, w, bits = orc.receive_frame(streams[f], 255, m, cp, d, qam, pilot=pilot)
        assert np.array_equal(out.bits[f].cpu().numpy(), bits)
        assert rel(out.H[f].cpu().numpy(), H) < REL_TOL
        assert rel(out.s_hat[f].cpu().numpy(), s_hat) < REL_TOL
        assert rel(out.weights[f].cpu().numpy(), w) < REL_TOL


BALANCED_CASES = [
    # (M, N, D, frames, BPSK pilot)
    (1024, 64, 10, 3, True), (1024, 8, 12, 2, True), (1024, 5, 3, 2, True), (1024, 100, 1, 2, True),
    (1024, 13, 7, 2, False), (1024, 1, 12, 2, True), (1024, 64, 10, 2, False),
    # D*N < workers: empty lanes sit between a symbol's owner and the lanes
    # continuing it (the owner must skip them, not stop)
    (1024, 2, 1, 2, True), (1024, 4, 2, 2, True), (1024, 10, 1, 2, True), (1024, 2, 5, 2, True),
    (1024, 3, 2, 1, True), (1024, 6, 1, 1, True), (1024, 7, 1, 1, True),
    # more data symbols than one CTA's lanes: the frame's workers span a cluster
    (1024, 16, 20, 2, True), (1024, 3, 40, 1, True),
    # M = 2048 (lanes of 64 threads) and M = 4096 (128 threads)
    (2048, 32, 10, 2, True), (2048, 3, 4, 2, True), (2048, 7, 1, 1, False), (2048, 256, 2, 1, True),
    (4096, 5, 3, 2, True), (4096, 1, 2, 1, True), (4096, 9, 6, 1, False),
]


@pytest.mark.parametrize("m,n_ant,d,nf,bpsk", BALANCED_CASES, ids=lambda c: str(c))
def test_balanced_kernel(P, m, n_ant, d, nf, bpsk):
    """The balanced kernel (rx_balanced.cu: pilot rows first, data rows split
    evenly over the frame's workers, H through L2, symbols spanning workers
    combined in the epilogue, over DSMEM when the workers span a cluster) at
    every batch mapping: frames received together and one at a time."""
    from paper_1901_07499_b200 import device

    cp = m // 8
    qam = 16
    pilot = orc.make_pilot(m) if bpsk else np.exp(2j * np.pi * np.random.default_rng(n_ant).random(m))
    caps = []
    for f in range(nf):
        bits = np.random.default_rng(200 + f).integers(0, 2, size=d * m * 4, dtype=np.uint8)
        tx, _, _ = orc.build_frame_samples(m, cp, qam, pilot, bits, orc.generate_pn())
        st, _ = orc.apply_channel(tx, n_ant, mode="flat_rayleigh", snr_db=15.0, rng_seed=f + 7)
        caps.append(st)
    streams = np.stack(caps)
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    x = torch.from_numpy(streams.astype(np.complex64)).cuda()
    desc = device.make_desc(nf, n_ant, m, cp, d, qam, 255, x.shape[2], n_ant * x.shape[2], rx_samples=x.numel())
    assert device.rx_plan(desc)["kernel"] == 1  # OFDMRX_KERNEL_BALANCED
    for want_h in (True, False):
        outs = [P.receive_frames(x, cfg, pilot, symbol0_offset=255, n_data=d, want_h=want_h)]
        outs += [P.receive_frames(x[f:f + 1], cfg, pilot, symbol0_offset=255, n_data=d, want_h=want_h)
                 for f in range(nf)]
        torch.cuda.synchronize()
        out = outs[0]
        assert int(out.flags.abs().sum()) == 0
        for f in range(nf):
            H, s_hat, w, bits = orc.receive_frame(streams[f], 255, m, cp, d, qam, pilot=pilot)
            assert np.array_equal(out.bits[f].cpu().numpy(), bits)
            assert rel(out.s_hat[f].cpu().numpy(), s_hat) < REL_TOL
            assert rel(out.weights[f].cpu().numpy(), w) < REL_TOL
            if want_h:
                assert rel(out.H[f].cpu().numpy(), H) < REL_TOL
            single = outs[1 + f]
            assert torch.equal(single.bits[0], out.bits[f]) and torch.equal(single.s_hat[0], out.s_hat[f])
