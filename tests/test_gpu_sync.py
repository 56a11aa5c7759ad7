"""PN packet detection on the device (sync.detect_packet / kernels.corr_metrics,
SURVEY.md §8(f) #1) against the oracle and the reference's golden vectors.

Bar: peak indices exact; peak metrics within 1e-6 of the reference (the
device reads cf32 samples, the reference complex128: the quantisation of the
input bounds the agreement; the fp32 metric error itself is removed by the
fp64 re-scoring of near-maximal windows).  Full fp32 metric arrays within
2e-5 absolute (3 P 2^-24 bound for P = 255).
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import ofdm_oracle as orc  # noqa: E402

PEAK_TOL = 1e-6
METRIC_TOL = 2e-5


@pytest.fixture(scope="module")
def S():
    from paper_1901_07499_b200 import device, sync

    device.require_cuda()
    return sync


@pytest.fixture(scope="module")
def gold(golden_dir):
    return dict(np.load(os.path.join(golden_dir, "sync_vectors.npz")))


def test_corr_metrics_vs_reference_golden(S, gold):
    got = S.corr_metrics(gold["corr_stream"], gold["corr_chips"])
    assert got.shape == gold["corr_out"].shape == (4000 - 255 + 1,)
    assert np.max(np.abs(got - gold["corr_out"])) < METRIC_TOL
    emb = S.corr_metrics(gold["emb_stream"], gold["emb_chips"])
    assert np.max(np.abs(emb - gold["emb_out"])) < METRIC_TOL
    assert int(np.argmax(emb)) == 300 and emb[300] > 0.99 and np.all(emb <= 1.0 + 1e-6)


@pytest.mark.parametrize("case", orc.SYNC_CASES, ids=lambda c: c[0])
def test_detect_packet_vs_reference_golden(S, gold, case):
    name = case[0]
    streams = orc.sync_capture(*case[1:])
    det = S.detect_packet(streams, orc.generate_pn())
    idx = [p[0] for p in det.per_antenna_peaks]
    met = np.array([p[1] for p in det.per_antenna_peaks])
    assert np.array_equal(idx, gold[f"{name}_peaks"])
    assert np.max(np.abs(met - gold[f"{name}_metrics"])) < PEAK_TOL
    assert det.detected == bool(gold[f"{name}_detected"])
    assert det.frame_start == idx[0] and det.symbol0_offset == idx[0] + 255


def test_noise_only_rows_vs_reference_golden(S, gold):
    pn = orc.generate_pn()
    for i, row in enumerate(gold["noise_streams"]):
        det = S.detect_packet(row[None, :], pn)
        assert det.frame_start == gold["noise_peaks"][i]
        assert abs(det.peak_metric - gold["noise_metrics"][i]) < PEAK_TOL
        assert not det.detected


def test_clean_detection_exact_offset_and_unit_peak(S):
    # tests/test_sync.py:17-27
    streams = orc.sync_capture(1, "identity", None, 1000, 0)
    det = S.detect_packet(streams, orc.generate_pn())
    assert det.detected and det.frame_start == 1000 and det.symbol0_offset == 1255
    assert abs(det.peak_metric - 1.0) < PEAK_TOL and len(det.per_antenna_peaks) == 1


def test_zero_db_detection_stays_exact(S):
    # tests/test_sync.py:40-52, batched: 50 trials in one call per offset set
    pn = orc.generate_pn()
    hits = 0
    for trial in range(50):
        off = int(np.random.default_rng(1000 + trial).integers(0, 300))
        det = S.detect_packet(orc.sync_capture(1, "flat_rayleigh", 0.0, off, trial), pn)
        hits += int(det.frame_start == off)
    assert hits >= 49


def test_shift_and_scale_invariance(S):
    # tests/test_sync.py:55-80
    pn = orc.generate_pn()
    base = S.detect_packet(orc.sync_capture(1, "identity", None, 0, 0), pn)
    for shift in (1, 17, 999, 1999):
        assert S.detect_packet(orc.sync_capture(1, "identity", None, shift, 0), pn).frame_start == \
            base.frame_start + shift
    cap = orc.sync_capture(1, "identity", None, 123, 0)
    b2 = S.detect_packet(cap, pn)
    rng = np.random.default_rng(6)
    for _ in range(5):
        scale = complex(rng.standard_normal(), rng.standard_normal())
        det = S.detect_packet(scale * cap, pn)
        assert det.frame_start == b2.frame_start and abs(det.peak_metric - b2.peak_metric) < PEAK_TOL


def test_short_stream_and_bad_chips_rejected(S):
    from paper_1901_07499_b200.errors import ContractError, InputError

    with pytest.raises(InputError):
        S.detect_packet(np.zeros((1, 100), dtype=complex), orc.generate_pn())
    with pytest.raises(ContractError):
        S.detect_packet(np.zeros((1, 400), dtype=complex), np.array([1j, 1.0]))


def test_degenerate_rows(S):
    pn = orc.generate_pn()
    # all-zero stream: every metric is 0, argmax is window 0 (np.argmax)
    det = S.detect_packet(np.zeros((2, 600), dtype=complex), pn)
    assert det.per_antenna_peaks == ((0, 0.0), (0, 0.0)) and not det.detected
    # exactly one window; one-chip PN
    rng = np.random.default_rng(3)
    x = rng.standard_normal((3, 255)) + 1j * rng.standard_normal((3, 255))
    det = S.detect_packet(x, pn)
    for a in range(3):
        ref = orc.corr_metrics(x[a], pn)
        assert det.per_antenna_peaks[a][0] == 0 and abs(det.per_antenna_peaks[a][1] - ref[0]) < PEAK_TOL
    y = rng.standard_normal(50) + 1j * rng.standard_normal(50)
    got = S.corr_metrics(y, np.array([1.0]))
    assert np.max(np.abs(got - orc.corr_metrics(y, np.array([1.0])))) < METRIC_TOL


@pytest.mark.parametrize("n_chips", [7, 15, 31, 255, 1023])
def test_chip_lengths_and_tile_edges(S, n_chips):
    # P % K tails, window counts straddling the 1920-window tile
    rng = np.random.default_rng(n_chips)
    chips = np.where(rng.integers(0, 2, n_chips) == 1, 1.0, -1.0)
    for s in (n_chips, n_chips + 1919, n_chips + 1920, n_chips + 4000):
        x = 0.3 * (rng.standard_normal((2, s)) + 1j * rng.standard_normal((2, s)))
        off = int(rng.integers(0, s - n_chips + 1))
        x[1, off:off + n_chips] += chips
        got = S.corr_metrics(x, chips)
        for a in range(2):
            ref = orc.corr_metrics(x[a], chips)
            assert np.max(np.abs(got[a] - ref)) < 3 * n_chips * 6e-8 + 1e-6
        det = S.detect_packet(x, chips)
        for a in range(2):
            ref = orc.corr_metrics(x[a], chips)
            i = det.per_antenna_peaks[a][0]
            assert i == int(np.argmax(ref)) or ref[i] >= ref.max() - PEAK_TOL
        assert det.per_antenna_peaks[1][0] == off


def test_batched_frames_feed_receive(S):
    """detect_frames over a batch of C2-sized captures with distinct timing
    offsets; symbol0_offset per frame equals the oracle's and the receive
    path decodes the payload from it."""
    from paper_1901_07499_b200 import frames
    import paper_1901_07499_b200 as P

    m, cp, n_ant, qam, d = 256, 32, 16, 16, 4
    pn = orc.generate_pn()
    offs = [0, 5, 131, 300]
    caps = []
    for i, off in enumerate(offs):
        bits = np.random.default_rng(i).integers(0, 2, size=d * m * 4, dtype=np.uint8)
        samples, _, _ = orc.build_frame_samples(m, cp, qam, orc.make_pilot(m), bits, pn)
        st, _ = orc.apply_channel(samples, n_ant, mode="flat_rayleigh", snr_db=10.0, timing_offset=off, rng_seed=i)
        full = np.zeros((n_ant, len(samples) + 300), dtype=np.complex128)
        full[:, :st.shape[1]] = st
        caps.append((full, bits))
    batch = np.stack([c[0] for c in caps])
    det = S.detect_frames(torch.from_numpy(batch.astype(np.complex64)).cuda(), pn)
    torch.cuda.synchronize()
    for i, (st, bits) in enumerate(caps):
        ok, start, s0, peak, peaks = orc.detect_packet(st, pn)
        assert [p[0] for p in peaks] == det.peak_index[i].cpu().tolist()
        assert np.max(np.abs(np.array([p[1] for p in peaks]) - det.peak_metric[i].cpu().numpy())) < PEAK_TOL
        assert start == offs[i] and bool(det.detected[i])
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    for i, (st, bits) in enumerate(caps):
        out = frames.receive_frames(torch.from_numpy(st.astype(np.complex64)).cuda(), cfg,
                                    symbol0_offset=int(det.symbol0_offset[i]), n_data=d)
        ref = orc.receive_frame(st, offs[i] + 255, m, cp, d, qam)[3]
        assert np.array_equal(out.bits[0].cpu().numpy(), ref)


@pytest.mark.parametrize("m,cp,n_ant,qam,d,shards,ants", [(1024, 72, 16, 16, 4, False, "first"),
                                                          (1024, 72, 16, 16, 4, True, "all"),
                                                          (256, 32, 8, 16, 6, True, "first"),
                                                          (64, 16, 4, 4, 10, False, "all")])
def test_receive_captures_device_timing(S, m, cp, n_ant, qam, d, shards, ants):
    """Raw captures with different timing offsets -> detect_frames ->
    ofdmrx_rx_frames_detected (per-frame symbol0 on the device): every
    detected frame decodes as the oracle at its true offset; a noise-only
    capture is flagged NOT_DETECTED and a truncated one OUT_OF_RANGE."""
    import paper_1901_07499_b200 as P
    from paper_1901_07499_b200 import _lib, frames

    pn = orc.generate_pn()
    offs = [0, 37, 250, 501]
    frame_len = 255 + (1 + d) * (m + cp)
    s_len = frame_len + 520
    rng = np.random.default_rng(m + d)
    caps = []
    for i, off in enumerate(offs):
        bits = rng.integers(0, 2, size=d * m * int(np.log2(qam)), dtype=np.uint8)
        samples, _, _ = orc.build_frame_samples(m, cp, qam, orc.make_pilot(m), bits, pn)
        st, _ = orc.apply_channel(samples, n_ant, mode="flat_rayleigh", snr_db=12.0, timing_offset=off, rng_seed=i)
        full = np.zeros((n_ant, s_len), dtype=np.complex128)
        full[:, :st.shape[1]] = st
        caps.append(full)
    caps.append(0.5 * (rng.standard_normal((n_ant, s_len)) + 1j * rng.standard_normal((n_ant, s_len))))  # noise only
    late = np.zeros((n_ant, s_len), dtype=np.complex128)  # packet starting too late to fit
    late[:, s_len - 400:] = caps[0][:, :400]
    caps.append(late)
    batch = np.stack(caps)
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    out, det = frames.receive_captures(torch.from_numpy(batch.astype(np.complex64)).cuda(), cfg, d, shards=shards,
                                       antennas=ants)
    assert det.peak_index.shape[1] == (n_ant if ants == "all" else 1)
    torch.cuda.synchronize()
    fl = out.flags.cpu().numpy()
    for i, off in enumerate(offs):
        assert int(det.frame_start[i]) == off and fl[i] == 0
        H, s_hat, w, bits = orc.receive_frame(caps[i].astype(np.complex64).astype(np.complex128), off + 255, m, cp, d,
                                              qam)
        assert np.array_equal(out.bits[i].cpu().numpy(), bits)
        assert np.linalg.norm(out.s_hat[i].cpu().numpy() - s_hat) / np.linalg.norm(s_hat) < 1e-4
    assert fl[len(offs)] & _lib.FLAG_NOT_DETECTED
    assert fl[len(offs) + 1] & _lib.FLAG_OUT_OF_RANGE


def test_files_to_bits(S, tmp_path):
    """Capture directories in the reference layout (rx_meta.txt +
    rx_ant<k>.cf32, cli._load_capture) -> ingest.load_captures (pinned) ->
    receive_captures on the device -> bits equal the oracle's."""
    import paper_1901_07499_b200 as P
    from paper_1901_07499_b200 import frames, ingest

    m, cp, n_ant, qam, d = 256, 32, 8, 16, 5
    cfg = P.OfdmConfig(m, cp, n_ant, qam_order=qam)
    pn = orc.generate_pn()
    dirs, truth = [], []
    for i, off in enumerate((0, 77, 300)):
        bits = np.random.default_rng(40 + i).integers(0, 2, size=d * m * 4, dtype=np.uint8)
        samples, _, _ = orc.build_frame_samples(m, cp, qam, orc.make_pilot(m), bits, pn)
        st, _ = orc.apply_channel(samples, n_ant, mode="flat_rayleigh", snr_db=12.0, timing_offset=off, rng_seed=i)
        ingest.write_capture(str(tmp_path / f"cap{i}"), st, cfg)
        dirs.append(str(tmp_path / f"cap{i}"))
        truth.append((st.astype(np.complex64).astype(np.complex128), off))
    metas, cfg2, host = ingest.load_captures(dirs, pinned=True)
    assert host.is_pinned() and cfg2 == cfg
    out, det = frames.receive_captures(host.cuda(non_blocking=True), cfg2, d)
    torch.cuda.synchronize()
    for i, (st, off) in enumerate(truth):
        assert int(det.frame_start[i]) == off and int(out.flags[i]) == 0
        H, s_hat, w, bits = orc.receive_frame(st, off + 255, m, cp, d, qam)
        assert np.array_equal(out.bits[i].cpu().numpy(), bits)
