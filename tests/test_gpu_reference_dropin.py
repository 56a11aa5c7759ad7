"""The drop-in claim against the UNMODIFIED reference package.

The reference (baseline/_ref, installed from /root/reference/pkg by
`pip install --target baseline/_ref`, never edited) runs its own
run_ring_pipeline / process_symbol (receiver.py:238-267, 308-348) with the
B200 engine plugged in exactly as INTEGRATION.md §1 shows: a `make_engine`
branch for variant "b200".  Bits must equal the reference's own
SequentialEngine / DataParallelEngine results; H and s_hat agree within
1e-4 (fp32 device path vs the fp64 reference, the north_star bar)."""

import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SITE = os.path.join(ROOT, "baseline", "_ref")
REL_TOL = 1e-4


def rel(a, b):
    a = np.asarray(a, np.complex128)
    b = np.asarray(b, np.complex128)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF_SITE, "ofdmrx")):
        pytest.skip("reference not installed in baseline/_ref (bench.py --impl reference installs it)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    if REF_SITE not in sys.path:
        sys.path.insert(0, REF_SITE)
    import ofdmrx.receiver as rr
    from ofdmrx import channel, sync, waveform

    assert os.path.dirname(rr.__file__).startswith(REF_SITE), rr.__file__  # the installed reference
    return rr, channel, sync, waveform


@pytest.fixture
def ref_with_b200(ref, monkeypatch):
    """the two lines a maintainer adds to the reference."""
    rr = ref[0]
    from paper_1901_07499_b200.receiver import B200Engine

    orig = rr.make_engine

    def make_engine(kind):
        if kind.variant == "b200":
            return B200Engine(variant="b200", worker_count=kind.worker_count)
        return orig(kind)

    monkeypatch.setattr(rr, "ENGINE_VARIANTS", ("sequential", "data_parallel", "b200"))
    monkeypatch.setattr(rr, "make_engine", make_engine)
    return ref


def frame_slots(ref, fft_len, cp_len, n_ant, qam, n_data, seed, snr_db=10.0):
    rr, channel, sync, wf = ref
    cfg = wf.OfdmConfig(fft_len, cp_len, n_ant, qam_order=qam)
    pilot = wf.make_pilot(fft_len)
    pn = wf.generate_pn()
    bits = np.random.default_rng(seed).integers(0, 2, size=n_data * fft_len * cfg.bits_per_qam_symbol,
                                                dtype=np.uint8)
    frame = wf.build_frame(cfg, pilot, bits, pn)
    cap = channel.apply_channel(frame, channel.ChannelModel("flat_rayleigh", snr_db=snr_db, timing_offset=37,
                                                            rng_seed=seed), cfg)
    det = sync.detect_packet(cap, pn)  # the reference's own detection
    assert det.detected
    return cfg, pilot, rr.extract_slots(cap, det, cfg, 1 + n_data)


@pytest.mark.parametrize("shape", [(64, 16, 8, 4, 10), (1024, 72, 64, 16, 10), (256, 32, 16, 64, 6)],
                         ids=["C1", "C3", "N16xM256q64"])
def test_reference_pipeline_with_b200_engine(ref_with_b200, shape):
    rr = ref_with_b200[0]
    cfg, pilot, slots = frame_slots(ref_with_b200, *shape, seed=shape[0] + 5)
    with rr.make_engine(rr.EngineKind("sequential")) as eng:
        want = rr.run_ring_pipeline(slots, cfg, eng, pilot=pilot)
    with rr.make_engine(rr.EngineKind("b200")) as eng:  # INTEGRATION.md §1 branch
        got = rr.run_ring_pipeline(slots, cfg, eng, pilot=pilot)
    assert np.array_equal(got.bits, want.bits)
    assert rel(got.estimate.gains, want.estimate.gains) < REL_TOL
    for a, b in zip(got.symbols, want.symbols):
        assert a.seq_no == b.seq_no
        assert rel(a.equalized, b.equalized) < REL_TOL
        assert rel(a.weight_norm, b.weight_norm) < REL_TOL
        assert np.array_equal(a.erased, b.erased)
    # the reference measured every stage around our engine calls
    assert len(got.timings) == len(slots) and all(t.fft_s > 0 and t.combine_s > 0 for t in got.timings)


def test_reference_process_symbol_with_b200_engine(ref_with_b200):
    rr = ref_with_b200[0]
    from paper_1901_07499_b200.receiver import B200Engine

    cfg, pilot, slots = frame_slots(ref_with_b200, 1024, 72, 32, 16, 3, seed=11)
    eng_ref = rr.SequentialEngine()
    eng = B200Engine()
    est_ref, _ = rr.process_symbol(slots[0], None, cfg, eng_ref, pilot=pilot)
    est, t = rr.process_symbol(slots[0], None, cfg, eng, pilot=pilot)
    assert t.kind == "pilot" and t.combine_stage == "ls"
    assert rel(est.gains, est_ref.gains) < REL_TOL
    for slot in slots[1:]:
        a, _ = rr.process_symbol(slot, est, cfg, eng, pilot=pilot)
        b, _ = rr.process_symbol(slot, est_ref, cfg, eng_ref, pilot=pilot)
        assert np.array_equal(a.bits, b.bits)
        assert rel(a.equalized, b.equalized) < REL_TOL
    with pytest.raises(rr.PipelineOrderError):
        rr.process_symbol(slots[1], None, cfg, eng, pilot=pilot)


def test_mirror_engines_match_reference_engines(ref):
    """The mirror's SequentialEngine / DataParallelEngine drive the reference
    pipeline and match the reference engines of the same name (the data-
    parallel one in the reference pairwise-tree antenna order)."""
    rr = ref[0]
    from paper_1901_07499_b200 import receiver as mr

    cfg, pilot, slots = frame_slots(ref, 256, 32, 16, 16, 8, seed=21)
    for mine, theirs in ((mr.SequentialEngine(), rr.SequentialEngine()),
                         (mr.DataParallelEngine(4), rr.DataParallelEngine(4))):
        assert mine.variant == theirs.variant and mine.worker_count == theirs.worker_count
        got = rr.run_ring_pipeline(slots, cfg, mine, pilot=pilot)
        want = rr.run_ring_pipeline(slots, cfg, theirs, pilot=pilot)
        theirs.close()
        assert np.array_equal(got.bits, want.bits)
        for a, b in zip(got.symbols, want.symbols):
            assert rel(a.equalized, b.equalized) < REL_TOL
    # and the mirror's own run_ring_pipeline (fused segment launch) on the reference slots
    got = mr.run_ring_pipeline(slots, cfg, mr.make_engine(mr.EngineKind("sequential")), pilot=pilot)
    want = rr.run_ring_pipeline(slots, cfg, rr.SequentialEngine(), pilot=pilot)
    assert np.array_equal(got.bits, want.bits)
    assert rel(got.estimate.gains, want.estimate.gains) < REL_TOL
