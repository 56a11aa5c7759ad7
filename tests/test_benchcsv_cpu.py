"""B200 sweep records in the reference bench CSV schema:
the reference's own tooling (ofdmrx.bench.read_bench_csv / speedup_table,
bench.py:217-249,282-299) reads what bench.py --sweep writes, and the
B200 engine's StageTimings map onto the reference STAGES."""

import os
import sys

import numpy as np
import pytest

from paper_1901_07499_b200 import benchcsv
from paper_1901_07499_b200.receiver import StageTimings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SITE = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ref_bench():
    if not os.path.isdir(os.path.join(REF_SITE, "ofdmrx")):
        pytest.skip("reference not installed in baseline/_ref")
    if REF_SITE not in sys.path:
        sys.path.insert(0, REF_SITE)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    from ofdmrx import bench

    return bench


class _Cfg:
    def __init__(self, m, cp, n):
        self.fft_len, self.cp_len, self.n_antennas = m, cp, n


def _timings(scale, n_data=10):
    out = [StageTimings("pilot", 1e-6 * scale, 2e-6 * scale, 3e-6 * scale, 4e-6 * scale)]
    out += [StageTimings("data", 1e-6 * scale, 2e-6 * scale, 5e-6 * scale, 6e-6 * scale) for _ in range(n_data)]
    return out


def _records():
    recs = []
    for m, cp, n in ((64, 16, 8), (1024, 72, 64)):
        cfg = _Cfg(m, cp, n)
        recs += benchcsv.records_for_engine(cfg, "sequential", 1, _timings(100.0), _timings(200.0))
        recs += benchcsv.records_for_engine(cfg, "b200", 1, _timings(1.0), _timings(2.0))
        recs.append(benchcsv.BenchRecord(m, cp, n, "b200_batched", 1, "demodulation", "fft", 0.2, 0.0, 640))
    return recs


def test_stage_names_are_the_reference_stages():
    recs = _records()
    assert {r.stage for r in recs} <= set(benchcsv.STAGES)
    assert {r.phase for r in recs} == set(benchcsv.PHASES)
    est = [r for r in recs if r.engine == "b200" and r.phase == "estimation" and r.stage == "ls"]
    assert len(est) == 2 and est[0].mean_us == pytest.approx(4.0) and est[0].n_symbols == 1


def test_speedup_table_local(tmp_path):
    path = tmp_path / "sweep.csv"
    benchcsv.write_bench_csv(_records(), path)
    back = benchcsv.read_bench_csv(path)
    assert back == _records()
    rows = benchcsv.speedup_table(back)
    assert all(r.speedup == pytest.approx(100.0) for r in rows)
    assert {r.stage for r in rows} == {"read", "cp_drop", "fft", "ls", "mrc", "total"}


def test_reference_tooling_reads_b200_csv(ref_bench, tmp_path):
    """The reference's read_bench_csv + speedup_table on the B200 CSV: the
    b200 engine in the data_parallel role, ratios sequential / b200."""
    path = tmp_path / "sweep.csv"
    benchcsv.write_bench_csv(_records(), path)
    recs = ref_bench.read_bench_csv(str(path))
    assert len(recs) == len(_records())
    rows = ref_bench.speedup_table(benchcsv.as_reference_pair(recs, parallel="b200"))
    assert rows and all(r.speedup == pytest.approx(100.0) for r in rows)
    # without the relabelling the reference tool rejects the cells (no data_parallel engine)
    from ofdmrx.errors import IncompleteDataError

    with pytest.raises(IncompleteDataError):
        ref_bench.speedup_table(recs)
    out = tmp_path / "speedup.csv"
    ref_bench.write_speedup_csv(rows, str(out))
    assert len(ref_bench.read_speedup_csv(str(out))) == len(rows)


def test_committed_sweep_loads_in_reference_tooling(ref_bench):
    """profiles/sweep_r02.csv (bench.py --sweep on a B200) through the
    reference tooling: every cell has its sequential / b200 pair."""
    path = os.path.join(ROOT, "profiles", "sweep_r02.csv")
    if not os.path.exists(path):
        pytest.skip("no round-2 sweep committed yet")
    recs = ref_bench.read_bench_csv(path)
    rows = ref_bench.speedup_table(benchcsv.as_reference_pair(recs, parallel="b200"))
    cells = {(r.fft_len, r.n_antennas) for r in recs}
    assert {(r.fft_len, r.n_antennas) for r in rows} == cells
    assert all(np.isfinite(r.speedup) and r.speedup > 0 for r in rows)
