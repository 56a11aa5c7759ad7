"""B200 records in the reference bench CSV schema (ofdmrx/bench.py:19-25,
63-130, 217-249, 266-341), so the reference's own tooling reads them.

* ``records_for_engine`` restates ``_records_for_engine`` / ``_stage_samples``
  (bench.py:87-150): per (phase, stage) mean/std of the StageTimings of a
  ``run_ring_pipeline`` run, plus the per-phase ``warmup`` record.  Stage
  names are the reference's STAGES (read, cp_drop, fft, ls, mrc, warmup);
  the B200 engine's timings come from the mirror's run_ring_pipeline, whose
  StageTimings keep the reference's meaning (receiver._run_fused).
* ``as_reference_pair`` relabels one engine as the reference's parallel
  engine ("data_parallel"), so ``ofdmrx.bench.speedup_table`` computes
  sequential / B200 ratios unchanged (its IncompleteDataError still fires
  for a cell without both engines).
* ``speedup_table`` is the same computation without importing the reference
  (sequential / ``parallel`` per stage plus the per-phase total).
"""

import csv
from dataclasses import dataclass, replace

import numpy as np

PHASES = ("estimation", "demodulation")                       # bench.py:19
STAGES = ("read", "cp_drop", "fft", "ls", "mrc", "warmup")    # bench.py:20
CSV_HEADER = "fft_len,cp_len,n_antennas,engine,workers,phase,stage,mean_us,std_us,n_symbols"  # bench.py:22-24


@dataclass(frozen=True)
class BenchRecord:
    """bench.py:51-61."""

    fft_len: int
    cp_len: int
    n_antennas: int
    engine: str
    workers: int
    phase: str
    stage: str
    mean_us: float
    std_us: float
    n_symbols: int


@dataclass(frozen=True)
class SpeedupRow:
    """bench.py:70-76."""

    fft_len: int
    n_antennas: int
    phase: str
    stage: str
    speedup: float


def _stage_samples(timings):
    """bench.py:79-97."""
    out = {(ph, st): [] for ph, sts in (("estimation", ("read", "cp_drop", "fft", "ls")),
                                          ("demodulation", ("read", "cp_drop", "fft", "mrc"))) for st in sts}
    for t in timings:
        phase = "estimation" if t.kind == "pilot" else "demodulation"
        out[(phase, "read")].append(t.read_s)
        out[(phase, "cp_drop")].append(t.cp_drop_s)
        out[(phase, "fft")].append(t.fft_s)
        out[(phase, "ls" if t.kind == "pilot" else "mrc")].append(t.combine_s)
    return out


def records_for_engine(cfg, engine_name, workers, timed_timings, warmup_timings):
    """bench.py:100-140: mean/std per (phase, stage) in µs, then warmup."""
    recs = []
    for (phase, stage), values in _stage_samples(timed_timings).items():
        if not values:
            continue
        arr = np.asarray(values)
        recs.append(BenchRecord(cfg.fft_len, cfg.cp_len, cfg.n_antennas, engine_name, workers, phase, stage,
                                float(arr.mean() * 1e6), float(arr.std() * 1e6), len(values)))
    for phase in PHASES:
        est = phase == "estimation"
        tot = sum(t.total_s for t in warmup_timings if (t.kind == "pilot") == est)
        recs.append(BenchRecord(cfg.fft_len, cfg.cp_len, cfg.n_antennas, engine_name, workers, phase, "warmup",
                                float(tot * 1e6), 0.0, sum(1 for t in warmup_timings if (t.kind == "pilot") == est)))
    return recs


def as_reference_pair(records, parallel="b200"):
    """Records of engine `parallel` relabelled "data_parallel" (others with
    that label dropped), for ofdmrx.bench.speedup_table."""
    out = []
    for r in records:
        if r.engine == "data_parallel":
            continue
        out.append(replace(r, engine="data_parallel") if r.engine == parallel else r)
    return out


def speedup_table(records, parallel="b200"):
    """bench.py:217-249 with `parallel` in the data_parallel role."""
    by_cell = {}
    for r in records:
        if r.stage == "warmup":
            continue
        by_cell.setdefault((r.fft_len, r.n_antennas, r.phase, r.stage), {})[r.engine] = r.mean_us
    missing = sorted(k for k, e in by_cell.items() if not {"sequential", parallel} <= e.keys())
    if missing:
        raise ValueError(f"{len(missing)} cell(s) lack a sequential/{parallel} pair: {missing[:4]}")
    rows, totals = [], {}
    for (m, n, phase, stage), e in sorted(by_cell.items()):
        seq, par = e["sequential"], e[parallel]
        rows.append(SpeedupRow(m, n, phase, stage, seq / par))
        tot = totals.setdefault((m, n, phase), [0.0, 0.0])
        tot[0] += seq
        tot[1] += par
    for (m, n, phase), (seq, par) in sorted(totals.items()):
        rows.append(SpeedupRow(m, n, phase, "total", seq / par))
    rows.sort(key=lambda r: (r.fft_len, r.n_antennas, r.phase, r.stage))
    return rows


def write_bench_csv(records, path):
    """bench.py:266-279 (repr floats, same header)."""
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(CSV_HEADER.split(","))
        for r in records:
            w.writerow((r.fft_len, r.cp_len, r.n_antennas, r.engine, r.workers, r.phase, r.stage,
                        repr(float(r.mean_us)), repr(float(r.std_us)), r.n_symbols))


def read_bench_csv(path):
    """bench.py:282-299."""
    with open(path, newline="", encoding="utf-8") as fh:
        rd = csv.DictReader(fh)
        if rd.fieldnames != CSV_HEADER.split(","):
            raise ValueError(f"CSV header {rd.fieldnames} does not match {CSV_HEADER}")
        return [BenchRecord(int(r["fft_len"]), int(r["cp_len"]), int(r["n_antennas"]), r["engine"], int(r["workers"]),
                            r["phase"], r["stage"], float(r["mean_us"]), float(r["std_us"]), int(r["n_symbols"]))
                for r in rd]

