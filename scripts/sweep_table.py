"""profiles/sweep_rNN.md from bench.py --sweep outputs (the .json summary next
to the reference-schema .csv).
usage: python scripts/sweep_table.py profiles/sweep_r02.json profiles/sweep_r02.md"""
import json
import sys

src, dst = sys.argv[1], sys.argv[2]
cells = json.load(open(src))
out = ["# C5 sweep: B200 vs the reference CPU path, per OFDM symbol (16-QAM, D = 10, default_cp)", "",
       f"Source: `bench.py --sweep` -> `{src}` and the reference-schema CSV next to it (read by the",
       "reference's own `ofdmrx.bench.read_bench_csv` / `speedup_table`, tests/test_benchcsv_cpu.py).", "",
       "* fused: one fused launch over F frames resident in HBM (CUDA-graph replays, GPU time), and its",
       "  fraction of the measured HBM roofline (algorithmic bytes, SURVEY §8(d));",
       "* batched stages: the staged kernels (each writes its intermediate to HBM);",
       "* pipeline: `run_ring_pipeline` on one frame's slots, per symbol, wall clock: the unmodified",
       "  reference (numba SequentialEngine, 1 core) vs the mirror's B200 engine (H2D + one launch + D2H",
       "  per pilot-led segment, the paper's regime); bits equal in every cell.", "",
       "| FFT | N | F | fused µs/sym | roofline | fft µs/sym | ls µs/pilot | mrc+demap µs/sym | ref pipeline µs/sym | B200 pipeline µs/sym | pipeline speedup |",
       "|---|---|---|---|---|---|---|---|---|---|---|"]
for c in sorted(cells, key=lambda c: (c["fft_len"], c["n_antennas"])):
    b = c["b200_batched_us_per_symbol"]
    pl = c.get("pipeline_us_per_symbol", {})
    r, g = pl.get("reference_sequential"), pl.get("b200")
    f = lambda x: "-" if x is None else (f"{x:.4f}" if x < 1 else (f"{x:.2f}" if x < 100 else f"{x:,.0f}"))  # noqa: E731
    out.append(f"| {c['fft_len']} | {c['n_antennas']} | {c['frames']} | {f(c['fused_us_per_symbol'])} | "
               f"{100 * c['roofline_frac']:.1f} % | {f(b['fft'])} | {f(b['ls'])} | {f(b['mrc+demap'])} | {f(r)} | "
               f"{f(g)} | {'-' if not (r and g) else f'{r / g:.1f}x'} |")
open(dst, "w").write("\n".join(out) + "\n")
