"""profiles/sweep_rNN.md from a bench.py --sweep CSV (reference bench schema)."""
import csv
import sys
from collections import defaultdict

src, dst = sys.argv[1], sys.argv[2]
rows = list(csv.DictReader(open(src)))
t = defaultdict(dict)
for r in rows:
    key = (int(r["fft_len"]), int(r["n_antennas"]))
    t[key][(r["engine"], r["phase"], r["stage"])] = float(r["mean_us"])
out = ["# C5 sweep: µs per OFDM symbol, B200 vs reference CPU (numba SequentialEngine, 1 core)", "",
       f"Source: `bench.py --sweep` -> `{src}` (reference bench CSV schema).  B200 stages are CUDA-graph",
       "replayed (GPU time only); data symbol = FFT + MRC + demap.", "",
       "| FFT | N ant | B200 fused µs/sym | B200 staged fft | B200 mrc+demap | CPU fft | CPU ls | CPU mrc+demap | CPU data-symbol / B200 fused |",
       "|---|---|---|---|---|---|---|---|---|"]
for (m, n), v in sorted(t.items()):
    fused = v.get(("b200", "demodulation", "fused"))
    fft = v.get(("b200", "estimation", "fft"))
    mrc = v.get(("b200", "demodulation", "mrc"))
    cf, cl, cm = (v.get(("sequential", ph, st)) for ph, st in
                  (("estimation", "fft"), ("estimation", "ls"), ("demodulation", "mrc")))
    ratio = f"{(cf + cm) / fused:,.0f}x" if cf and cm and fused else "-"
    f = lambda x: "-" if x is None else (f"{x:.3f}" if x < 10 else f"{x:.1f}")  # noqa: E731
    out.append(f"| {m} | {n} | {f(fused)} | {f(fft)} | {f(mrc)} | {f(cf)} | {f(cl)} | {f(cm)} | {ratio} |")
open(dst, "w").write("\n".join(out) + "\n")
