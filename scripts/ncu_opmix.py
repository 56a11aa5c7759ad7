"""Executed-instruction mix by SASS opcode from an ncu report (source page,
--print-source sass): warp-level instructions executed per opcode, and per
unit of work when a divisor is given (e.g. rows processed by the launch).
usage: python scripts/ncu_opmix.py <rep> [divisor] [top]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
mix = collections.Counter()
for r in rows[2:]:
    try:
        n = float(r[ix["Instructions Executed"]].replace(",", ""))
    except (ValueError, IndexError):
        continue
    src = r[ix["Source"]].strip()
    toks = src.split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    mix[op.split(".")[0]] += n
tot = sum(mix.values())
print(f"total warp instructions {tot:.4g}  per unit {tot / div:.1f}")
for op, n in mix.most_common(top):
    print(f"  {op:10s} {n / div:9.1f} per unit  {100 * n / tot:5.1f}%")
