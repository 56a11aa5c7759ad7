"""Top SASS instructions of an ncu report by any source-page column (e.g.
'L1 Wavefronts Shared Excessive').  usage: python scripts/ncu_col.py REP COLUMN [N]
With COLUMN = '?' lists the available columns."""
import csv
import subprocess
import sys

rep, col = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
if col == "?":
    print("\n".join(hdr))
    sys.exit(0)
ix = {h: i for i, h in enumerate(hdr)}


def f(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except Exception:
        return 0.0


data = rows[2:]
tot = sum(f(r, col) for r in data) or 1.0
print(col, "total", tot)
for r in sorted(data, key=lambda r: -f(r, col))[:n]:
    print(f"{r[ix['Address']][-5:]} {r[ix['Source']][:70]:70s} {f(r, col):12.0f} {100 * f(r, col) / tot:5.1f}%")
