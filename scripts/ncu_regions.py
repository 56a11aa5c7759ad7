"""Stall samples and executed instructions of an ncu report split at marker
opcodes (developer tool): prints cumulative sample shares in SASS address
order with the positions of MUFU / BAR / STG instructions, to attribute time
to kernel regions.  usage: python scripts/ncu_regions.py REP"""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}


def f(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except Exception:
        return 0.0


data = rows[2:]
tot = sum(f(r, "# Samples") for r in data) or 1.0
cum = 0.0
last_print = -1.0
for r in data:
    cum += f(r, "# Samples")
    src = r[ix["Source"]]
    mark = any(k in src for k in ("MUFU", "BAR.SYNC", "BAR.ARV", "STG", "SYNCS.ARRIVE", "TCGEN05", "UTCBAR", "EXIT"))
    if mark or cum / tot - last_print > 0.05:
        print(f"{r[ix['Address']][-5:]} cum {100 * cum / tot:5.1f}%  x{int(f(r, 'Instructions Executed')):>9d}  {src[:60]}")
        last_print = cum / tot
