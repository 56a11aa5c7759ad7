"""Top SASS instructions by stall samples from an ncu report (source page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}


def f(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except Exception:
        return 0.0


tot = sum(f(r, "# Samples") for r in data)
print("instructions:", len(data), "samples:", tot)
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for r in sorted(data, key=lambda r: -f(r, "# Samples"))[:n]:
    st = {k[6:]: int(f(r, k)) for k in stall_cols if f(r, k) > 0}
    st = dict(sorted(st.items(), key=lambda x: -x[1])[:3])
    print(f"{r[ix['Address']][-5:]} {r[ix['Source']][:58]:58s} {100*f(r,'# Samples')/tot:5.1f}% x{int(f(r,'Instructions Executed'))} {st}")
