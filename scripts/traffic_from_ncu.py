"""Write profiles/traffic_<cfg>.json from an ncu --set full report of one
rx_fused launch: dram__bytes_read.sum + dram__bytes_write.sum per frame.
usage: python scripts/traffic_from_ncu.py <rep> <frames_in_launch> <cfg> [label]"""
import csv
import json
import subprocess
import sys

rep, frames, cfg = sys.argv[1], int(sys.argv[2]), sys.argv[3]
label = sys.argv[4] if len(sys.argv) > 4 else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
d = {}
for h, u, v in zip(hdr, units, vals):
    try:
        d[h] = (float(v.replace(",", "")), u)
    except ValueError:
        pass
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = d["dram__bytes_read.sum"][0] * scale[d["dram__bytes_read.sum"][1]]
wr = d["dram__bytes_write.sum"][0] * scale[d["dram__bytes_write.sum"][1]]
dur = d["gpu__time_duration.sum"][0] * {"ns": 1e-9, "us": 1e-6, "ms": 1e-3}[d["gpu__time_duration.sum"][1]]
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import bench  # noqa: E402

out = {"dram_bytes_per_frame": (rd + wr) / frames, "kernel_source_hash": bench.kernel_source_hash(), "dram_read_bytes": rd, "dram_write_bytes": wr,
       "frames_in_launch": frames, "ncu_duration_s": dur, "source": label,
       "note": "ncu --set full --clock-control none, one launch of the product kernel; writes still resident in L2 at "
               "kernel end are not counted by dram__bytes_write"}
json.dump(out, open(f"profiles/traffic_{cfg}.json", "w"), indent=1)
print(out)
