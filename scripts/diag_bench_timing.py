"""Developer diagnosis: host enqueue cost vs GPU time of receive_frames (C3)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1901_07499_b200 import frames  # noqa: E402

n, m, cp, qam, d, F = bench.CONFIGS["C3"]
cfg, rx, bits, s0 = bench.make_inputs("C3")
dev = torch.device("cuda", 0)
x = torch.from_numpy(rx).to(dev).repeat((F + 15) // 16, 1, 1)[:F].contiguous()
out = frames.allocate_outputs(F, n, m, d, qam, dev)
stream = torch.cuda.current_stream()


def step():
    frames.receive_frames(x, cfg, symbol0_offset=s0, n_data=d, out=out)


for _ in range(5):
    step()
torch.cuda.synchronize()
import subprocess  # noqa: E402
smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,"
                        "clocks_event_reasons.active", "--format=csv,noheader", "-lms", "20"],
                       stdout=open("gpurun_out/diag_smi.csv", "w"), stderr=subprocess.DEVNULL)
time.sleep(0.5)
for rep in range(8):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a.record(stream)
    for i in range(50):
        step()
    b.record(stream)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"gpu {a.elapsed_time(b) / 50:.4f} ms/step  host enqueue {(t1 - t0) * 1e3 / 50:.4f} ms/call  "
          f"wall {(t2 - t0) * 1e3 / 50:.4f} ms/step", flush=True)
time.sleep(0.3)
smi.terminate()
# pure host cost of the Python wrapper pieces
import numpy as np  # noqa: E402
from paper_1901_07499_b200 import device  # noqa: E402

pv = frames._pilot_values(None, m)
t0 = time.perf_counter()
for _ in range(200):
    frames._pilot_values(None, m)
print(f"_pilot_values {(time.perf_counter() - t0) * 1e3 / 200:.4f} ms")
t0 = time.perf_counter()
for _ in range(200):
    device.pilot_options(pv)
print(f"pilot_options {(time.perf_counter() - t0) * 1e3 / 200:.4f} ms")
t0 = time.perf_counter()
for _ in range(200):
    frames._PILOTS.get(pv, dev)
print(f"_PILOTS.get {(time.perf_counter() - t0) * 1e3 / 200:.4f} ms")
