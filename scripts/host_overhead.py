"""Host-side cost of one receive_frames call (developer tool): wall time per
call enqueued back to back with no sync, vs the device time per call, and a
cProfile of the Python wrapper.  usage: python scripts/host_overhead.py [CFG]"""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1901_07499_b200 import frames  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
n, m, cp, qam, d, F = bench.CONFIGS[name]
cfg, rx, bits, s0 = bench.make_inputs(name)
x = torch.from_numpy(rx).cuda().repeat((F + len(rx) - 1) // len(rx), 1, 1)[:F].contiguous()
out = frames.allocate_outputs(F, n, m, d, qam, x.device)
for _ in range(5):
    frames.receive_frames(x, cfg, symbol0_offset=s0, n_data=d, out=out)
torch.cuda.synchronize()
reps = 200
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
a.record()
for _ in range(reps):
    frames.receive_frames(x, cfg, symbol0_offset=s0, n_data=d, out=out)
b.record()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"{name}: host enqueue {1e6 * (t1 - t0) / reps:.1f} us/call, device {1e3 * a.elapsed_time(b) / reps:.1f} us/call")
pr = cProfile.Profile()
pr.enable()
for _ in range(reps):
    frames.receive_frames(x, cfg, symbol0_offset=s0, n_data=d, out=out)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
