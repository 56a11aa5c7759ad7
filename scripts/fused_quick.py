"""A/B timing of the fused receive kernel (developer tool, not the bench).

    OFDMRX_VARIANT_LIB=build/variants/libofdmrx_b200_X.so python scripts/fused_quick.py [C3] [frames]

Prints ms per launch, µs per frame and the fraction of the measured HBM peak
(algorithmic bytes), plus BER of the tiled frames vs truth."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1901_07499_b200 import _lib, frames  # noqa: E402

if os.environ.get("OFDMRX_VARIANT_LIB"):  # experiment build (build.py --variant); the package itself never does this
    _lib.LIB_PATH = os.environ["OFDMRX_VARIANT_LIB"]

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "C3"
if cfg_name not in bench.CONFIGS:  # "NxM": N antennas, FFT M, CP M/8, 16-QAM, 10 data symbols
    n_, m_ = (int(v) for v in cfg_name.split("x"))
    bench.CONFIGS[cfg_name] = (n_, m_, max(1, m_ // 8), 16, 10, 1024)
n, m, cp, qam, d, F = bench.CONFIGS[cfg_name]
if len(sys.argv) > 2:
    F = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
cfg, rx, bits, s0 = bench.make_inputs(cfg_name)
x = torch.from_numpy(rx).cuda().repeat((F + len(rx) - 1) // len(rx), 1, 1)[:F].contiguous()
out = frames.allocate_outputs(F, n, m, d, qam, x.device)
for _ in range(3):
    frames.receive_frames(x, cfg, symbol0_offset=s0, n_data=d, out=out)
torch.cuda.synchronize()
ber = float((out.bits[:len(rx)].cpu().numpy() != bits[:min(len(rx), F)]).mean())
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    frames.receive_frames(x, cfg, symbol0_offset=s0, n_data=d, out=out)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
peak, _ = bench.load_peaks()
bpf = bench.frame_bytes(n, m, qam, d)
print(json.dumps({"lib": os.environ.get("OFDMRX_VARIANT_LIB", "in-tree"), "cfg": cfg_name, "frames": F, "reps": reps, "ms": ms,
                  "us_per_frame": ms * 1e3 / F, "frac": bpf * F / (ms * 1e-3) / 1e9 / peak, "ber": ber}))
