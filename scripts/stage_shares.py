"""Per-stage shares of the fused kernel's lane time (ofdmrx_rx_frames_profiled)
for a config at a batch size (developer tool)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1901_07499_b200 import frames  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
F = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
n, m, cp, qam, d, _ = bench.CONFIGS[name]
cfg, rx, bits, s0 = bench.make_inputs(name)
x = torch.from_numpy(rx).cuda().repeat((F + len(rx) - 1) // len(rx), 1, 1)[:F].contiguous()
for _ in range(2):
    out = frames.receive_frames(x, cfg, symbol0_offset=s0, n_data=d, profile=True)
torch.cuda.synchronize()
sh = out.stage_shares()
print(json.dumps({"cfg": name, "frames": F, "shares": dict(zip(["pilot_fft", "ls", "data_fft", "mrc", "epilogue"],
                                                              [round(v, 4) for v in sh]))}))
