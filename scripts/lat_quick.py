"""Single-frame latency-path timing (developer tool): C3 and C1, one frame,
receive_frames(latency=True) replayed from a CUDA graph."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1901_07499_b200 import _lib, frames  # noqa: E402

if os.environ.get("OFDMRX_VARIANT_LIB"):  # experiment build; the package itself never does this
    _lib.LIB_PATH = os.environ["OFDMRX_VARIANT_LIB"]

for name in sys.argv[1:] or ["C3", "C1"]:
    n, m, cp, qam, d, _ = bench.CONFIGS[name]
    cfg, rx, bits, s0 = bench.make_inputs(name)
    x = torch.from_numpy(rx[:1]).cuda()
    out = frames.allocate_outputs(1, n, m, d, qam, x.device)
    for lat in (True, False):
        fn = lambda: frames.receive_frames(x, cfg, symbol0_offset=s0, n_data=d, out=out, latency=lat)  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            fn()
            torch.cuda.synchronize()
            with torch.cuda.graph(g):
                fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        ok = bool((out.bits[0].cpu().numpy() == bits[0]).mean() > 0.99)
        print(json.dumps({"cfg": name, "latency_plan": lat, "us_per_frame": a.elapsed_time(b) / 50 * 1e3, "ok": ok}))
