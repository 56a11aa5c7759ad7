"""Pinned H2D bandwidth: one stream vs several concurrent streams."""
import torch
n = 1 << 27  # complex64 elements = 1 GiB
host = torch.empty(n, dtype=torch.complex64).pin_memory()
dev = torch.empty(n, dtype=torch.complex64, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = n // ns
    best = 0
    for _ in range(5):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i, s in enumerate(streams):
            s.wait_event(a)
            with torch.cuda.stream(s):
                dev[i * chunk:(i + 1) * chunk].copy_(host[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        b.record(); b.synchronize()
        best = max(best, n * 8 / (a.elapsed_time(b) * 1e-3) / 1e9)
    print(f"streams={ns} H2D {best:.1f} GB/s")
