"""Time sync.detect_frames on C3-sized captures (developer A/B tool)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_07499_b200 import _lib, sync, synth, OfdmConfig  # noqa: E402

if os.environ.get("OFDMRX_VARIANT_LIB"):  # experiment build; the package itself never does this
    _lib.LIB_PATH = os.environ["OFDMRX_VARIANT_LIB"]
F = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cfg = OfdmConfig(1024, 72, 64, qam_order=16)
out = synth.synth_frames(cfg, 10, F, seed=1, snr_db=10.0, timing_offset=0)
pn = synth.generate_pn_chips()
det = sync.detect_frames(out.rx, pn)
torch.cuda.synchronize()
ok = bool((det.frame_start == 0).all())
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    sync.detect_frames(out.rx, pn)
b.record(); torch.cuda.synchronize()
print(json.dumps({"lib": os.environ.get("OFDMRX_VARIANT_LIB", "in-tree"), "frames": F, "us_per_frame": a.elapsed_time(b) / 10 * 1e3 / F, "ok": ok}))
