"""Small-shape invocations of every device kernel, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  Developer tool.

    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py [case ...]

Cases: balanced (C3 1 and 13 frames, C4 1 frame: cluster + DSMEM epilogue,
M=4096, N<workers), fused (C1/C2 shapes, ZF, non-BPSK pilot), partials,
staged, detect (corr_fft_kernel + refine), corr (direct corr_kernel),
synth, peer (self-mapped inbox: routed partials, signal/wait, finish)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_07499_b200 as P  # noqa: E402
from paper_1901_07499_b200 import _lib  # noqa: E402
from oracle import ofdm_oracle as orc  # noqa: E402

if os.environ.get("OFDMRX_VARIANT_LIB"):  # sanitizer build (scripts/sanitize.sh); the package never does this
    _lib.LIB_PATH = os.environ["OFDMRX_VARIANT_LIB"]


def caps(m, cp, n, qam, d, k, seed=0):
    cs = [orc.synth_capture(m, cp, n, qam, d, seed + i, snr_db=10.0) for i in range(k)]
    return torch.from_numpy(np.stack([c[0] for c in cs]).astype(np.complex64)).cuda(), cs[0][2], cs


def check(out, cs, m, cp, d, qam, s0):
    for i, c in enumerate(cs):
        _, _, _, bits = orc.receive_frame(c[0], s0, m, cp, d, qam)
        assert np.array_equal(out.bits[i].cpu().numpy(), bits)


def balanced():
    for (n, m, cp, qam, d, k) in ((64, 1024, 72, 16, 10, 1), (64, 1024, 72, 16, 10, 13), (256, 2048, 256, 64, 10, 1),
                                  (4, 4096, 512, 16, 3, 2), (2, 1024, 72, 4, 2, 3)):
        x, s0, cs = caps(m, cp, n, qam, d, k)
        out = P.receive_frames(x, P.OfdmConfig(m, cp, n, qam_order=qam), symbol0_offset=s0, n_data=d)
        torch.cuda.synchronize()
        check(out, cs, m, cp, d, qam, s0)
        out = P.receive_frames(x, P.OfdmConfig(m, cp, n, qam_order=qam), symbol0_offset=s0, n_data=d, zf=True)
        torch.cuda.synchronize()


def latency():
    for (n, m, cp, qam, d, k) in ((64, 1024, 72, 16, 10, 2), (8, 64, 16, 4, 10, 3), (16, 2048, 256, 64, 3, 1)):
        x, s0, cs = caps(m, cp, n, qam, d, k)
        cfg = P.OfdmConfig(m, cp, n, qam_order=qam)
        out = P.receive_frames(x, cfg, symbol0_offset=s0, n_data=d, latency=True)
        torch.cuda.synchronize()
        check(out, cs, m, cp, d, qam, s0)
        P.receive_frames(x, cfg, symbol0_offset=s0, n_data=d, latency=True, zf=True, profile=True)
        torch.cuda.synchronize()


def fused():
    for (n, m, cp, qam, d, k) in ((8, 64, 16, 4, 10, 5), (16, 256, 32, 16, 10, 3), (3, 512, 64, 64, 20, 2)):
        x, s0, cs = caps(m, cp, n, qam, d, k)
        cfg = P.OfdmConfig(m, cp, n, qam_order=qam)
        out = P.receive_frames(x, cfg, symbol0_offset=s0, n_data=d)
        torch.cuda.synchronize()
        check(out, cs, m, cp, d, qam, s0)
        P.receive_frames(x, cfg, symbol0_offset=s0, n_data=d, zf=True)
        pil = P.PilotDefinition(np.exp(1j * np.linspace(0, 6, m)))
        P.receive_frames(x, cfg, pil, symbol0_offset=s0, n_data=d)
        torch.cuda.synchronize()


def partials():
    from paper_1901_07499_b200 import frames
    for (n, m, cp, qam, d, k) in ((16, 256, 32, 16, 5, 4), (32, 2048, 256, 64, 3, 2)):
        x, s0, cs = caps(m, cp, n, qam, d, k)
        cfg = P.OfdmConfig(m, cp, n, qam_order=qam)
        _, num, den, fl = frames.receive_partials(x, cfg, symbol0_offset=s0, n_data=d)
        frames.finish_partials(num[None], den[None], qam)
        torch.cuda.synchronize()


def staged():
    from paper_1901_07499_b200 import frames, receiver as R
    eng = R.B200Engine(fused=False)
    tree = R.B200Engine(tree=True, fused=False)
    for m in (64, 1024, 4096):
        t = (np.random.default_rng(m).standard_normal((4, m)) + 1j).astype(np.complex128)
        y = eng.freq_transform(t)
        h = eng.ls_divide(y, np.sign(np.random.default_rng(1).standard_normal(m)) + 0j)
        eng.mrc(y, h, 1e-12)
        tree.mrc(y, h, 1e-12)
        P.waveform.qam_demap(y[0], 16)
    x, s0, cs = caps(256, 32, 16, 16, 4, 2)
    cfg = P.OfdmConfig(256, 32, 16, qam_order=16)
    st = frames.stage_symbols(x, cfg, symbol0_offset=s0, n_data=4)
    frames.receive_staged(st, cfg)
    torch.cuda.synchronize()


def detect():
    from paper_1901_07499_b200 import sync
    x, s0, cs = caps(1024, 72, 4, 16, 3, 2)
    cfg = P.OfdmConfig(1024, 72, 4, qam_order=16)
    P.frames.receive_captures(x, cfg, 3)
    sync.detect_frames(x, orc.generate_pn(), antennas="all")
    torch.cuda.synchronize()


def corr():
    from paper_1901_07499_b200 import sync
    x, s0, cs = caps(64, 16, 2, 4, 2, 1)
    sync.corr_metrics(x[0, 0].cpu().numpy(), orc.generate_pn())
    torch.cuda.synchronize()


def synth():
    from paper_1901_07499_b200 import synth as sy
    sy.synth_batch(P.OfdmConfig(256, 32, 4, qam_order=16), 3, range(3), snr_db=10.0)
    torch.cuda.synchronize()


CASES = {f.__name__: f for f in (balanced, latency, fused, partials, staged, detect, corr, synth)}

if __name__ == "__main__":
    torch.cuda.set_device(0)
    for name in (sys.argv[1:] or list(CASES)):
        CASES[name]()
        print("case", name, "ok", flush=True)
