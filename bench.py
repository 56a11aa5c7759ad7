#!/usr/bin/env python
"""Benchmark of the fused B200 uplink receive path (BASELINE.json metric:
OFDM symbols/s at 64 antennas x FFT-1024, 16-QAM, 1 pilot + 10 data
symbols per frame; frame-sharded over 1/2/4/8 GPUs, weak scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

One step = one fused launch over F frames per GPU resident in HBM (inputs
6.3 GB/GPU >> 126 MB L2, so no L2 flush is needed between steps).
Prints one JSON line on rank 0.
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (N antennas, M, CP, QAM, D data symbols, frames per GPU)
    "C1": (8, 64, 16, 4, 10, 65536),
    "C2": (16, 256, 32, 16, 10, 1000),
    "C3": (64, 1024, 72, 16, 10, 1024),
    "C4": (256, 2048, 256, 64, 10, 64),
}
METRIC = "OFDM symbols/s & per-stage µs/symbol at 64 ant × FFT 1024, 1/2/4/8 B200"
DISTINCT = 16  # distinct synthetic frames, tiled on the device


def frame_bytes(n, m, qam, d):
    """Algorithmic HBM bytes per frame: rx samples of the
    1+D symbols without CP, H written once, s_hat, bits as u8."""
    b = int(math.log2(qam))
    return 8 * n * m * (1 + d) + 8 * n * m + 8 * m * d + b * m * d


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []  # (host receipt time, csv line)
        self.window = None

    def mark(self, t0, t1):
        """Host wall-clock (time.time()) bounds of the timed region: only
        samples nvidia-smi timestamped inside it enter the summary (idle
        samples would mask a power cap)."""
        self.window = (t0, t1)

    @staticmethod
    def _stamp(text):
        import datetime

        try:
            return datetime.datetime.strptime(text.strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except ValueError:
            return None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "10"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True, bufsize=1)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            line = line.strip()
            self.lines.append((self._stamp(line.split(",")[0]), line))

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if self.window is not None:
            t0, t1 = self.window
            inside = [x for x in lines if x[0] is not None and t0 <= x[0] <= t1]
            if not inside:  # region shorter than the period: the first sample after it started
                inside = [x for x in lines if x[0] is not None and x[0] >= t0][:1]
            lines = inside
        for _, line in lines:
            parts = [p.strip() for p in line.split(",")][1:]  # drop the timestamp
            if len(parts) < 6:
                continue
            if len(parts) > 6:
                try:
                    power.append(float(parts[6].split()[0]))
                except (ValueError, IndexError):
                    pass
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": ["unsampled"]}
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
               "window": "timed region only" if self.window is not None else "whole sampler run"}
        if power:
            out["power_w_median"] = statistics.median(power)
        return out


def dist_setup(n_gpus):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # OFDMRX_DIST_BACKEND=gloo + OFDMRX_SAME_DEVICE=1 run every rank on cuda:0
    # (single-GPU smoke test of the multi-rank code path; not a measurement)
    backend = os.environ.get("OFDMRX_DIST_BACKEND", "nccl")
    dev = 0 if os.environ.get("OFDMRX_SAME_DEVICE") == "1" else local
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, dev


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def allreduce_max(world, value):
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def make_inputs(cfg_name, seed_base=0):
    from paper_1901_07499_b200 import synth
    from paper_1901_07499_b200.waveform import OfdmConfig

    n, m, cp, qam, d, _ = CONFIGS[cfg_name]
    cfg = OfdmConfig(m, cp, n, qam_order=qam)
    rx, bits, s0 = synth.synth_batch(cfg, d, range(seed_base, seed_base + DISTINCT), snr_db=10.0)
    return cfg, rx, bits, s0


# ---------------------------------------------------------------------------
# CPU baselines
# ---------------------------------------------------------------------------

def cpu_port_baseline(cfg_name, rx_host, budget_s=10.0):
    """The oracle port (numpy restatement of the reference path), 1 thread,
    on a bounded sample of the same frames."""
    from oracle import ofdm_oracle as orc

    n, m, cp, qam, d, _ = CONFIGS[cfg_name]
    x = rx_host.astype(np.complex128)
    frames = 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < budget_s:
        orc.receive_frame(x[frames % x.shape[0]], 0, m, cp, d, qam)
        frames += 1
    dt = time.perf_counter() - t0
    return {"value": frames * (1 + d) / dt, "unit": "symbols/s", "cores": 1, "kind": "port",
            "sample": f"{frames} {cfg_name} frames ({frames * (1 + d)} OFDM symbols), oracle/ofdm_oracle.py "
                      f"receive_frame (numpy radix-2 as reference numpy_backend), {dt:.1f} s"}


_REF_NUMPY_SNIPPET = r"""
import json, sys, time
import numpy as np
from ofdmrx import receiver as rref, waveform as wref
from ofdmrx.kernels import BACKEND
from ofdmrx.sync import DetectionResult
x = np.load(sys.argv[1]).astype(np.complex128)
m, cp, n, qam, d, budget = (float(v) if i == 5 else int(v) for i, v in enumerate(sys.argv[2:8]))
cfg = wref.OfdmConfig(m, cp, n, qam_order=qam)
pilot = wref.make_pilot(m)
class Cap:
    def __init__(self, s): self.streams = s
det = DetectionResult(True, 0, 0, 1.0, ())
slots = [rref.extract_slots(Cap(f), det, cfg, 1 + d) for f in x]
eng = rref.make_engine(rref.EngineKind("sequential"))
frames, t0 = 0, time.perf_counter()
while time.perf_counter() - t0 < budget:
    rref.run_ring_pipeline(slots[frames % len(slots)], cfg, eng, pilot=pilot)
    frames += 1
dt = time.perf_counter() - t0
print(json.dumps({"frames": frames, "seconds": dt, "backend": BACKEND}))
"""


def cpu_reference_numpy_baseline(cfg_name, rx_host, budget_s=10.0):
    """The reference's own numpy CPU path (baseline/_ref with
    OFDMRX_BACKEND=numpy: the north star's "reference numpy CPU path"),
    SequentialEngine, 1 thread, timed in a subprocess (the backend is fixed
    at import) on a bounded sample of the same frames.  None if the
    reference is not installed."""
    import tempfile

    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "ofdmrx")):
        return None
    n, m, cp, qam, d, _ = CONFIGS[cfg_name]
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "frames.npy")
        np.save(path, rx_host)
        env = dict(os.environ, OFDMRX_BACKEND="numpy", PYTHONPATH=ref, OMP_NUM_THREADS="1",
                   OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
        try:
            out = subprocess.run([sys.executable, "-c", _REF_NUMPY_SNIPPET, path, str(m), str(cp), str(n), str(qam),
                                  str(d), str(budget_s)], env=env, capture_output=True, text=True,
                                 timeout=budget_s * 4 + 120)
            res = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception:  # noqa: BLE001
            return None
    return {"value": res["frames"] * (1 + d) / res["seconds"], "unit": "symbols/s", "cores": 1, "kind": "reference",
            "sample": f"{res['frames']} {cfg_name} frames ({res['frames'] * (1 + d)} OFDM symbols), unmodified "
                      f"reference ofdmrx run_ring_pipeline, backend={res['backend']}, SequentialEngine, "
                      f"{res['seconds']:.1f} s"}


def reference_importable():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "ofdmrx")):
        if ref not in sys.path:
            sys.path.insert(0, ref)
        return True
    return False


def run_reference_arm(args, cfg_name, world, rank):
    """--impl reference: the reference's own CPU implementation of the path
    (baseline/_ref = unmodified ofdmrx, run_ring_pipeline) on this host's
    cores; falls back to the oracle port when the install is absent."""
    n, m, cp, qam, d, _ = CONFIGS[cfg_name]
    if rank != 0:
        return None
    ncores = len(os.sched_getaffinity(0))
    from paper_1901_07499_b200 import synth
    from paper_1901_07499_b200.waveform import OfdmConfig

    cfg = OfdmConfig(m, cp, n, qam_order=qam)
    caps = [synth.synth_capture(cfg, d, s, 10.0) for s in range(4)]
    line = {"metric": METRIC, "unit": "symbols/s", "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "c128", "data": "synthetic (reference TX + flat Rayleigh 10 dB)",
            "config": {"workload": f"{cfg_name}: {n} ant x FFT {m} (CP {cp}), {qam}-QAM, 1 pilot + {d} data "
                                   "symbols/frame", "frames_per_step": None}}
    if not reference_importable():
        # oracle port (numpy restatement) as the reference CPU implementation
        from oracle import ofdm_oracle as orc

        def step(nf):
            for i in range(nf):
                c = caps[i % len(caps)]
                orc.receive_frame(c.streams, c.symbol0_offset, m, cp, d, qam)
        engine_desc, kind, cores = "oracle port (numpy, 1 thread)", "port", 1
    else:
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/ofdmrx_numba_cache")
        from ofdmrx import receiver as rref, waveform as wref
        from ofdmrx.sync import DetectionResult

        class _Cap:
            def __init__(self, s):
                self.streams = s

        rcfg = wref.OfdmConfig(m, cp, n, qam_order=qam)
        pilot = wref.make_pilot(m)
        slot_sets = [rref.extract_slots(_Cap(c.streams), DetectionResult(True, 0, c.symbol0_offset, 1.0, ()),
                                        rcfg, 1 + d) for c in caps]
        engines = {"sequential": rref.EngineKind("sequential"),
                   f"data_parallel({ncores})": rref.EngineKind("data_parallel", ncores)}
        best = None
        for name, kind_ in engines.items():
            with rref.make_engine(kind_) as eng:
                rref.run_ring_pipeline(slot_sets[0], rcfg, eng, pilot=pilot)  # JIT / pool warm-up
                t0 = time.perf_counter()
                rref.run_ring_pipeline(slot_sets[1], rcfg, eng, pilot=pilot)
                dt = time.perf_counter() - t0
            if best is None or dt < best[1]:
                best = (name, dt, kind_)
        from ofdmrx import kernels as kref

        chosen = best[2]
        eng = rref.make_engine(chosen)

        def step(nf):
            for i in range(nf):
                rref.run_ring_pipeline(slot_sets[i % len(slot_sets)], rcfg, eng, pilot=pilot)
        engine_desc = f"reference ofdmrx run_ring_pipeline, backend={kref.BACKEND}, engine={best[0]} " \
                      f"(fastest of sequential / data_parallel({ncores}))"
        kind = "reference"
        cores = ncores if chosen.variant == "data_parallel" else 1
    # size each step to ~2 s of CPU work
    t0 = time.perf_counter()
    step(1)
    per_frame = max(time.perf_counter() - t0, 1e-4)
    nf = max(1, int(2.0 / per_frame))
    for _ in range(args.warmup):
        step(nf)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step(nf)
    dt = time.perf_counter() - t0
    value = args.steps * nf * (1 + d) / dt
    line.update({"value": value, "ms_per_step": dt / args.steps * 1e3,
                 "cpu_baseline": {"value": value, "unit": "symbols/s", "cores": cores, "kind": kind,
                                  "sample": f"{nf} frames/step x {args.steps} steps; {engine_desc}"},
                 "e2e": {"value": value, "unit": "symbols/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
    line["config"]["frames_per_step"] = nf
    return line


# ---------------------------------------------------------------------------
# the B200 arm
# ---------------------------------------------------------------------------

def run_b200(args, cfg_name, world, rank, local):
    import torch

    import paper_1901_07499_b200 as P
    from paper_1901_07499_b200 import frames

    n, m, cp, qam, d, F = CONFIGS[cfg_name]
    if args.frames:
        F = args.frames
    dev = torch.device("cuda", torch.cuda.current_device())
    antenna_sharded = cfg_name == "C4" and world > 1
    # frame sharding: distinct frames per rank; antenna sharding: every rank
    # holds its antenna rows of the SAME frames
    cfg, rx_host, bits_truth, s0 = make_inputs(cfg_name, seed_base=0 if antenna_sharded else 1000 * rank)
    base = torch.from_numpy(rx_host).to(dev)
    reps = (F + DISTINCT - 1) // DISTINCT
    x = base.repeat(reps, 1, 1)[:F].contiguous()
    del base
    out = frames.allocate_outputs(F, n, m, d, qam, dev)
    stream = torch.cuda.current_stream()

    sharded = None
    if antenna_sharded:
        # antenna-sharded MRC: every rank holds N/world antennas of the same frames
        from paper_1901_07499_b200 import sharding

        sharded = sharding.AntennaShardedReceiver(cfg, d, symbol0_offset=s0, mode=args.exchange)
        x = x[:, sharded.ant_lo:sharded.ant_hi].contiguous()

    own = slice(None)
    if sharded is not None and args.exchange == "peer":  # each rank finishes its F/world frames
        own = slice(rank * (F // world), (rank + 1) * (F // world))

    def step():
        if sharded is not None:
            s_hat, w, bits, fl, _ = sharded.receive(x)
            out.bits[own].copy_(bits)
            out.flags[own].copy_(fl)
        else:
            frames.receive_frames(x, cfg, symbol0_offset=s0, n_data=d, out=out)

    # correctness spot-check of the benchmarked configuration (bits vs truth)
    step()
    torch.cuda.synchronize()
    lo = own.start or 0
    hi = min(own.stop if own.stop is not None else F, lo + DISTINCT)
    idx = np.arange(lo, hi)
    ber = float((out.bits[lo:hi].cpu().numpy() != bits_truth[idx % len(bits_truth)]).mean())
    flags_bad = int((out.flags != 0).sum())
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        time.sleep(0.3)  # sampler running before the warm-up
        # the warm-up steps run right before the timed region: an idle gap here
        # lets the SM clock drop and the first timed launches pay the ramp
        for _ in range(max(0, args.warmup - 1)):
            step()
        torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        t_start = torch.cuda.Event(enable_timing=True)
        t_stop = torch.cuda.Event(enable_timing=True)
        h0 = time.time()
        t_start.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        t_stop.record(stream)
        torch.cuda.synchronize()
        clocks.mark(h0, time.time())
        time.sleep(0.25)  # let nvidia-smi deliver the samples it took inside the window
        barrier(world)
    total_ms = t_start.elapsed_time(t_stop)
    kernel_ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    ms_step = allreduce_max(world, total_ms / args.steps)
    # frame sharding: every rank owns F distinct frames; antenna sharding: all
    # ranks cooperate on the same F frames
    value = (1 if sharded is not None else world) * F * (1 + d) / (ms_step * 1e-3)

    peak, peak_kind = load_peaks()
    bpf = frame_bytes(n // (world if sharded is not None else 1), m, qam, d)
    achieved = bpf * F / (kernel_ms * 1e-3) / 1e9
    traffic = traffic_detail = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{cfg_name}.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            tj = json.load(fh)
        if "dram_bytes_per_frame" in tj:
            # same units as `achieved`: the ncu-measured DRAM bytes of one launch
            # of this size over the live kernel time
            traffic = tj["dram_bytes_per_frame"] * F / (kernel_ms * 1e-3) / 1e9
            traffic_detail = {"dram_bytes_per_launch": int(tj["dram_bytes_per_frame"] * F),
                              "algorithmic_bytes_per_launch": int(frame_bytes(n // (world if sharded is not None else 1),
                                                                              m, qam, d) * F),
                              "source": tj.get("source")}

    line = {
        "metric": METRIC, "value": value, "unit": "symbols/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32 (cf32 I/O)",
        "data": "synthetic: reference TX (PN|pilot|data, Gray QAM) through flat Rayleigh at 10 dB; "
                f"{DISTINCT} distinct frames tiled on device",
        "config": {"workload": f"{cfg_name}: {n} ant x FFT {m} (CP {cp}), {qam}-QAM, 1 pilot + {d} data symbols/frame",
                   "frames_per_gpu": F, "global_frames": F if sharded is not None else F * world, "parallelism": (f"antenna-sharded x{world} ({args.exchange} exchange of MRC partials"
                                   f"{' over peer memory, no NCCL' if args.exchange == 'peer' else ' over NCCL'})"
                                   if sharded is not None else f"frame-sharded x{world}"),
                   "input_bytes_per_gpu": int(x.numel() * 8), "l2": "inputs 6.3 GB/GPU > L2, no flush needed"
                   if x.numel() * 8 > 126e6 else "inputs smaller than L2"},
        "gpu_launches": args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_detail": traffic_detail, "peak_source": peak_kind,
                     "bytes_per_frame": bpf, "kernel_ms": kernel_ms},
        "clocks": clocks.summary(),
        "check": {"ber_vs_tx": ber, "flagged_frames": flags_bad},
        "data_symbols_per_s": world * F * d / (ms_step * 1e-3),
    }
    if args.e2e_frames > 0:
        line["e2e"] = run_e2e(args, cfg, x, s0, d, world)
    if not args.no_stages and world == 1 and cfg_name != "C4":
        try:
            line["stages"] = run_stages(args, cfg, x, s0, d)
        except Exception as exc:  # noqa: BLE001
            line["stages"] = {"error": repr(exc)[:300]}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = (cpu_reference_numpy_baseline(cfg_name, rx_host[:4], budget_s=args.cpu_seconds)
                                or cpu_port_baseline(cfg_name, rx_host[:4], budget_s=args.cpu_seconds))
    return line


def run_e2e(args, cfg, x_dev, s0, d, world):
    """Same metric through the public API from pinned host memory: every step
    streams its frames H2D (chunked, overlapped with the fused kernel and the
    D2H of the bits via frames.StreamingReceiver) and reads the bits back."""
    import torch

    from paper_1901_07499_b200 import frames

    Fe = min(args.e2e_frames, x_dev.shape[0])
    host = torch.empty((Fe,) + tuple(x_dev.shape[1:]), dtype=torch.complex64, pin_memory=True)
    host.copy_(x_dev[:Fe].cpu())
    bits_host = torch.empty((Fe, d * cfg.fft_len * cfg.bits_per_qam_symbol), dtype=torch.uint8, pin_memory=True)
    rx = frames.StreamingReceiver(cfg, min(args.e2e_chunk, Fe), d, symbol0_offset=s0,
                                  samples_per_row=x_dev.shape[2])
    for _ in range(args.warmup):
        rx.run(host, bits_host)
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        rx.run(host, bits_host)
    torch.cuda.synchronize()
    ms = allreduce_max(world, (time.perf_counter() - t0) * 1e3 / args.steps)
    h2d = int(Fe * cfg.n_antennas * (1 + d) * cfg.fft_len * 8)
    link = pcie_h2d_gbs(host)
    return {"value": world * Fe * (1 + d) / (ms * 1e-3), "unit": "symbols/s",
            "bound": {"kind": "pcie_h2d", "achieved_gbs": h2d / (ms * 1e-3) / 1e9, "peak_gbs": link,
                      "frac": h2d / (ms * 1e-3) / 1e9 / link,
                      "peak_source": "plain pinned->device copy_ of the same host buffer, best of 5, CUDA events"},
            "h2d_bytes_per_step": int(Fe * cfg.n_antennas * (1 + d) * cfg.fft_len * 8),
            "d2h_bytes_per_step": int(bits_host.numel()),
            "frames_per_step": Fe, "ms_per_step": ms, "chunk_frames": min(args.e2e_chunk, Fe),
            "path": "pinned host cf32 captures -> frames.StreamingReceiver (ofdmrx_stage_symbols strided H2D of the "
                    "FFT windows only, CP never crosses PCIe | fused kernel | D2H bits, on 3 streams) "
                    "-> pinned host bits; host-timed around whole steps (includes sync)"}


def pcie_h2d_gbs(host):
    """Plain contiguous pinned->device copy bandwidth (the e2e ceiling)."""
    import torch

    dst = torch.empty(host.shape, dtype=host.dtype, device="cuda")
    best = 0.0
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(host, non_blocking=True)
        b.record()
        b.synchronize()
        best = max(best, host.numel() * 8 / (a.elapsed_time(b) * 1e-3) / 1e9)
    del dst
    return best


def run_stages(args, cfg, x_dev, s0, d, with_sync=True):
    """Per-stage µs/symbol through the staged kernels (the reference's
    StageTimings split: fft incl. CP drop + shift, ls, mrc, demap), CUDA
    events on F_s frames; plus the fused kernel on the same frames."""
    import torch

    from paper_1901_07499_b200 import device as dv
    from paper_1901_07499_b200 import frames

    Fs = min(args.stage_frames, x_dev.shape[0])
    x = x_dev[:Fs]
    n, m = cfg.n_antennas, cfg.fft_len
    pv = torch.from_numpy(np.ascontiguousarray(
        __import__("paper_1901_07499_b200").make_pilot(m).values, dtype=np.complex64)).cuda()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    res = {}

    def timed(fn, reps=20):
        """GPU time of fn: captured once in a CUDA graph and replayed, so the
        host-side cost of the Python/ctypes call does not leak into
        kernel-only stage timings."""
        out = fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            out = fn()
        g.replay()
        a, b = ev(), ev()
        torch.cuda.synchronize()
        a.record()
        for _ in range(reps):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps * 1e3, out  # µs

    t_fft, Y = timed(lambda: frames.fft_symbols(x, cfg, symbol0_offset=s0, n_data=d))
    Yp, Yd = Y[:, 0].contiguous(), Y[:, 1:].contiguous()
    t_ls, H = timed(lambda: dv.ls(Yp, pv))
    t_mrc, (sh, _w) = timed(lambda: dv.mrc(Yd, H))
    t_dm, _ = timed(lambda: dv.demap(sh.reshape(-1), cfg.qam_order))
    out = frames.allocate_outputs(Fs, n, m, d, cfg.qam_order, x.device)
    t_fused, _ = timed(lambda: frames.receive_frames(x, cfg, symbol0_offset=s0, n_data=d, out=out))
    del Y, Yp, Yd, H
    sync = synth_t = None
    if with_sync:  # auxiliary §8(f) stages must never cost the bench line
        try:
            sync = run_sync_stage(cfg, d, Fs, timed)
        except Exception as exc:  # noqa: BLE001
            sync = {"error": repr(exc)[:300]}
        try:
            synth_t = run_synth_stage(cfg, d, Fs, timed)
        except Exception as exc:  # noqa: BLE001
            synth_t = {"error": repr(exc)[:300]}
    res = {"frames": Fs,
           "fft_us_per_symbol": t_fft / (Fs * (1 + d)),
           "ls_us_per_pilot_symbol": t_ls / Fs,
           "mrc_us_per_data_symbol": t_mrc / (Fs * d),
           "demap_us_per_data_symbol": t_dm / (Fs * d),
           "fused_us_per_symbol": t_fused / (Fs * (1 + d)),
           "note": "staged kernels write every intermediate (Y, H) to HBM; the fused kernel keeps them on chip; "
                   "every stage CUDA-graph captured and replayed 20x between CUDA events (GPU time only)",
           "sync": sync, "synth": synth_t}
    return res


def run_synth_stage(cfg, d, Fs, timed):
    """Device frame synthesizer (synth.synth_frames: device bits, flat
    Rayleigh, 10 dB AWGN, PN preamble) over Fs frames: µs per frame and the
    write bandwidth of the rx it produces."""
    from paper_1901_07499_b200 import synth

    t, out = timed(lambda: synth.synth_frames(cfg, d, Fs, seed=7, snr_db=10.0))
    nbytes = out.rx.numel() * 8
    return {"frames": Fs, "us_per_frame": t / Fs, "rx_write_gbs": nbytes / (t * 1e-6) / 1e9,
            "path": "ofdmrx_synth_frames: bits/gains hash RNG, tx_kernel IFFT+CP, sigpow + channel_kernel"}


def run_sync_stage(cfg, d, Fs, timed):
    """PN detection (sync.detect_frames) over Fs whole captures (PN preamble
    included) of this config: µs per frame and the correlation's complex-MAC
    rate (fp32 FMA-pipe bound: rows x windows x chips MACs)."""
    import torch

    from paper_1901_07499_b200 import sync, synth

    rx, _, _ = synth.synth_batch(cfg, d, range(min(Fs, DISTINCT)), strip_preamble=False)
    base = torch.from_numpy(rx).cuda()
    x = base.repeat((Fs + base.shape[0] - 1) // base.shape[0], 1, 1)[:Fs].contiguous()
    pn = synth.generate_pn_chips()
    t, det = timed(lambda: sync.detect_frames(x, pn))
    ok = bool((det.frame_start == 0).all()) and bool((det.symbol0_offset == pn.size).all())
    rows, wins = Fs * cfg.n_antennas, x.shape[2] - pn.size + 1
    from paper_1901_07499_b200 import frames

    # the whole device pipeline on raw captures: detection -> per-frame timing -> fused receive
    tp, (outp, detp) = timed(lambda: frames.receive_captures(x, cfg, d, pn))
    pipe = {"us_per_frame": tp / Fs, "symbols_per_s": Fs * (1 + d) / (tp * 1e-6),
            "flagged_frames": int((outp.flags != 0).sum()),
            "path": "frames.receive_captures: ofdmrx_detect + ofdmrx_rx_frames_detected, no host round trip"}
    return {"frames": Fs, "samples_per_row": int(x.shape[2]), "us_per_frame": t / Fs, "pipeline": pipe,
            "cmac_per_s": rows * wins * pn.size / (t * 1e-6), "all_offsets_found": ok,
            "path": "ofdmrx_detect: fp32 corr_kernel (FFMA2) + fp64 refine of near-max windows"}


# ---------------------------------------------------------------------------
# C5 sweep: antennas x FFT size, per-stage timing vs the reference CPU path,
# written in the reference bench CSV schema (ofdmrx/bench.py:22-24)
# ---------------------------------------------------------------------------

CSV_HEADER = "fft_len,cp_len,n_antennas,engine,workers,phase,stage,mean_us,std_us,n_symbols"


def run_sweep(args):
    import csv

    import torch

    from paper_1901_07499_b200 import synth
    from paper_1901_07499_b200.waveform import OfdmConfig, default_cp

    torch.cuda.set_device(0)
    ants = [int(a) for a in args.sweep_antennas.split(",")]
    ffts = [int(m) for m in args.sweep_ffts.split(",")]
    qam, d = 16, 10
    ref = reference_importable()
    if ref:
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/ofdmrx_numba_cache")
        from ofdmrx import receiver as rref, waveform as wref
    rows = []
    summary = []
    for m in ffts:
        cp = default_cp(m)
        for n in ants:
            cfg = OfdmConfig(m, cp, n, qam_order=qam)
            rx, _, s0 = synth.synth_batch(cfg, d, range(2), snr_db=10.0)
            F = max(2, min(4096, (1 << 26) // (n * m * (1 + d))))
            x = torch.from_numpy(rx).cuda().repeat((F + 1) // 2, 1, 1)[:F].contiguous()
            st = run_stages(argparse.Namespace(stage_frames=F), cfg, x, s0, d, with_sync=False)
            g = [("estimation", "fft", st["fft_us_per_symbol"], F),
                 ("estimation", "ls", st["ls_us_per_pilot_symbol"], F),
                 ("demodulation", "fft", st["fft_us_per_symbol"], F * d),
                 ("demodulation", "mrc", st["mrc_us_per_data_symbol"] + st["demap_us_per_data_symbol"], F * d),
                 ("demodulation", "fused", st["fused_us_per_symbol"], F * (1 + d))]
            for phase, stage, us, ns in g:
                rows.append((m, cp, n, "b200", 1, phase, stage, us, 0.0, ns))
            cpu = {}
            if ref:
                rcfg = wref.OfdmConfig(m, cp, n, qam_order=qam)
                pilot = wref.make_pilot(m)
                eng = rref.SequentialEngine()
                x0 = rx[0].astype(np.complex128)
                sym = lambda k: x0[:, s0 + k * (m + cp): s0 + (k + 1) * (m + cp)]  # noqa: E731

                def best(fn, reps=3):
                    ts = []
                    for _ in range(reps):
                        t0 = time.perf_counter()
                        out = fn()
                        ts.append(time.perf_counter() - t0)
                    return min(ts) * 1e6, out

                best(lambda: rref.to_freq(rref.cp_drop(sym(0), rcfg), eng), 1)  # JIT
                t_fft, Y0 = best(lambda: rref.to_freq(rref.cp_drop(sym(0), rcfg), eng))
                t_ls, est = best(lambda: rref.ls_estimate(Y0, pilot, eng))
                Y1 = rref.to_freq(rref.cp_drop(sym(1), rcfg), eng)

                def mrc_demap():
                    c = rref.mrc_combine(Y1, est, eng)
                    c.bits = wref.qam_demap(c.equalized, qam)
                    return c

                t_mrc, _ = best(mrc_demap)
                cpu = {"fft": t_fft, "ls": t_ls, "mrc": t_mrc}
                for phase, stage, us in (("estimation", "fft", t_fft), ("estimation", "ls", t_ls),
                                         ("demodulation", "fft", t_fft), ("demodulation", "mrc", t_mrc)):
                    rows.append((m, cp, n, "sequential", 1, phase, stage, us, 0.0, 1))
            summary.append({"fft_len": m, "n_antennas": n, "frames": F,
                            "b200_us_per_symbol": {"fft": st["fft_us_per_symbol"], "ls": st["ls_us_per_pilot_symbol"],
                                                   "mrc+demap": st["mrc_us_per_data_symbol"] + st["demap_us_per_data_symbol"],
                                                   "fused": st["fused_us_per_symbol"]},
                            "cpu_us_per_symbol": cpu})
            del x
            torch.cuda.empty_cache()
            print(json.dumps(summary[-1]), file=sys.stderr, flush=True)
    with open(args.sweep_csv, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(CSV_HEADER.split(","))
        for r in rows:
            w.writerow(r[:7] + (repr(float(r[7])), repr(float(r[8])), r[9]))
    return {"metric": "C5 sweep: per-stage µs/symbol, b200 vs reference CPU", "csv": args.sweep_csv,
            "configs": len(summary), "reference_cpu": bool(ref),
            "cpu_cores_used": 1, "engine_cpu": "reference SequentialEngine (numba backend)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS))
    ap.add_argument("--frames", type=int, default=0, help="frames per GPU (default per config)")
    ap.add_argument("--e2e-frames", type=int, default=256)
    ap.add_argument("--e2e-chunk", type=int, default=32)
    ap.add_argument("--stage-frames", type=int, default=64)
    ap.add_argument("--no-stages", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="gather", choices=["gather", "allreduce", "peer"],
                    help="C4 antenna-sharded exchange: NCCL all-gather / all-reduce, or fused peer-memory stores")
    ap.add_argument("--sweep", action="store_true", help="C5: antennas x FFT per-stage sweep -> CSV")
    ap.add_argument("--sweep-antennas", default="1,2,4,8,16,32,64,128")
    ap.add_argument("--sweep-ffts", default="64,128,256,512,1024,2048,4096")
    ap.add_argument("--sweep-csv", default="gpurun_out/sweep.csv")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.sweep:
        print(json.dumps(run_sweep(args)), flush=True)
        return
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        line = run_reference_arm(args, args.config, world, rank)
        if line is not None:
            line["n_gpus"] = world
            print(json.dumps(line), flush=True)
        return
    world, rank, local = dist_setup(args.gpus)
    line = run_b200(args, args.config, world, rank, local)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
