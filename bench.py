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
    "C4": (256, 2048, 256, 64, 10, 296),
}
METRIC = "OFDM symbols/s & per-stage µs/symbol at 64 ant × FFT 1024, 1/2/4/8 B200"
DISTINCT = 16  # distinct synthetic frames, tiled on the device


def frame_bytes(n, m, qam, d):
    """Algorithmic HBM bytes per frame: rx samples of the
    1+D symbols without CP, H written once, s_hat, bits as u8."""
    b = int(math.log2(qam))
    return 8 * n * m * (1 + d) + 8 * n * m + 8 * m * d + b * m * d


KERNEL_SOURCES = ("rx_balanced.cu", "rx_fused.cu", "rx_latency.cu", "ofdmrx_fft.cuh", "ofdmrx_internal.h", "capi.cu")


def kernel_source_hash():
    """Hash of the receive kernels' sources: profiles/traffic_<cfg>.json
    records it, so a capture taken on another kernel version reads as stale."""
    import hashlib

    h = hashlib.sha256()
    for name in KERNEL_SOURCES:
        with open(os.path.join(ROOT, "paper_1901_07499_b200", "csrc", name), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


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
            # NCCL's init log (ranks, transports) into a file, not stdout: the
            # JSON line stays the only stdout line; comm_info() quotes it
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", f"/tmp/ofdmrx_nccl.{rank}.%p.log")
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

        chunk = F // 4 if args.exchange == "scatter" and F % 4 == 0 and (F // 4) % world == 0 else None
        sharded = sharding.AntennaShardedReceiver(cfg, d, symbol0_offset=s0, mode=args.exchange, chunk_frames=chunk)
        x = x[:, sharded.ant_lo:sharded.ant_hi].contiguous()

    own = slice(None)
    lo, hi = 0, min(F, DISTINCT)
    if sharded is not None and args.exchange in ("peer", "scatter"):  # each rank finishes its F/world frames
        own = torch.tensor(sharded.owned_frames(F) if args.exchange == "scatter" else
                           list(range(rank * (F // world), (rank + 1) * (F // world))), device=dev)
        lo = int(own[0])
        hi = lo + min(DISTINCT, (sharded.chunk_frames or F) // world)

    def step():
        if sharded is not None:
            s_hat, w, bits, fl, _ = sharded.receive(x)
            out.bits[own] = bits
            out.flags[own] = fl
        else:
            frames.receive_frames(x, cfg, symbol0_offset=s0, n_data=d, out=out)

    # correctness spot-check of the benchmarked configuration (bits vs truth)
    step()
    torch.cuda.synchronize()
    idx = np.arange(lo, hi)
    ber = float((out.bits[lo:hi].cpu().numpy() != bits_truth[idx % len(bits_truth)]).mean())
    flags_bad = int((out.flags != 0).sum())
    torch.cuda.synchronize()
    if sharded is not None and args.oracle_frames:  # untimed: s_hat / weights of the owned frames for the check
        s_hat, w, _, _, _ = sharded.receive(x)
        out.s_hat[own] = s_hat
        out.weights[own] = w
        torch.cuda.synchronize()
    oracle_check = (check_vs_oracle(cfg_name, rx_host, s0, out, lo, hi, args.oracle_frames, check_h=sharded is None)
                    if args.oracle_frames else None)

    # one step = one receive_frames call; unless --eager, the call is captured
    # once in a CUDA graph and replayed, so host-side Python / enqueue jitter
    # cannot starve short steps (C2: 0.13 ms) inside the device-timed regions
    launch_mode = "eager"
    if sharded is None and not args.eager:
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        with torch.cuda.stream(cap):
            step()
        stream.wait_stream(cap)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        step = graph.replay  # noqa: F811
        launch_mode = "cuda_graph"
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
        h1 = time.time()
        sustained = None
        if args.sustained_steps > 0:
            # a second, longer timed region right after the burst: the board's
            # power cap engages after ~100 ms of back-to-back launches
            barrier(world)
            torch.cuda.synchronize()
            s_start, s_stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h2 = time.time()
            s_start.record(stream)
            for _ in range(args.sustained_steps):
                step()
            s_stop.record(stream)
            torch.cuda.synchronize()
            h3 = time.time()
            sustained = (s_start.elapsed_time(s_stop), h2, h3)
        time.sleep(0.25)  # let nvidia-smi deliver the samples it took inside the windows
        barrier(world)
    clocks.mark(h0, h1)
    burst_clocks = clocks.summary()
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
        fresh = tj.get("kernel_source_hash") == kernel_source_hash()
        if "dram_bytes_per_frame" in tj and fresh:
            # same units as `achieved`: the ncu-measured DRAM bytes of one launch
            # of this size over the live kernel time (only when the capture was
            # taken on the kernel sources being measured)
            traffic = tj["dram_bytes_per_frame"] * F / (kernel_ms * 1e-3) / 1e9
            traffic_detail = {"dram_bytes_per_launch": int(tj["dram_bytes_per_frame"] * F),
                              "algorithmic_bytes_per_launch": int(frame_bytes(n // (world if sharded is not None else 1),
                                                                              m, qam, d) * F),
                              "source": tj.get("source"), "kernel_source_hash": tj.get("kernel_source_hash")}
        elif "dram_bytes_per_frame" in tj:
            traffic_detail = {"stale": f"{tj.get('source')} was captured on other kernel sources "
                                       f"({tj.get('kernel_source_hash')} != {kernel_source_hash()})"}

    line = {
        "metric": METRIC, "value": value, "unit": "symbols/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32 (cf32 I/O)",
        "data": "synthetic: reference TX (PN|pilot|data, Gray QAM) through flat Rayleigh at 10 dB; "
                f"{DISTINCT} distinct frames tiled on device",
        "config": {"workload": f"{cfg_name}: {n} ant x FFT {m} (CP {cp}), {qam}-QAM, 1 pilot + {d} data symbols/frame",
                   "frames_per_gpu": F, "global_frames": F if sharded is not None else F * world, "parallelism": (f"antenna-sharded x{world} ({args.exchange} exchange of MRC partials"
                                   f"{' over peer memory, no NCCL' if args.exchange == 'peer' else ' over ' + _dist_backend_name()})"
                                   if sharded is not None else f"frame-sharded x{world}"),
                   "input_bytes_per_gpu": int(x.numel() * 8),
                   "l2": f"inputs {x.numel() * 8 / 1e9:.2f} GB/GPU > L2 (126 MB), no flush needed"
                   if x.numel() * 8 > 126e6 else "inputs smaller than L2",
                   "launch": ("one receive_frames call per step, captured once in a CUDA graph and replayed"
                              if launch_mode == "cuda_graph" else "one receive / exchange call per step, eager")},
        "gpu_launches": args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_detail": traffic_detail, "peak_source": peak_kind,
                     "bytes_per_frame": bpf, "kernel_ms": kernel_ms},
        "clocks": burst_clocks,
        "check": {"ber_vs_tx": ber, "flagged_frames": flags_bad, **(oracle_check or {})},
        "data_symbols_per_s": world * F * d / (ms_step * 1e-3),
    }
    if sustained is not None:
        clocks.mark(sustained[1], sustained[2])
        s_ms = allreduce_max(world, sustained[0] / args.sustained_steps)
        s_val = (1 if sharded is not None else world) * F * (1 + d) / (s_ms * 1e-3)
        line["sustained"] = {"steps": args.sustained_steps, "ms_per_step": s_ms, "value": s_val,
                             "roofline_frac": bpf * F / (s_ms * 1e-3) / 1e9 / peak, "clocks": clocks.summary(),
                             "note": "same launches back to back for ~{:.0f} ms right after the burst; the headline "
                                     "value is the {}-step burst".format(sustained[0], args.steps)}
    if world > 1:
        line["clocks_per_rank"] = gather_objects(world, {"rank": rank, "device": local, **burst_clocks})
        line["check_per_rank"] = gather_objects(world, {"rank": rank, "frames": [lo, hi], "ber_vs_tx": ber,
                                                        "flagged_frames": flags_bad, **(oracle_check or {})})
        line["comm"] = comm_info(world, "none (frame sharding)" if sharded is None else
                                  f"{args.exchange} exchange of the MRC partial sums")
    if args.e2e_frames > 0:
        line["e2e"] = run_e2e(args, cfg, x, s0, d, world)
    if not args.no_stages and world == 1 and cfg_name != "C4":
        try:
            line["stages"] = run_stages(args, cfg, x, s0, d)
        except Exception as exc:  # noqa: BLE001
            line["stages"] = {"error": repr(exc)[:300]}
    if world == 1 and args.sweep_cells and cfg_name != "C4":
        try:  # compact C5 sweep in the default line (full sweep: --sweep)
            cells = [tuple(int(v) for v in c.split("x")) for c in args.sweep_cells.split(",")]
            line["sweep"] = sweep_cells(cells, reps=1)[1]
        except Exception as exc:  # noqa: BLE001
            line["sweep"] = {"error": repr(exc)[:300]}
    if world == 1 and args.latency and cfg_name != "C4":
        try:
            line["latency"] = run_latency(args)
        except Exception as exc:  # noqa: BLE001
            line["latency"] = {"error": repr(exc)[:300]}
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = (cpu_reference_numpy_baseline(cfg_name, rx_host[:4], budget_s=args.cpu_seconds)
                                or cpu_port_baseline(cfg_name, rx_host[:4], budget_s=args.cpu_seconds))
    return line


def check_vs_oracle(cfg_name, rx_host, s0, out, lo, hi, max_frames, check_h=True):
    """Parity of the benchmarked launch: the distinct frames' bits against the
    CPU oracle (oracle/ofdm_oracle.py, the numpy restatement of the reference
    pinned to reference-generated golden vectors), s_hat / H / weights within
    north_star's 1e-4.  A checker outside the timed region, never measured."""
    from oracle import ofdm_oracle as orc

    n, m, cp, qam, d, _ = CONFIGS[cfg_name]
    k = min(hi - lo, max_frames)
    mism, worst = 0, {"s_hat": 0.0, "H": 0.0, "weights": 0.0}
    bits_dev = out.bits[lo:lo + k].cpu().numpy()
    sh_dev = out.s_hat[lo:lo + k].cpu().numpy()
    w_dev = out.weights[lo:lo + k].cpu().numpy()
    h_dev = out.H[lo:lo + k].cpu().numpy() if check_h and getattr(out, "H", None) is not None else None

    def rel(a, b):
        return float(np.linalg.norm(np.asarray(a, np.complex128) - b) / max(np.linalg.norm(b), 1e-300))

    for i in range(k):
        H, s_hat, w, bits = orc.receive_frame(rx_host[(lo + i) % len(rx_host)].astype(np.complex128), s0, m, cp, d, qam)
        mism += int((bits_dev[i] != bits).sum())
        worst["s_hat"] = max(worst["s_hat"], rel(sh_dev[i], s_hat))
        worst["weights"] = max(worst["weights"], rel(w_dev[i], w))
        if h_dev is not None:
            worst["H"] = max(worst["H"], rel(h_dev[i], H))
    return {"bits_vs_oracle": "exact" if mism == 0 else f"{mism} bits differ",
            "oracle_frames": k, "oracle_bits": int(k * bits_dev.shape[1]),
            "max_rel_err": worst, "rel_tol": 1e-4,
            "oracle_ok": mism == 0 and max(worst.values()) < 1e-4,
            "checker": "oracle/ofdm_oracle.py receive_frame (fp64 numpy restatement of the reference path), "
                       "outside the timed region"}


def gather_objects(world, obj):
    import torch.distributed as dist

    objs = [None] * world
    dist.all_gather_object(objs, obj)
    return objs


def comm_info(world, data_path):
    import torch
    import torch.distributed as dist

    info = {"backend": dist.get_backend(), "world_size": dist.get_world_size()}
    if info["backend"] == "nccl":
        v = torch.cuda.nccl.version()
        info["nccl_version"] = ".".join(str(x) for x in v) if isinstance(v, tuple) else str(v)
    info["data_path_collective"] = data_path
    import glob

    rank = dist.get_rank()
    for path in sorted(glob.glob(f"/tmp/ofdmrx_nccl.{rank}.{os.getpid()}.log")):
        with open(path, errors="replace") as fh:
            keep = [ln.strip()[-160:] for ln in fh if "nranks" in ln or "Init COMPLETE" in ln or "NVLS" in ln]
        info["nccl_init_log"] = keep[:4]
    return info


def _dist_backend_name():
    import torch.distributed as dist

    return (dist.get_backend().upper() if dist.is_available() and dist.is_initialized() else "NCCL")


def run_latency(args):
    """The paper's regime: ONE frame, pinned host capture
    -> device -> fused receive -> bits back on the host, per call, with the
    latency plan (OFDMRX_OPT_LATENCY: the frame spread over a whole
    thread-block cluster).  Per config (C1, C3): the public-API call's wall
    time (median / p99 over `latency_reps` calls: H2D + kernel + D2H + sync),
    the same sequence replayed as a CUDA graph (no Python), the kernel alone
    (graph-replayed, CUDA events; also with the default throughput plan) and
    its per-stage split from the kernel's own stage attribution
    (ofdmrx_rx_frames_profiled), per OFDM symbol."""
    import torch

    from paper_1901_07499_b200 import frames

    def graph_time_us(fn, reps=50):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(3):
                fn()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps * 1e3, g

    res = {}
    for name in ("C1", "C3"):
        n, m, cp, qam, d, _ = CONFIGS[name]
        cfg, rx_host, _, s0 = make_inputs(name)
        host = torch.from_numpy(rx_host[:1]).pin_memory()
        dev_x = torch.empty(host.shape, dtype=host.dtype, device="cuda")
        dev_x.copy_(host)
        out = frames.allocate_outputs(1, n, m, d, qam, dev_x.device)
        bits_host = torch.empty(out.bits.shape, dtype=torch.uint8, pin_memory=True)

        def kernel(lat=True):
            frames.receive_frames(dev_x, cfg, symbol0_offset=s0, n_data=d, out=out, latency=lat)

        def seq():
            dev_x.copy_(host, non_blocking=True)
            kernel()
            bits_host.copy_(out.bits, non_blocking=True)

        def call():
            seq()
            torch.cuda.current_stream().synchronize()

        for _ in range(20):
            call()
        ts = []
        for _ in range(args.latency_reps):
            t0 = time.perf_counter()
            call()
            ts.append(time.perf_counter() - t0)
        ts.sort()
        _, g = graph_time_us(seq, reps=1)
        gts = []
        for _ in range(args.latency_reps):
            t0 = time.perf_counter()
            g.replay()
            torch.cuda.current_stream().synchronize()
            gts.append(time.perf_counter() - t0)
        gts.sort()
        k_us, _ = graph_time_us(kernel)
        k_tp_us, _ = graph_time_us(lambda: kernel(False))
        h2d_us, _ = graph_time_us(lambda: dev_x.copy_(host, non_blocking=True))
        prof = frames.receive_frames(dev_x, cfg, symbol0_offset=s0, n_data=d, profile=True, latency=True)
        torch.cuda.synchronize()
        shares = prof.stage_shares()
        sym = 1 + d
        med, p99 = ts[len(ts) // 2] * 1e6, ts[min(len(ts) - 1, int(len(ts) * 0.99))] * 1e6
        gmed = gts[len(gts) // 2] * 1e6
        res[name] = {
            "frames": 1, "symbols_per_frame": sym, "plan": "latency (OFDMRX_OPT_LATENCY)",
            "h2d_bytes": int(host.numel() * 8), "d2h_bytes": int(bits_host.numel()),
            "api_us_per_frame": {"median": med, "p99": p99}, "api_us_per_symbol": med / sym,
            "graph_us_per_frame": gmed, "graph_us_per_symbol": gmed / sym,
            "h2d_alone_us": h2d_us,
            "kernel_us_per_frame": k_us, "kernel_us_per_symbol": k_us / sym,
            "kernel_us_per_frame_throughput_plan": k_tp_us,
            "kernel_stage_us_per_symbol": {
                "fft": k_us * (shares[0] + shares[2]) / sym, "ls": k_us * shares[1],
                "mrc": k_us * shares[3] / max(d, 1), "combine_demap": k_us * shares[4] / max(d, 1)},
            "path": "pinned host [N, S] capture -> copy_ H2D -> frames.receive_frames(latency=True) (one fused "
                    "launch) -> bits D2H -> stream sync; host perf_counter around each call; kernel times are "
                    "CUDA-graph replays between CUDA events"}
        del dev_x, out
    return res


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
            "d2h": "bits only (PipelineResult.bits); s_hat / H / weights stay in HBM",
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

def sweep_cells(cells, with_cpu=True, reps=3, max_frames=4096):
    """C5 sweep cells (N antennas, FFT M): per-stage timing on the B200 next
    to the reference CPU path, in the reference bench CSV schema
    (ofdmrx/bench.py:19-25; paper_1901_07499_b200.benchcsv).

    Per cell, on the same reference-built slots of one frame:
      engine "sequential"  the unmodified reference run_ring_pipeline with its
                           SequentialEngine (numba backend), records made by
                           the reference's own _records_for_engine;
      engine "b200"        the mirror's run_ring_pipeline (one fused launch,
                           StageTimings with the reference's meaning: the
                           paper's per-symbol regime incl. H2D/D2H);
      engine "b200_batched" the staged kernels over F frames resident in HBM
                           (GPU time per symbol: fft, ls, mrc = MRC + demap).
    Plus, per cell, the fused kernel's time at batch F and its HBM roofline
    fraction.  Returns (records, summary)."""
    import torch

    from paper_1901_07499_b200 import benchcsv, synth
    from paper_1901_07499_b200 import receiver as mr
    from paper_1901_07499_b200.waveform import OfdmConfig, default_cp

    qam, d = 16, 10
    ref = with_cpu and reference_importable()
    if ref:
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/ofdmrx_numba_cache")
        from ofdmrx import bench as bref, receiver as rref, waveform as wref
        from ofdmrx.sync import DetectionResult
    peak, _ = load_peaks()
    records, summary = [], []
    for n, m in cells:
        cp = default_cp(m)
        cfg = OfdmConfig(m, cp, n, qam_order=qam)
        rx, _, s0 = synth.synth_batch(cfg, d, range(2), snr_db=10.0)
        # enough frames to fill the GPU (>= 2 CTAs per SM), at most ~4 GB of input
        F = max(296, min(max_frames, (1 << 29) // (n * m * (1 + d))))
        F = min(F, max(2, (1 << 32) // (8 * n * m * (1 + d))))
        x = torch.from_numpy(rx).cuda().repeat((F + 1) // 2, 1, 1)[:F].contiguous()
        st = run_stages(argparse.Namespace(stage_frames=F), cfg, x, s0, d, with_sync=False)
        bpf = frame_bytes(n, m, qam, d)
        fused_frame_us = st["fused_us_per_symbol"] * (1 + d)
        frac = bpf / (fused_frame_us * 1e-6) / 1e9 / peak
        for phase, stage, us, ns in (("estimation", "fft", st["fft_us_per_symbol"], F),
                                     ("estimation", "ls", st["ls_us_per_pilot_symbol"], F),
                                     ("demodulation", "fft", st["fft_us_per_symbol"], F * d),
                                     ("demodulation", "mrc",
                                      st["mrc_us_per_data_symbol"] + st["demap_us_per_data_symbol"], F * d)):
            records.append(benchcsv.BenchRecord(m, cp, n, "b200_batched", 1, phase, stage, us, 0.0, ns))
        cell = {"fft_len": m, "n_antennas": n, "frames": F, "fused_us_per_symbol": st["fused_us_per_symbol"],
                "roofline_frac": frac, "bytes_per_frame": bpf,
                "b200_batched_us_per_symbol": {"fft": st["fft_us_per_symbol"], "ls": st["ls_us_per_pilot_symbol"],
                                               "mrc+demap": st["mrc_us_per_data_symbol"]
                                               + st["demap_us_per_data_symbol"]}}
        del x
        torch.cuda.empty_cache()
        if ref:
            rcfg = wref.OfdmConfig(m, cp, n, qam_order=qam)
            pilot = wref.make_pilot(m)

            class _Cap:
                def __init__(self, s):
                    self.streams = s

            slots = rref.extract_slots(_Cap(rx[0].astype(np.complex128)), DetectionResult(True, 0, s0, 1.0, ()),
                                       rcfg, 1 + d)
            with rref.make_engine(rref.EngineKind("sequential")) as eng:
                warm = rref.run_ring_pipeline(slots, rcfg, eng, pilot=pilot)
                timed = []
                for _ in range(reps):
                    res = rref.run_ring_pipeline(slots, rcfg, eng, pilot=pilot)
                    timed.extend(res.timings)
            records.extend(benchcsv.BenchRecord(**vars(r)) for r in
                           bref._records_for_engine(rcfg, "sequential", 1, timed, warm.timings))
            eng = mr.make_engine(mr.EngineKind("b200"))
            warm_b = mr.run_ring_pipeline(slots, rcfg, eng, pilot=pilot)
            timed_b = []
            same = np.array_equal(warm_b.bits, warm.bits)
            for _ in range(reps):
                res_b = mr.run_ring_pipeline(slots, rcfg, eng, pilot=pilot)
                same = same and np.array_equal(res_b.bits, warm.bits)
                timed_b.extend(res_b.timings)
            records.extend(benchcsv.records_for_engine(rcfg, "b200", 1, timed_b, warm_b.timings))
            cell["bits_equal_reference"] = bool(same)
            per = lambda ts: sum(t.total_s for t in ts) / len(ts) * 1e6  # noqa: E731
            cell["pipeline_us_per_symbol"] = {"reference_sequential": per(timed), "b200": per(timed_b)}
        summary.append(cell)
        print(json.dumps(cell), file=sys.stderr, flush=True)
    return records, summary


def run_sweep(args):
    import torch

    from paper_1901_07499_b200 import benchcsv

    torch.cuda.set_device(0)
    ants = [int(a) for a in args.sweep_antennas.split(",")]
    ffts = [int(m) for m in args.sweep_ffts.split(",")]
    records, summary = sweep_cells([(n, m) for m in ffts for n in ants])
    benchcsv.write_bench_csv(records, args.sweep_csv)
    with open(os.path.splitext(args.sweep_csv)[0] + ".json", "w") as fh:
        json.dump(summary, fh, indent=1)
    return {"metric": "C5 sweep: per-stage µs/symbol, b200 vs reference CPU", "csv": args.sweep_csv,
            "configs": len(summary), "reference_cpu": reference_importable(),
            "cpu_cores_used": 1, "engine_cpu": "reference SequentialEngine (numba backend)",
            "min_roofline_frac": min(c["roofline_frac"] for c in summary),
            "all_bits_equal_reference": all(c.get("bits_equal_reference", True) for c in summary)}


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
    ap.add_argument("--sustained-steps", type=int, default=100,
                    help="second timed region of back-to-back steps (power-cap regime); 0 = off")
    ap.add_argument("--oracle-frames", type=int, default=16,
                    help="distinct frames of the benched launch checked against the CPU oracle; 0 = off")
    ap.add_argument("--eager", action="store_true",
                    help="call receive_frames eagerly in the timed loops instead of replaying its CUDA graph")
    ap.add_argument("--no-latency", dest="latency", action="store_false",
                    help="skip the single-frame latency section (C1 and C3)")
    ap.add_argument("--latency-reps", type=int, default=200)
    ap.add_argument("--exchange", default="scatter", choices=["gather", "allreduce", "scatter", "peer"],
                    help="C4 antenna-sharded exchange: NCCL all-gather / all-reduce / all-to-all (reduce-scatter shaped, "
                         "chunk-overlapped), or fused peer-memory stores")
    ap.add_argument("--sweep", action="store_true", help="C5: antennas x FFT per-stage sweep -> CSV")
    ap.add_argument("--sweep-antennas", default="1,2,4,8,16,32,64,128")
    ap.add_argument("--sweep-ffts", default="64,128,256,512,1024,2048,4096")
    ap.add_argument("--sweep-csv", default="gpurun_out/sweep.csv")
    ap.add_argument("--sweep-cells", default="8x64,16x256,64x1024,128x4096",
                    help="compact C5 sweep (NxM cells) in the default line; '' = off")
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
