"""The frame-sharded bench path with world size 2 on one GPU (SURVEY.md
§8(e)): `bench.py` under torchrun, gloo for the rank plumbing, both ranks on
cuda:0 (OFDMRX_SAME_DEVICE=1; a code-path test, not a measurement).  Each
rank receives its own distinct frames; every rank's benched bits must equal
the CPU oracle's, and the line must carry per-rank clocks and checks, the
communicator description and a CPU baseline."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_frame_sharded_bench_two_ranks():
    env = dict(os.environ, OFDMRX_DIST_BACKEND="gloo", OFDMRX_SAME_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--frames", "48", "--e2e-frames", "0", "--no-stages",
           "--sustained-steps", "0", "--oracle-frames", "4", "--cpu-seconds", "1", "--no-latency"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "weak"
    assert line["config"]["global_frames"] == 96
    checks = line["check_per_rank"]
    assert [c["rank"] for c in checks] == [0, 1]
    for c in checks:
        assert c["bits_vs_oracle"] == "exact" and c["oracle_ok"], c
        assert c["flagged_frames"] == 0
    assert len(line["clocks_per_rank"]) == 2
    assert line["comm"]["world_size"] == 2 and line["comm"]["data_path_collective"].startswith("none")
    assert line["cpu_baseline"]["value"] > 0
