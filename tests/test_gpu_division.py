"""The branch-free division fast path of the receive epilogue (ofdmrx_fft.cuh:
recip / div_fast under the in_range guards of finish_points_qb) is
bit-identical to IEEE division -- numpy's float32 quotient in
s_hat = num / den (receiver.py:225-236) and s_hat / scale (waveform.py:179-197).

Compiles tests/cuda/div_check.cu with the library's nvcc flags and runs its
sweeps on the GPU: every divisor mantissa at 12 exponents, the demap
divisions against the three QAM scales, and random bit patterns (~2^27
quotients through the fast path)."""
import json
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_division_fast_path_bit_identical(tmp_path):
    exe = tmp_path / "div_check"
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                    "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "paper_1901_07499_b200", "csrc"),
                    "-o", str(exe), os.path.join(ROOT, "tests", "cuda", "div_check.cu")],
                   check=True, capture_output=True, timeout=300)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["mismatches"] == 0, res
    assert res["fast_path"] > 100_000_000, res
