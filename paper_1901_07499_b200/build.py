"""Build libofdmrx_b200.so in-tree with nvcc for sm_100a.

    python -m paper_1901_07499_b200.build [--verbose]

The shared library is the product: the Python package loads it with ctypes
and fails loudly when it is missing.  It links cudart statically, so loading
it needs only the NVIDIA driver at call time (import works without a GPU).
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libofdmrx_b200.so")
SOURCES = ["capi.cu", "rx_fused.cu", "rx_balanced.cu", "rx_latency.cu", "rx_staged.cu", "sync.cu", "synth.cu", "peer.cu"]
HEADERS = ["ofdmrx_fft.cuh", "ofdmrx_internal.h", "ofdmrx_twiddles.inc", "gen_twiddles.py",
           os.path.join("..", "..", "include", "ofdmrx_b200.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-cudart", "static"]


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = SOURCES + HEADERS + [os.path.basename(__file__)]
    return any(os.path.getmtime(os.path.join(CSRC if d != os.path.basename(__file__) else HERE, d)) > t
               for d in deps)


def build_variant(name, defines, sources=None):
    """Experiment build: libofdmrx_b200_<name>.so under build/variants with
    extra -D flags (A/B timing via OFDMRX_VARIANT_LIB in scripts/fused_quick.py; never the product)."""
    outdir = os.path.join(HERE, "..", "build", "variants")
    os.makedirs(outdir, exist_ok=True)
    lib = os.path.abspath(os.path.join(outdir, f"libofdmrx_b200_{name}.so"))
    objs, procs = [], []
    for src in sources or SOURCES:
        obj = os.path.join(outdir, f"{name}_{src.replace('.cu', '.o')}")
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode:
            sys.stderr.write(out)
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")
    subprocess.run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", lib, *objs], check=True)
    for o in objs:
        os.remove(o)
    return lib


def build(force=False, verbose=False):
    sys.path.insert(0, CSRC)
    try:
        import gen_twiddles
        gen_twiddles.main()
    finally:
        sys.path.pop(0)
    if not force and not _stale():
        return LIB
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, "-dc" if False else "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    for cmd, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode:
            sys.stderr.write(out)
        if p.returncode:
            raise RuntimeError(f"nvcc failed ({p.returncode}): {' '.join(cmd)}")
    tmp = LIB + ".tmp"
    link = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    subprocess.run(link, check=True)
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        print(build_variant(sys.argv[i + 1], sys.argv[i + 2:]))
    else:
        print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
