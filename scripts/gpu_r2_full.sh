#!/bin/bash
# round-2 full check: GPU tests, smoke, per-config timing, default bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
for a in "C3 1024" "C3 64" "C3 1" "C4 64" "C4 148" "C2 1000" "C1 65536"; do timeout 120 python scripts/fused_quick.py $a; done 2>&1 | tee gpurun_out/quick.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json | head -c 3000
