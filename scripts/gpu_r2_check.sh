#!/bin/bash
# round-2 quick GPU check: new kernel parity + batch invariance + C3/C4 timing
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu -k "balanced or invariance or golden" 2>&1 | tail -30
for a in "C3 1024" "C3 64" "C3 8" "C4 64" "C4 148" "C2 1000" "C1 65536"; do timeout 120 python scripts/fused_quick.py $a; done
