#!/bin/bash
# round-end evidence in one call: gpu_r2_final.sh (smoke, GPU tests, C3 ncu + traffic, bench, launches,
# reference arm), the C4 / C2 / C1 bench lines, and the full sweep
bash scripts/gpu_r2_final.sh
bash scripts/gpu_r2_lines.sh
timeout 1500 python bench.py --sweep --sweep-csv gpurun_out/final/sweep_r02.csv > gpurun_out/final/sweep_r02.out 2> gpurun_out/final/sweep_r02.err; echo "sweep rc=$?"; cat gpurun_out/final/sweep_r02.out
