#!/bin/bash
# refresh after a kernel change: C4/C2/C1 bench lines, the full sweep, and the
# C3 shared-store excess wavefronts by SASS line
mkdir -p gpurun_out/final
bash scripts/gpu_r2_lines.sh
timeout 1500 python bench.py --sweep --sweep-csv gpurun_out/final/sweep_r02.csv > gpurun_out/final/sweep_r02.out 2> gpurun_out/final/sweep_r02.err; echo "sweep rc=$?"
rm -f /tmp/prof_c3h.ncu-rep
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:"rx_balanced" -s 3 -c 1 -o /tmp/prof_c3h python scripts/fused_quick.py C3 1024 3 > /dev/null 2>&1
python scripts/ncu_col.py /tmp/prof_c3h.ncu-rep 'L1 Wavefronts Shared Excessive' 30 > gpurun_out/final/c3_smem_excess.txt 2>&1
python scripts/ncu_col.py /tmp/prof_c3h.ncu-rep '?' > gpurun_out/final/c3_cols.txt 2>&1
