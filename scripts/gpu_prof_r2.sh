#!/bin/bash
# ncu captures of the balanced kernel: C4 (148 frames) and C3 (1024 frames)
mkdir -p gpurun_out
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:rx_balanced -s 3 -c 1 -o gpurun_out/prof_c4 python scripts/fused_quick.py C4 148 > gpurun_out/ncu_c4.log 2>&1
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:rx_balanced -s 3 -c 1 -o gpurun_out/prof_c3 python scripts/fused_quick.py C3 1024 > gpurun_out/ncu_c3.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_c4.ncu-rep > gpurun_out/ncu_c4.txt 2>&1
python scripts/ncu_hot.py gpurun_out/prof_c4.ncu-rep 40 >> gpurun_out/ncu_c4.txt 2>&1
python scripts/ncu_summary.py gpurun_out/prof_c3.ncu-rep > gpurun_out/ncu_c3.txt 2>&1
python scripts/ncu_hot.py gpurun_out/prof_c3.ncu-rep 40 >> gpurun_out/ncu_c3.txt 2>&1
cat gpurun_out/ncu_c4.txt gpurun_out/ncu_c3.txt
