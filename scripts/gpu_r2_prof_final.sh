#!/bin/bash
# ncu summaries of the C2 and C4 product kernels on the final round-2 sources
mkdir -p gpurun_out/final
rm -f /tmp/prof_c2.ncu-rep /tmp/prof_c4.ncu-rep
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:"rx_" -s 3 -c 1 -o /tmp/prof_c2 python scripts/fused_quick.py C2 1000 3 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/prof_c2.ncu-rep > gpurun_out/final/ncu_C2_1000.txt 2>&1
python scripts/ncu_hot.py /tmp/prof_c2.ncu-rep 30 >> gpurun_out/final/ncu_C2_1000.txt 2>&1
python scripts/ncu_opmix.py /tmp/prof_c2.ncu-rep 176000 40 > gpurun_out/final/opmix_C2_1000.txt 2>&1
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:"rx_" -s 3 -c 1 -o /tmp/prof_c4 python scripts/fused_quick.py C4 296 3 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/prof_c4.ncu-rep > gpurun_out/final/ncu_C4_296.txt 2>&1
python scripts/ncu_hot.py /tmp/prof_c4.ncu-rep 40 >> gpurun_out/final/ncu_C4_296.txt 2>&1
python scripts/ncu_opmix.py /tmp/prof_c4.ncu-rep 833536 40 > gpurun_out/final/opmix_C4_296.txt 2>&1
python scripts/traffic_from_ncu.py /tmp/prof_c4.ncu-rep 296 C4 "profiles/ncu_r02_C4_296.txt" > /dev/null 2>&1; cp profiles/traffic_C4.json gpurun_out/final/traffic_C4.json 2>/dev/null
ls -la gpurun_out/final/
