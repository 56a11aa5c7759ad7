#!/bin/bash
mkdir -p gpurun_out
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:"rx_" -s 3 -c 1 -o /tmp/prof_c4 python scripts/fused_quick.py C4 296 3 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/prof_c4.ncu-rep > gpurun_out/ncu_C4_296.txt 2>&1
python scripts/ncu_hot.py /tmp/prof_c4.ncu-rep 40 >> gpurun_out/ncu_C4_296.txt 2>&1
python scripts/ncu_opmix.py /tmp/prof_c4.ncu-rep 833536 40 > gpurun_out/opmix_C4_296.txt 2>&1
