#!/bin/bash
mkdir -p gpurun_out
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:"rx_" -s 3 -c 1 -o /tmp/prof_c2 python scripts/fused_quick.py C2 1000 3 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/prof_c2.ncu-rep > gpurun_out/ncu_C2_fused.txt 2>&1
python scripts/ncu_hot.py /tmp/prof_c2.ncu-rep 50 >> gpurun_out/ncu_C2_fused.txt 2>&1
python scripts/ncu_opmix.py /tmp/prof_c2.ncu-rep 176000 40 > gpurun_out/opmix_C2_fused.txt 2>&1
ncu -i /tmp/prof_c2.ncu-rep --page details --csv 2>/dev/null | grep -i "occupancy\|Block Limit\|Waves\|Registers\|Shared Memory" | head -30 > gpurun_out/occ_C2.txt
