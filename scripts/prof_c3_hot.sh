#!/bin/bash
rm -f /tmp/prof_c3h.ncu-rep
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:"rx_balanced" -s 3 -c 1 -o /tmp/prof_c3h python scripts/fused_quick.py C3 1024 3 > /dev/null 2>&1
python scripts/ncu_hot.py /tmp/prof_c3h.ncu-rep 60 > gpurun_out/c3_hot60.txt 2>&1
python scripts/ncu_col.py /tmp/prof_c3h.ncu-rep '?' > gpurun_out/c3_cols.txt 2>&1
