#!/bin/bash
# paired sub-warp FFT lanes in the balanced kernel (M=256/512), staged segment path
mkdir -p gpurun_out
for a in "C2 1000" "C2 2000" "C3 1024" "C1 65536"; do timeout 120 python scripts/fused_quick.py $a; done 2>&1 | tee gpurun_out/quick_rb.log
timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests 2>&1 | tail -6
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:"rx_" -s 3 -c 1 -o /tmp/prof_c2 python scripts/fused_quick.py C2 1000 3 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/prof_c2.ncu-rep > gpurun_out/ncu_C2_rb.txt 2>&1
python scripts/ncu_hot.py /tmp/prof_c2.ncu-rep 30 >> gpurun_out/ncu_C2_rb.txt 2>&1
python scripts/ncu_opmix.py /tmp/prof_c2.ncu-rep 176000 30 > gpurun_out/opmix_C2_rb.txt 2>&1
head -24 gpurun_out/ncu_C2_rb.txt; head -12 gpurun_out/opmix_C2_rb.txt
