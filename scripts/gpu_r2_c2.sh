#!/bin/bash
# C2 on the balanced kernel (M=256 plan P=8 x 32), latency plan, full GPU tests, sanitizers, bench
mkdir -p gpurun_out
for a in "C2 1000" "C1 65536" "C3 1024" "C3 64" "C4 296"; do timeout 120 python scripts/fused_quick.py $a; done 2>&1 | tee gpurun_out/quick_c2.log
timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests -x 2>&1 | tail -15
timeout 900 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench rc=$?"; tail -3 gpurun_out/bench3.err
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:"rx_" -s 3 -c 1 -o /tmp/prof_c2 python scripts/fused_quick.py C2 1000 3 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/prof_c2.ncu-rep > gpurun_out/ncu_C2_1000_bal.txt 2>&1
python scripts/ncu_hot.py /tmp/prof_c2.ncu-rep 30 >> gpurun_out/ncu_C2_1000_bal.txt 2>&1
head -24 gpurun_out/ncu_C2_1000_bal.txt
bash scripts/sanitize.sh 2>&1 | tail -40
