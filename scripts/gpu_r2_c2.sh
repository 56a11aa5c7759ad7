#!/bin/bash
# after an rx_fused plan change: GPU tests, C2/C1 bench lines, C2 ncu summary, full sweep
mkdir -p gpurun_out/final
timeout 1800 python -m pytest -q -p no:cacheprovider -m gpu tests > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/final/pytest_gpu.log
timeout 900 python bench.py --config C2 --no-cpu-baseline --sweep-cells '' --no-latency > gpurun_out/final/bench_C2.json 2> gpurun_out/final/bench_C2.err; echo "C2 rc=$?"
python -c "
import json
for c in ('C2',):
    d=json.load(open(f'gpurun_out/final/bench_{c}.json')); print(c, d['value'], d['roofline']['frac'], d['check'].get('bits_vs_oracle'), d.get('sustained',{}).get('roofline_frac'))
"
rm -f /tmp/prof_c2.ncu-rep
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:"rx_" -s 3 -c 1 -o /tmp/prof_c2 python scripts/fused_quick.py C2 1000 3 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/prof_c2.ncu-rep > gpurun_out/final/ncu_C2_1000.txt 2>&1
python scripts/ncu_hot.py /tmp/prof_c2.ncu-rep 30 >> gpurun_out/final/ncu_C2_1000.txt 2>&1
python scripts/ncu_opmix.py /tmp/prof_c2.ncu-rep 176000 40 > gpurun_out/final/opmix_C2_1000.txt 2>&1
ncu -i /tmp/prof_c2.ncu-rep --page details --csv 2>/dev/null | grep -i "occupancy\|Block Limit\|Waves\|Registers\|Shared Memory" | head -30 > gpurun_out/final/occ_C2.txt
timeout 1500 python bench.py --sweep --sweep-csv gpurun_out/final/sweep_r02.csv > gpurun_out/final/sweep_r02.out 2> gpurun_out/final/sweep_r02.err; echo "sweep rc=$?"; cat gpurun_out/final/sweep_r02.out
