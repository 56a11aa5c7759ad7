#!/bin/bash
# bench lines for C4 and C2 (and C1), round-2 sources
mkdir -p gpurun_out/final
timeout 900 python bench.py --config C4 --no-cpu-baseline > gpurun_out/final/bench_C4.json 2> gpurun_out/final/bench_C4.err; echo "C4 rc=$?"
timeout 900 python bench.py --config C2 --no-cpu-baseline --sweep-cells '' --no-latency > gpurun_out/final/bench_C2.json 2> gpurun_out/final/bench_C2.err; echo "C2 rc=$?"
timeout 900 python bench.py --config C1 --no-cpu-baseline --sweep-cells '' --no-latency --e2e-frames 0 > gpurun_out/final/bench_C1.json 2> gpurun_out/final/bench_C1.err; echo "C1 rc=$?"
python -c "
import json
for c in ('C4','C2','C1'):
    d=json.load(open(f'gpurun_out/final/bench_{c}.json')); print(c, d['value'], d['roofline']['frac'], d['check'].get('bits_vs_oracle'), d.get('sustained',{}).get('roofline_frac'))
"
