#!/bin/bash
# bench lines with graph-replayed steps: C3 default, then C4 / C2 / C1 as gpu_r2_lines.sh runs them
mkdir -p gpurun_out/final
timeout 600 python bench.py --sweep-cells '' --no-latency --no-cpu-baseline > gpurun_out/final/bench_C3g.json 2> gpurun_out/final/bench_C3g.err; echo "C3 rc=$?"
bash scripts/gpu_r2_lines.sh
python -c "
import json
d=json.load(open('gpurun_out/final/bench_C3g.json')); print('C3', d['value'], d['roofline']['frac'], d['check'].get('bits_vs_oracle'), d['sustained']['roofline_frac'], d['config']['launch'])
"
