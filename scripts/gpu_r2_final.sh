#!/bin/bash
# round-2 final validation: smoke, GPU tests, default bench, reference arm, ncu launch list of the bench
# command, ncu --set full of the C3 product kernel (traffic for the bench line), sanitizer summary
mkdir -p gpurun_out/final gpurun_out/san
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1800 python -m pytest -q -p no:cacheprovider -m gpu tests > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/final/pytest_gpu.log
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:"rx_balanced" -s 3 -c 1 -o /tmp/prof_c3 python scripts/fused_quick.py C3 1024 3 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/prof_c3.ncu-rep > gpurun_out/final/ncu_C3_1024.txt 2>&1
python scripts/ncu_hot.py /tmp/prof_c3.ncu-rep 40 >> gpurun_out/final/ncu_C3_1024.txt 2>&1
python scripts/ncu_opmix.py /tmp/prof_c3.ncu-rep 720896 45 > gpurun_out/final/opmix_C3_1024.txt 2>&1
python scripts/traffic_from_ncu.py /tmp/prof_c3.ncu-rep 1024 C3 "profiles/ncu_r02_C3_1024.txt" > /dev/null 2>&1; cp profiles/traffic_C3.json gpurun_out/final/traffic_C3.json
timeout 600 python bench.py > gpurun_out/final/bench_C3.json 2> gpurun_out/final/bench_C3.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_C3.csv python bench.py --steps 2 --warmup 3 --sustained-steps 0 --no-stages --sweep-cells '' --no-latency --no-cpu-baseline --oracle-frames 0 > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err; echo "ref rc=$?"
python -c "
import json
d=json.load(open('gpurun_out/final/bench_C3.json'))
print('value', d['value'], 'frac', d['roofline']['frac'], 'traffic', d['roofline']['traffic'], 'check', d['check']['bits_vs_oracle'], 'sustained', d['sustained']['roofline_frac'], 'e2e', d['e2e']['value'])
print('latency C3 kernel', d['latency']['C3']['kernel_us_per_frame'], 'graph', d['latency']['C3']['graph_us_per_frame'])
r=json.load(open('gpurun_out/final/bench_ref.json')); print('ref', r['value'])
"
