#!/bin/bash
# grouped den (latency plan), C3 op mix
mkdir -p gpurun_out
for a in "C3 1024" "C4 296" "C2 1000"; do timeout 120 python scripts/fused_quick.py $a; done 2>&1 | tee gpurun_out/quick_lat.log
timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests -k "invariance or parity or latency or golden or fuzz or balanced" 2>&1 | tail -4
timeout 600 python bench.py --steps 5 --warmup 3 --sustained-steps 0 --e2e-frames 0 --no-stages --sweep-cells '' --no-cpu-baseline --oracle-frames 0 > gpurun_out/bench_lat.json 2> gpurun_out/bench_lat.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_lat.json'));print(json.dumps(d.get('latency'))[:3000])"
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:"rx_" -s 3 -c 1 -o /tmp/prof_c3 python scripts/fused_quick.py C3 1024 3 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/prof_c3.ncu-rep > gpurun_out/ncu_C3_1024.txt 2>&1
python scripts/ncu_hot.py /tmp/prof_c3.ncu-rep 40 >> gpurun_out/ncu_C3_1024.txt 2>&1
python scripts/ncu_opmix.py /tmp/prof_c3.ncu-rep 720896 45 > gpurun_out/opmix_C3_1024.txt 2>&1
python scripts/traffic_from_ncu.py /tmp/prof_c3.ncu-rep 1024 C3 "profiles/ncu_r02_C3_1024.txt" > /dev/null 2>&1; cp profiles/traffic_C3.json gpurun_out/traffic_C3.json
cat gpurun_out/opmix_C3_1024.txt
