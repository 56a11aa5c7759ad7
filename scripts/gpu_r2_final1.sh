#!/bin/bash
# validation after reverting C2 to rx_fused: full GPU tests, C2/C1/C3 quick, sanitizer on fused, bench C2 line
mkdir -p gpurun_out/san
for a in "C2 1000" "C1 65536" "C3 1024"; do timeout 120 python scripts/fused_quick.py $a; done 2>&1 | tee gpurun_out/quick_f1.log
timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests 2>&1 | tail -6
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python scripts/sanitize_cases.py fused > gpurun_out/san/racecheck_fused_f1.log 2>&1; grep "RACECHECK SUMMARY" gpurun_out/san/racecheck_fused_f1.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python scripts/sanitize_cases.py fused balanced > gpurun_out/san/memcheck_f1.log 2>&1; grep "ERROR SUMMARY" gpurun_out/san/memcheck_f1.log
timeout 900 python bench.py --config C2 --no-cpu-baseline --sweep-cells '' --no-latency > gpurun_out/bench_r02_C2.json 2> gpurun_out/bench_r02_C2.err; echo "bench C2 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_r02_C2.json'));print(d['value'], d['roofline']['frac'], d['check']['bits_vs_oracle'])"
