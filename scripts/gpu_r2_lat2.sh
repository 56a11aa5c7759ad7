#!/bin/bash
# row-parallel latency path: tests, sanitizer, latency bench section
mkdir -p gpurun_out/san
timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests 2>&1 | tail -6
for tool in memcheck racecheck synccheck; do timeout 600 compute-sanitizer --tool $tool --print-limit 10 python scripts/sanitize_cases.py latency > gpurun_out/san/${tool}_latency.log 2>&1; echo "$tool latency $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/${tool}_latency.log | tail -1)"; done
timeout 600 python bench.py --steps 5 --warmup 3 --sustained-steps 0 --e2e-frames 0 --no-stages --sweep-cells '' --no-cpu-baseline --oracle-frames 0 > gpurun_out/bench_lat2.json 2> gpurun_out/bench_lat2.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_lat2.json'));print(json.dumps(d.get('latency'))[:3000])"
for a in "C3 1024" "C4 296"; do timeout 120 python scripts/fused_quick.py $a; done
