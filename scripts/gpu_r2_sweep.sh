#!/bin/bash
# full C5 sweep (reference CSV schema) + default bench + C4 bench line
mkdir -p gpurun_out
timeout 1500 python bench.py --sweep --sweep-csv gpurun_out/sweep_r02.csv > gpurun_out/sweep_r02.out 2> gpurun_out/sweep_r02.err; echo "sweep rc=$?"; cat gpurun_out/sweep_r02.out
timeout 900 python bench.py > gpurun_out/bench_r02_C3.json 2> gpurun_out/bench_r02_C3.err; echo "bench rc=$?"
timeout 900 python bench.py --config C4 --no-cpu-baseline > gpurun_out/bench_r02_C4.json 2> gpurun_out/bench_r02_C4.err; echo "bench C4 rc=$?"
timeout 900 python bench.py --config C2 --no-cpu-baseline --sweep-cells '' > gpurun_out/bench_r02_C2.json 2> gpurun_out/bench_r02_C2.err; echo "bench C2 rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_r02_ref.json 2> gpurun_out/bench_r02_ref.err; echo "ref rc=$?"
