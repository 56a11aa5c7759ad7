set -x
timeout -k 10 400 python bench.py --steps 50 --warmup 5 --cpu-seconds 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout -k 10 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
