timeout -k 10 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout -k 10 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-frames 0 --no-stages > gpurun_out/bench.json 2> gpurun_out/bench.err
for c in C1 C2 C4; do timeout -k 10 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-frames 0 --no-stages > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
