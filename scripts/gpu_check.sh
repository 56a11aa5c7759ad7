set -x
timeout -k 10 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout -k 10 300 python bench.py --steps 10 --warmup 3 --e2e-frames 32 --cpu-seconds 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:rx_fused -s 3 -c 1 -o gpurun_out/prof_fused python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-frames 0 --frames 512 > gpurun_out/ncu_full.log 2>&1
