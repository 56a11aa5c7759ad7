for c in C1 C2 C4; do
  timeout -k 10 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-frames 0 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout -k 10 600 ncu --set full --clock-control none -k regex:rx_fused -s 3 -c 1 -o gpurun_out/prof_C2 python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline --e2e-frames 0 --no-stages > /dev/null 2>&1
timeout -k 10 600 ncu --set full --clock-control none -k regex:rx_fused -s 3 -c 1 -o gpurun_out/prof_C1 python bench.py --config C1 --steps 1 --warmup 3 --no-cpu-baseline --e2e-frames 0 --no-stages --frames 16384 > /dev/null 2>&1
