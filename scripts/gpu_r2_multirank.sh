#!/bin/bash
# 2-rank smoke of the bench under torchrun on ONE GPU (gloo plumbing, OFDMRX_SAME_DEVICE): exercises the
# multi-rank code paths (frame sharding with graph-replayed steps; antenna-sharded C4 scatter exchange),
# not a scaling number
mkdir -p gpurun_out/final
export OFDMRX_DIST_BACKEND=gloo OFDMRX_SAME_DEVICE=1
timeout -k 10 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --frames 256 --e2e-frames 32 --sweep-cells '' --no-latency > gpurun_out/final/bench_mr.json 2> gpurun_out/final/bench_mr.err; echo "frame-sharded rc=$?"
timeout -k 10 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --config C4 --gpus 2 --steps 5 --warmup 3 --frames 64 --e2e-frames 0 --sweep-cells '' --no-latency --no-cpu-baseline > gpurun_out/final/bench_mr_c4.json 2> gpurun_out/final/bench_mr_c4.err; echo "antenna-sharded rc=$?"
python -c "
import json
for f in ('bench_mr','bench_mr_c4'):
    d=json.load(open(f'gpurun_out/final/{f}.json')); print(f, d['n_gpus'], d['value'], d['config']['parallelism'], d['check'].get('bits_vs_oracle'), d['config'].get('launch'))
"
