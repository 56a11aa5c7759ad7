export OFDMRX_DIST_BACKEND=gloo OFDMRX_SAME_DEVICE=1
timeout -k 10 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --frames 256 --e2e-frames 32 > gpurun_out/bench_mr.json 2> gpurun_out/bench_mr.err
timeout -k 10 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_mr_ref.json 2> gpurun_out/bench_mr_ref.err
