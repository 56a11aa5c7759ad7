# C4 antenna-sharded, 2 ranks on one GPU (OFDMRX_SAME_DEVICE), peer-memory exchange vs NCCL-free gloo gather
export OFDMRX_DIST_BACKEND=gloo OFDMRX_SAME_DEVICE=1
timeout -k 10 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --config C4 --gpus 2 --steps 5 --warmup 3 --frames 32 --exchange peer --e2e-frames 0 --no-cpu-baseline > gpurun_out/bench_c4_peer.json 2> gpurun_out/bench_c4_peer.err
