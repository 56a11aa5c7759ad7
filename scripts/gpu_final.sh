# round-end style validation on one B200: smoke, all GPU tests, default bench, reference arm, 2-rank smoke
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout -k 10 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout -k 10 500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout -k 10 500 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
bash scripts/gpu_multirank.sh
