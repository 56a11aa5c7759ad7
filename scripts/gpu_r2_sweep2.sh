#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_receiver_api.py tests/test_gpu_reference_dropin.py 2>&1 | tail -3
timeout 1500 python bench.py --sweep --sweep-csv gpurun_out/sweep_r02.csv > gpurun_out/sweep_r02.out 2> gpurun_out/sweep_r02.err; echo "sweep rc=$?"; cat gpurun_out/sweep_r02.out
