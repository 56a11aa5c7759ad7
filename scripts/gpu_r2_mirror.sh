#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_receiver_api.py tests/test_gpu_reference_dropin.py tests/test_gpu_invariance.py tests/test_gpu_parity.py 2>&1 | tail -4
timeout 900 python - <<'PY'
import json, sys
sys.path.insert(0, ".")
import bench
recs, summ = bench.sweep_cells([(8, 64), (16, 256), (64, 1024), (128, 4096)], reps=3)
for c in summ:
    print(c["fft_len"], c["n_antennas"], json.dumps(c.get("pipeline_us_per_symbol")), c.get("bits_equal_reference"))
PY
