#!/bin/bash
# branch-free epilogue: bit-identity test, parity subset, A/B against the per-subcarrier epilogue
timeout 300 python -m pytest -q -p no:cacheprovider tests/test_gpu_division.py 2>&1 | grep -v "^\s*$" | tail -15
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_invariance.py 2>&1 | tail -3
for c in "C3 1024" "C2 1000" "C1 65536" "C4 296"; do bash scripts/ab_variants.sh "$c" base epiplain; done
