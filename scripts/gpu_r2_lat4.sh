#!/bin/bash
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests/test_gpu_invariance.py tests/test_gpu_parity.py -k "latency" 2>&1 | tail -3
timeout 300 python scripts/lat_quick.py C3 C1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/lat.csv python scripts/lat_quick.py C3 > /dev/null 2>&1
grep "lat_rows\|lat_combine" /tmp/lat.csv | tail -3 | awk -F'","' '{print $5, $(NF)}'
