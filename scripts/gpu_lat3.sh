#!/bin/bash
timeout 300 python scripts/lat_quick.py C3 C1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lat_launches.csv python scripts/lat_quick.py C3 > /dev/null 2>&1
grep -E "lat_|rx_" gpurun_out/lat_launches.csv | awk -F'","' '{print $5, $NF}' | sed 's/(.*//' | sort | uniq -c | head; grep "lat_rows\|lat_combine" gpurun_out/lat_launches.csv | tail -3 | awk -F'","' '{print $5, $(NF)}'
timeout 900 python -m pytest -q -p no:cacheprovider -m gpu tests -k "latency or invariance" 2>&1 | tail -3
