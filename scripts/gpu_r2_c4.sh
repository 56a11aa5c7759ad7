#!/bin/bash
# racecheck logs of the hazard-reporting cases; C4 plan (V for L2 residency) timing + ncu; invariance
mkdir -p gpurun_out/san
for c in fused partials staged; do
  timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 6 python scripts/sanitize_cases.py $c > gpurun_out/san/racecheck_${c}.log 2>&1
  echo "racecheck $c rc=$? $(grep -E 'RACECHECK SUMMARY' gpurun_out/san/racecheck_${c}.log | tail -1)"
done
for a in "C4 64" "C4 148" "C4 256" "C3 1024" "C3 64"; do timeout 120 python scripts/fused_quick.py $a; done 2>&1 | tee gpurun_out/quick_c4.log
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_invariance.py tests/test_gpu_parity.py 2>&1 | tail -3
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:"rx_" -s 3 -c 1 -o /tmp/prof_c4 python scripts/fused_quick.py C4 148 3 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/prof_c4.ncu-rep > gpurun_out/ncu_C4_148_v48.txt 2>&1
python scripts/ncu_hot.py /tmp/prof_c4.ncu-rep 30 >> gpurun_out/ncu_C4_148_v48.txt 2>&1
head -24 gpurun_out/ncu_C4_148_v48.txt
