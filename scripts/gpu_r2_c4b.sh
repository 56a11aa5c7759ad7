#!/bin/bash
# racecheck after the single-issuer TMA change; antenna-major phase B timing; tests; bench
mkdir -p gpurun_out/san
for c in fused partials staged; do
  timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 6 python scripts/sanitize_cases.py $c > gpurun_out/san/racecheck2_${c}.log 2>&1
  echo "racecheck $c rc=$? $(grep -E 'RACECHECK SUMMARY' gpurun_out/san/racecheck2_${c}.log | tail -1)"
done
for a in "C4 64" "C4 148" "C4 296" "C3 1024" "C3 64" "C2 1000" "C1 65536"; do timeout 120 python scripts/fused_quick.py $a; done 2>&1 | tee gpurun_out/quick_c4b.log
timeout 1200 python -m pytest -q -p no:cacheprovider -m gpu tests 2>&1 | tail -4
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:"rx_" -s 3 -c 1 -o /tmp/prof_c4 python scripts/fused_quick.py C4 148 3 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/prof_c4.ncu-rep > gpurun_out/ncu_C4_148_amaj.txt 2>&1
python scripts/ncu_hot.py /tmp/prof_c4.ncu-rep 30 >> gpurun_out/ncu_C4_148_amaj.txt 2>&1
head -24 gpurun_out/ncu_C4_148_amaj.txt
timeout 900 python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench rc=$?"; tail -3 gpurun_out/bench2.err
