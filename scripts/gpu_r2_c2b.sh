#!/bin/bash
# C2 balanced (M=256) + latency plan + all-arrive ring barriers: timing, tests, racecheck on rx_fused, bench
mkdir -p gpurun_out/san
for a in "C2 1000" "C2 2000" "C1 65536" "C3 1024" "C4 296"; do timeout 120 python scripts/fused_quick.py $a; done 2>&1 | tee gpurun_out/quick_c2b.log
timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests 2>&1 | tail -8
for c in fused partials staged; do
  timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 10 python scripts/sanitize_cases.py $c > gpurun_out/san/racecheck_${c}.log 2>&1
  echo "racecheck product $c rc=$? $(grep -E 'RACECHECK SUMMARY' gpurun_out/san/racecheck_${c}.log | tail -1)"
  OFDMRX_VARIANT_LIB=build/variants/libofdmrx_b200_racecheck.so timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 10 python scripts/sanitize_cases.py $c > gpurun_out/san/racecheck_serial_${c}.log 2>&1
  echo "racecheck serial $c rc=$? $(grep -E 'RACECHECK SUMMARY' gpurun_out/san/racecheck_serial_${c}.log | tail -1)"
done
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:"rx_" -s 3 -c 1 -o /tmp/prof_c2 python scripts/fused_quick.py C2 1000 3 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/prof_c2.ncu-rep > gpurun_out/ncu_C2_1000_bal.txt 2>&1
python scripts/ncu_hot.py /tmp/prof_c2.ncu-rep 30 >> gpurun_out/ncu_C2_1000_bal.txt 2>&1
head -24 gpurun_out/ncu_C2_1000_bal.txt
timeout 900 python bench.py > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo "bench rc=$?"; tail -3 gpurun_out/bench4.err
