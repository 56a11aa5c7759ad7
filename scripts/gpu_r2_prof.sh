#!/bin/bash
# round 2: fixed-test check, compute-sanitizer on every kernel, ncu --set full of C2 / C3 / C4
mkdir -p gpurun_out/san
timeout 600 python -m pytest -q -p no:cacheprovider tests/test_gpu_receiver_api.py tests/test_gpu_reference_dropin.py 2>&1 | tail -3
for tool in memcheck racecheck synccheck initcheck; do
  for c in balanced fused partials staged detect corr synth; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py $c > gpurun_out/san/${tool}_${c}.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/${tool}_${c}.log | tail -1)"
  done
done
for spec in "C2 1000" "C4 148" "C4 64" "C3 1024"; do
  set -- $spec
  timeout -k 10 900 ncu --set full --clock-control none --import-source on -k regex:"rx_|finish" -s 3 -c 1 -o gpurun_out/prof_${1}_$2 python scripts/fused_quick.py $1 $2 3 > gpurun_out/ncu_${1}_$2.log 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_${1}_$2.ncu-rep > gpurun_out/ncu_${1}_$2.txt 2>&1
  python scripts/ncu_hot.py gpurun_out/prof_${1}_$2.ncu-rep 30 >> gpurun_out/ncu_${1}_$2.txt 2>&1
  head -30 gpurun_out/ncu_${1}_$2.txt
done
