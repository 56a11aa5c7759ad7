#!/bin/bash
# compute-sanitizer over every kernel (scripts/sanitize_cases.py) -> gpurun_out/san/
#   memcheck / synccheck / initcheck on the product library;
#   racecheck on the product library AND on the OFDMRX_RACECHECK_SERIAL build
#   (sub-warp FFT lanes of rx_fused issue / wait on their TMA mbarriers one lane
#   at a time; see rx_fused.cu "issue"), which racecheck can attribute.
# Build the variant first (CPU is fine):
#   python -m paper_1901_07499_b200.build --variant racecheck OFDMRX_RACECHECK_SERIAL
mkdir -p gpurun_out/san
CASES="balanced latency fused partials staged detect corr synth"
for tool in memcheck synccheck initcheck racecheck; do
  for c in $CASES; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 10 python scripts/sanitize_cases.py $c > gpurun_out/san/${tool}_${c}.log 2>&1
    echo "$tool product $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/${tool}_${c}.log | tail -1)"
  done
done
for c in fused partials staged; do
  OFDMRX_VARIANT_LIB=build/variants/libofdmrx_b200_racecheck.so timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 10 python scripts/sanitize_cases.py $c > gpurun_out/san/racecheck_serial_${c}.log 2>&1
  echo "racecheck serial-build $c rc=$? $(grep -E 'RACECHECK SUMMARY' gpurun_out/san/racecheck_serial_${c}.log | tail -1)"
done
