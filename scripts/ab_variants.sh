#!/bin/bash
# A/B of experiment builds (build.py --variant NAME DEFINES...): fused_quick per variant
# usage: bash scripts/ab_variants.sh "C3 1024" name1 name2 ...   (libs under build/variants)
cfg=$1; shift
for i in 1 2; do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=""; else lib=build/variants/libofdmrx_b200_$v.so; fi
    OFDMRX_VARIANT_LIB=$lib timeout 120 python scripts/fused_quick.py $cfg | sed "s/^/$v /"
  done
done
