# usage: bash scripts/ab_sustained.sh CFG FRAMES REPS variant1 variant2 ...  (sleep between runs to cool)
cfg=$1; fr=$2; reps=$3; shift 3
for v in "$@"; do
  sleep 5
  OFDMRX_VARIANT_LIB=build/variants/libofdmrx_b200_$v.so timeout 200 python scripts/fused_quick.py $cfg $fr $reps 2>&1 | tail -1
done
