# usage: bash scripts/ab.sh CFG FRAMES variant1 variant2 ...   (A/B of build/variants/*.so)
cfg=$1; fr=$2; shift 2
for v in "$@"; do
  OFDMRX_VARIANT_LIB=build/variants/libofdmrx_b200_$v.so timeout 120 python scripts/fused_quick.py $cfg $fr 2>&1 | tail -1
done
