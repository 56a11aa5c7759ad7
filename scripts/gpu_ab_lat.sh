#!/bin/bash
for i in 1 2; do
  timeout 300 python scripts/lat_quick.py C3 | head -1
  OFDMRX_VARIANT_LIB=build/variants/libofdmrx_b200_oldcomb.so timeout 300 python scripts/lat_quick.py C3 | head -1 | sed 's/^/old /'
done
