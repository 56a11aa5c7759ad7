#!/bin/bash
# A/B of rx_fused CTA shapes at M = 64 (developer tool)
for c in "C1 65536" "64x64 4096" "128x64 4096" "4x64 4096"; do
  bash scripts/ab_variants.sh "$c" base m64x4 m64x3
done
