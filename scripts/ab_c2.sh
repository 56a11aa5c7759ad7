#!/bin/bash
# A/B of the M = 128 CTA shape over a few sweep cells (developer tool)
for c in "4x128 4096" "16x128 4096" "64x128 4096" "128x128 2978"; do
  bash scripts/ab_variants.sh "$c" base m128x3
done
