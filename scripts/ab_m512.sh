#!/bin/bash
# A/B of rx_fused CTA shapes at M = 512 (developer tool)
for c in "4x512 4096" "16x512 4096" "64x512 1489" "128x512 744"; do
  bash scripts/ab_variants.sh "$c" base m512x2
done
