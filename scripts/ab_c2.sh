#!/bin/bash
# A/B over the rx_fused shapes (developer tool): usage bash scripts/ab_c2.sh variant...
for c in "C2 1000" "C2 2000" "16x128 4096" "128x128 2978" "C1 65536"; do
  bash scripts/ab_variants.sh "$c" "$@"
done
