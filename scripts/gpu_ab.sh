#!/bin/bash
# A/B of variant builds over the four bench configs (developer tool)
# usage: bash scripts/gpu_ab.sh name1 name2 ...   (base = the in-tree library)
for c in "C3 1024" "C2 1000" "C1 2048" "C4 296"; do
  bash scripts/ab_variants.sh "$c" "$@"
done
