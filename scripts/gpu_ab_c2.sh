#!/bin/bash
# C2 A/B: product (paired lanes, 1 CTA/SM), min2 (paired lanes at 85 registers, 2 CTAs/SM), nobal256 (rx_fused)
bash scripts/ab_variants.sh "C2 1000" base min2 nobal256
bash scripts/ab_variants.sh "C2 2000" base min2 nobal256
