#!/bin/bash
# A/B: C4 L2 residency experiments (pdesc, hlast, both) and the FFT form-1 FFMA2 butterfly (f1fma) on C3/C4
bash scripts/ab_variants.sh "C4 296" base pdesc hlast both f1fma
bash scripts/ab_variants.sh "C3 1024" base pdesc f1fma
