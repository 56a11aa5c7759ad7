#!/bin/bash
bash scripts/ab_variants.sh "C4 296" base coopden coopden2
bash scripts/ab_variants.sh "C3 1024" coopden coopden2
