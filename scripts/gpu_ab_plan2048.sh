#!/bin/bash
bash scripts/ab_variants.sh "C4 296" base plan2048
bash scripts/ab_variants.sh "C4 64" base plan2048
