#!/bin/bash
bash scripts/ab_variants.sh "C3 1024" base macpipe
bash scripts/ab_variants.sh "C4 296" base macpipe
