#!/bin/bash
# Work items per warp slot re-checked with the round-2 kernels.
out=gpurun_out/${OUT:-r02jj}; mkdir -p $out
timeout 3000 python scripts/ab_variants.py rmat24:10,orkut,friendster paper_2009_12457_b200/libbbtc.so "env:BBTC_ITEMS_PER_SLOT=256" "env:BBTC_ITEMS_PER_SLOT=512" "env:BBTC_ITEMS_PER_SLOT=768" > $out/ab.jsonl 2>> $out/err.txt
echo done >> $out/steps.txt
