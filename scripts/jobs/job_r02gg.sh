#!/bin/bash
# Coarser work items for the bit-row tasks (BBTC_DENSE_CHUNK_X).
out=gpurun_out/${OUT:-r02gg}; mkdir -p $out
timeout 2400 python scripts/ab_variants.py rmat24:10,orkut paper_2009_12457_b200/libbbtc.so "env:BBTC_DENSE_CHUNK_X=2" "env:BBTC_DENSE_CHUNK_X=4" "env:BBTC_DENSE_CHUNK_X=8" paper_2009_12457_b200/libbbtc.so > $out/ab.jsonl 2>> $out/err.txt
echo done >> $out/steps.txt
