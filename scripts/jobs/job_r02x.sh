#!/bin/bash
# Pipelined column runs in the bitmap kernel variant (BBTC_RUN_PIPE_BM=1) re-checked with the round-2 kernel.
out=gpurun_out/${OUT:-r02x}; mkdir -p $out
timeout 2400 python scripts/ab_variants.py rmat24:10,orkut paper_2009_12457_b200/libbbtc.so build_ab/pipebm/libbbtc.so > $out/ab.jsonl 2>> $out/err.txt
echo done >> $out/steps.txt
