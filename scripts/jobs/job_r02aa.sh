#!/bin/bash
# L2 prefetch of the next batch's row offsets in the hash-only list kernel (BBTC_PF_ROWS) — friendster A/B.
out=gpurun_out/${OUT:-r02aa}; mkdir -p $out
timeout 2400 python scripts/ab_variants.py friendster paper_2009_12457_b200/libbbtc.so build_ab/pfrows/libbbtc.so paper_2009_12457_b200/libbbtc.so build_ab/pfrows/libbbtc.so > $out/ab.jsonl 2>> $out/err.txt
echo done >> $out/steps.txt
