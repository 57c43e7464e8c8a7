#!/bin/bash
out=gpurun_out/${OUT:-ab3}; mkdir -p $out
BBTC_DENSE_WALK=row timeout 1500 python scripts/ab_variants.py rmat24:10,orkut paper_2009_12457_b200/libbbtc.so > $out/ab_dense_row.jsonl 2>> $out/err.txt
for r in 2 4 8; do for b in 4096 8192 16384; do
  BBTC_DENSE_RATIO=$r BBTC_DENSE_BITS=$b timeout 900 python scripts/ab_variants.py rmat24:10 paper_2009_12457_b200/libbbtc.so | sed "s/^{/{\"ratio\": $r, \"bits\": $b, /" >> $out/ab_dense_grid.jsonl 2>> $out/err.txt
done; done
echo done >> $out/steps.txt
