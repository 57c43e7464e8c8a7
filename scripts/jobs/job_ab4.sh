#!/bin/bash
out=gpurun_out/${OUT:-ab4}; mkdir -p $out
for r in 2 4 8 16; do for b in 8192 16384; do
  BBTC_DENSE_RATIO=$r BBTC_DENSE_BITS=$b timeout 900 python scripts/ab_variants.py rmat24:10,rmat24:8,rmat24:12 paper_2009_12457_b200/libbbtc.so | sed "s/^{/{\"ratio\": $r, \"bits\": $b, /" >> $out/ab_dense_grid_row.jsonl 2>> $out/err.txt
done; done
for r in 2 4 8; do BBTC_DENSE_RATIO=$r timeout 900 python scripts/ab_variants.py orkut paper_2009_12457_b200/libbbtc.so | sed "s/^{/{\"ratio\": $r, /" >> $out/ab_dense_orkut.jsonl 2>> $out/err.txt; done
timeout 900 python -m pytest tests -m gpu -q -x -k "dense or karate or rmat16_p_grid or stream" > $out/tests.log 2>&1
echo done >> $out/steps.txt
