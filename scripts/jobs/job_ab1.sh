#!/bin/bash
out=gpurun_out/${OUT:-ab1}; mkdir -p $out
timeout 1800 python scripts/ab_variants.py rmat24,orkut,friendster paper_2009_12457_b200/libbbtc.so build_ab/min6/libbbtc.so > $out/ab_min6.jsonl 2>> $out/err.txt
BBTC_ITEM_COST=merge timeout 1800 python scripts/ab_variants.py rmat24,orkut,friendster paper_2009_12457_b200/libbbtc.so > $out/ab_itemcost_merge.jsonl 2>> $out/err.txt
for p in 8 10 12; do timeout 900 python bench.py --no-cpu-baseline --no-ncu --p $p > $out/bench_rmat24_p$p.json 2>> $out/err.txt; done
timeout 600 python -m pytest tests -m gpu -q -x -k "bucket or counting_sort or packed" > $out/tests.log 2>&1
echo done >> $out/steps.txt
