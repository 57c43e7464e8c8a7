#!/bin/bash
out=gpurun_out/${OUT:-ab2}; mkdir -p $out
timeout 1500 python scripts/ab_variants.py rmat24:10,rmat24:12,orkut paper_2009_12457_b200/libbbtc.so > $out/ab_default.jsonl 2>> $out/err.txt
BBTC_DENSE_WALK=row timeout 1500 python scripts/ab_variants.py rmat24:10,rmat24:12,orkut paper_2009_12457_b200/libbbtc.so > $out/ab_dense_row.jsonl 2>> $out/err.txt
timeout 1500 python -m pytest tests -m gpu -q -x -k "multi or shard or nccl or bench_two" > $out/tests_multi.log 2>&1
echo done >> $out/steps.txt
