#!/bin/bash
out=gpurun_out/${OUT:-ab6}; mkdir -p $out
timeout 2400 python scripts/ab_variants.py friendster:4,friendster:8,friendster:16,rmat24:10,orkut paper_2009_12457_b200/libbbtc.so > $out/ab_order_kji.jsonl 2>> $out/err.txt
BBTC_TASK_ORDER=ikj timeout 2400 python scripts/ab_variants.py friendster:4,friendster:8,friendster:16,rmat24:10,orkut paper_2009_12457_b200/libbbtc.so > $out/ab_order_ikj.jsonl 2>> $out/err.txt
echo done >> $out/steps.txt
