#!/bin/bash
out=gpurun_out/${OUT:-ab9}; mkdir -p $out
timeout 2400 python scripts/ab_variants.py rmat24:10,orkut,friendster paper_2009_12457_b200/libbbtc.so build_ab/hint/libbbtc.so > $out/ab_hint.jsonl 2>> $out/err.txt
echo done >> $out/steps.txt
