#!/bin/bash
out=gpurun_out/${OUT:-r02ee}; mkdir -p $out
timeout 2400 python scripts/balance_study.py rmat24:10 orkut:8 friendster:4 friendster:8 rmat24:16 > $out/balance.jsonl 2> $out/err.txt
echo done >> $out/steps.txt
