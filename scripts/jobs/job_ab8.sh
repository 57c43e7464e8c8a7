#!/bin/bash
out=gpurun_out/${OUT:-ab8}; mkdir -p $out
for c in rmat24 orkut; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-ncu > $out/bench_${c}_seq.json 2>> $out/err.txt
  BBTC_DENSE_CONCURRENT=1 timeout 900 python bench.py --config $c --no-cpu-baseline --no-ncu > $out/bench_${c}_conc.json 2>> $out/err.txt
done
BBTC_DENSE_CONCURRENT=1 timeout 900 python -m pytest tests -m gpu -q -x -k "dense or karate or rmat16_p_grid" > $out/tests_conc.log 2>&1
echo done >> $out/steps.txt
