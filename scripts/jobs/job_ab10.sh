#!/bin/bash
out=gpurun_out/${OUT:-ab10}; mkdir -p $out
for mn in 37 1; do
  for c in orkut friendster; do
    BBTC_TRACE=1 BBTC_BATCHED_MIN_NB=$mn timeout 1500 python bench.py --config $c --no-cpu-baseline --no-ncu --steps 3 --warmup 2 --e2e-steps 1 > $out/bench_${c}_mn$mn.json 2> $out/trace_${c}_mn$mn.log
  done
done
echo done >> $out/steps.txt
