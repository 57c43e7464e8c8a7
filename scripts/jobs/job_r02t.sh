#!/bin/bash
# p re-check after the sort-tile change: bench step (no ncu / baseline) at several p.
out=gpurun_out/${OUT:-r02t}; mkdir -p $out
for p in 8 10 12; do timeout 900 python bench.py --config rmat24 --p $p --steps 10 --warmup 3 --no-cpu-baseline --no-ncu --e2e-steps 1 > $out/bench_rmat24_p$p.json 2>> $out/err.txt; done
for p in 4 6 8; do timeout 900 python bench.py --config orkut --p $p --steps 10 --warmup 3 --no-cpu-baseline --no-ncu --e2e-steps 1 > $out/bench_orkut_p$p.json 2>> $out/err.txt; done
for p in 2 3 4; do timeout 1500 python bench.py --config friendster --p $p --steps 3 --warmup 3 --no-cpu-baseline --no-ncu --e2e-steps 1 > $out/bench_friendster_p$p.json 2>> $out/err.txt; done
echo done >> $out/steps.txt
