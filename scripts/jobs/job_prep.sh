#!/bin/bash
out=gpurun_out/${OUT:-prep}; mkdir -p $out
timeout 1800 python -m pytest tests -m gpu -q -x -k "bucket or preprocessing or round_trip or packed or rmat16_p_grid or full_size or many_parts or random_graphs or karate or degenerate or hash_canon" > $out/tests.log 2>&1; echo "tests rc=$?" >> $out/steps.txt
BBTC_TRACE=1 timeout 900 python bench.py --no-cpu-baseline --no-ncu --steps 5 --warmup 3 > $out/bench_rmat24.json 2> $out/bench_rmat24.err; echo "bench rc=$?" >> $out/steps.txt
for p in 8 10 12; do timeout 900 python bench.py --no-cpu-baseline --no-ncu --p $p > $out/bench_rmat24_p$p.json 2>> $out/err.txt; done
timeout 900 python bench.py --config orkut --no-cpu-baseline --no-ncu > $out/bench_orkut.json 2>> $out/err.txt
timeout 1500 python bench.py --config friendster --no-cpu-baseline --no-ncu --steps 3 --warmup 3 > $out/bench_friendster.json 2>> $out/err.txt
echo done >> $out/steps.txt
