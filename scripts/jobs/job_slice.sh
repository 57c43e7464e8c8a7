#!/bin/bash
out=gpurun_out/${OUT:-slice}; mkdir -p $out
BBTC_TRACE=1 timeout 1800 python bench.py --config friendster --no-cpu-baseline --no-ncu --steps 3 --warmup 2 --e2e-steps 1 > $out/bench_friendster.json 2> $out/trace_friendster.log
BBTC_L2_SLICE_MB=0 BBTC_TRACE=1 timeout 1800 python bench.py --config friendster --no-cpu-baseline --no-ncu --steps 3 --warmup 2 --e2e-steps 1 > $out/bench_friendster_noslice.json 2> $out/trace_friendster_noslice.log
timeout 1200 python -m pytest tests -m gpu -q -x -k "full_size or preprocessing or shard" > $out/tests.log 2>&1
echo done >> $out/steps.txt
