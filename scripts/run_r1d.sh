#!/bin/bash
# Re-entry check of HEAD: bench lines, prep trace, GPU tests.
set -x
out=gpurun_out/r1d; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu.txt
timeout 600 python bench.py > $out/bench_rmat24.json 2> $out/bench_rmat24.err
BBTC_TRACE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $out/trace_rmat24.json 2> $out/trace_rmat24.err
BBTC_TRACE=1 timeout 900 python bench.py --config friendster --no-cpu-baseline > $out/bench_friendster.json 2> $out/bench_friendster.err
timeout 1800 python -m pytest tests -m gpu -q -x > $out/gpu_tests.log 2>&1
echo done
