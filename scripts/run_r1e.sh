#!/bin/bash
set -x
out=gpurun_out/r1e; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x -k "dense_and_sparse or graph_load or streaming" > $out/gpu_tests.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > $out/bench_rmat24.json 2> $out/bench_rmat24.err
echo done
