#!/bin/bash
out=gpurun_out/r1n; mkdir -p $out
timeout 600 python -m pytest tests -m gpu -q -x -k "auto_p or graph_load" > $out/gpu_tests.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > $out/bench_rmat24.json 2> $out/bench_rmat24.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_count -s 0 -c 1 -o $out/prof_list_orkut python scripts/profile_count.py orkut > $out/ncu_orkut.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_count -s 0 -c 1 -o $out/prof_list_friendster python scripts/profile_count.py friendster > $out/ncu_friendster.log 2>&1
ls -la $out
