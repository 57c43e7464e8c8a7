#!/bin/bash
# Evidence after the bitmap change: ncu of both count kernels (rmat24), bench lines, GPU tests.
set -x
out=gpurun_out/r1s; mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_count -s 0 -c 2 -o $out/prof_rmat24 python scripts/profile_count.py rmat24 > $out/ncu_rmat24.log 2>&1
timeout 600 python bench.py > $out/bench_rmat24.json 2> $out/bench_rmat24.err
timeout 600 python bench.py --config orkut --no-cpu-baseline > $out/bench_orkut.json 2> $out/bench_orkut.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_rmat24.csv python scripts/profile_step.py rmat24 > $out/launches_rmat24.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $out/gpu_tests.log 2>&1
echo done
