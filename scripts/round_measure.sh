#!/bin/bash
# One GPU session producing the round's evidence under gpurun_out/ (copied to profiles/ by hand).
set -x
out=gpurun_out/r1; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu.txt
timeout 600 python bench.py > $out/bench_rmat24.json 2> $out/bench_rmat24.err
timeout 900 python bench.py --config friendster --no-cpu-baseline > $out/bench_friendster.json 2> $out/bench_friendster.err
timeout 600 python bench.py --config orkut --no-cpu-baseline > $out/bench_orkut.json 2> $out/bench_orkut.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_reference.json 2> $out/bench_reference.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_rmat24.csv python scripts/profile_step.py rmat24 > $out/launches_rmat24.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_count -s 1 -c 1 -o $out/prof_rmat24 python scripts/profile_count.py rmat24 > $out/ncu_rmat24.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_count -s 1 -c 1 -o $out/prof_friendster python scripts/profile_count.py friendster > $out/ncu_friendster.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $out/gpu_tests.log 2>&1
echo done
