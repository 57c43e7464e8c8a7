#!/bin/bash
# Evidence after the work-item change: GPU tests, bench lines, ncu of the list kernel, launch list.
set -x
out=gpurun_out/r1y; mkdir -p $out
timeout 1800 python -m pytest tests -m gpu -q > $out/gpu_tests.log 2>&1
timeout 600 python bench.py > $out/bench_rmat24.json 2> $out/bench_rmat24.err
timeout 600 python bench.py --config orkut --no-cpu-baseline > $out/bench_orkut.json 2> $out/bench_orkut.err
timeout 900 python bench.py --config friendster --no-cpu-baseline > $out/bench_friendster.json 2> $out/bench_friendster.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_count -s 0 -c 1 -o $out/prof_list_rmat24 python scripts/profile_count.py rmat24 > $out/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_count_dense -s 0 -c 1 -o $out/prof_dense_rmat24 python scripts/profile_count.py rmat24 > $out/ncu_dense.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_rmat24.csv python scripts/profile_step.py rmat24 > $out/launches_rmat24.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
echo done
