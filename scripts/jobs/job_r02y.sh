#!/bin/bash
# Evidence at HEAD (round 2 final): smoke, bench lines (rmat24 with in-run ncu + oracle baseline, orkut,
# friendster), reference arm, GPU tests, ncu --set full of both count kernels, launch list.
out=gpurun_out/${OUT:-r02y}; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $out/gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/steps.txt
timeout 1200 python bench.py --steps 20 --warmup 5 > $out/bench_rmat24.json 2> $out/bench_rmat24.err; echo "bench rc=$?" >> $out/steps.txt
timeout 1200 python bench.py --config orkut > $out/bench_orkut.json 2> $out/bench_orkut.err
timeout 2400 python bench.py --config friendster --no-cpu-baseline --steps 5 --warmup 3 > $out/bench_friendster.json 2> $out/bench_friendster.err; echo "benches rc=$?" >> $out/steps.txt
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $out/ref_rmat24.json 2> $out/ref.err; echo "ref rc=$?" >> $out/steps.txt
timeout 2700 python -m pytest tests -m gpu -q > $out/gpu_tests.log 2>&1; echo "tests rc=$?" >> $out/steps.txt
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'^k_count$' -s 1 -c 1 -o $out/prof_list_rmat24 python scripts/profile_count.py rmat24 > $out/ncu_list.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_count_dense' -s 1 -c 1 -o $out/prof_dense_rmat24 python scripts/profile_count.py rmat24 > $out/ncu_dense.log 2>&1
timeout 2400 ncu --set full --clock-control none -k regex:'^k_count$' -s 1 -c 1 -o $out/prof_list_friendster python scripts/profile_count.py friendster > $out/ncu_friendster.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $out/launches_rmat24.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-ncu --e2e-steps 1 > $out/launches.log 2>&1; echo "ncu rc=$?" >> $out/steps.txt
echo done >> $out/steps.txt
