out=gpurun_out/r1c; mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_count_dense -s 1 -c 1 -o $out/prof_dense_rmat24 python scripts/profile_count.py rmat24 > $out/ncu_dense_rmat24.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_count -s 2 -c 2 -o $out/prof_both_rmat24 python scripts/profile_count.py rmat24 > $out/ncu_both_rmat24.log 2>&1
timeout 600 python bench.py > $out/bench_rmat24.json 2> $out/bench_rmat24.err
timeout 1800 python -m pytest tests -m gpu -q -x > $out/gpu_tests.log 2>&1
echo done
