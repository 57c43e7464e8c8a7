#!/bin/bash
# Round-1 closing evidence (after the streaming work): bench lines, launch list, GPU tests.
set -x
out=gpurun_out/r1z; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu.txt
timeout 600 python bench.py > $out/bench_rmat24.json 2> $out/bench_rmat24.err
timeout 900 python bench.py --config friendster --no-cpu-baseline > $out/bench_friendster.json 2> $out/bench_friendster.err
timeout 600 python bench.py --config orkut --no-cpu-baseline > $out/bench_orkut.json 2> $out/bench_orkut.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_reference.json 2> $out/bench_reference.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_rmat24.csv python scripts/profile_step.py rmat24 > $out/launches_rmat24.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $out/gpu_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
echo done
