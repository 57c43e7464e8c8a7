#!/bin/bash
# HEAD check on a B200: smoke, default bench line, GPU tests, launch list of one bench step.
out=gpurun_out/${OUT:-r02a}; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
timeout 900 python bench.py > $out/bench_rmat24.json 2> $out/bench_rmat24.err
timeout 1500 python -m pytest tests -m gpu -q -x > $out/gpu_tests.log 2>&1
echo done
