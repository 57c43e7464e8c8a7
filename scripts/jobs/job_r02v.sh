#!/bin/bash
# HEAD check after the A/B code removals: GPU tests (incl. 5-rank sharded build), smoke, rmat24 bench.
out=gpurun_out/${OUT:-r02v}; mkdir -p $out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/steps.txt
timeout 2700 python -m pytest tests -m gpu -q > $out/gpu_tests.log 2>&1; echo "tests rc=$?" >> $out/steps.txt
timeout 1200 python bench.py --steps 20 --warmup 5 > $out/bench_rmat24.json 2> $out/bench_rmat24.err; echo "bench rc=$?" >> $out/steps.txt
echo done >> $out/steps.txt
