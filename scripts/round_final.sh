#!/bin/bash
# Final confirmation of HEAD: GPU tests, default bench line, smoke, reference arm.
out=gpurun_out/final; mkdir -p $out
timeout 1800 python -m pytest tests -m gpu -q > $out/gpu_tests.log 2>&1
timeout 600 python bench.py > $out/bench_rmat24.json 2> $out/bench_rmat24.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_reference.json 2> $out/bench_reference.err
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1
echo done
