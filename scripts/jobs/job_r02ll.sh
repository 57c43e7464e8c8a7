#!/bin/bash
# Final: what the driver runs — smoke, pytest -m gpu, bench.py (defaults), bench.py --impl reference (defaults).
out=gpurun_out/${OUT:-r02ll}; mkdir -p $out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/steps.txt
timeout 2700 python -m pytest tests -x -q -m gpu > $out/gpu_tests.log 2>&1; echo "tests rc=$?" >> $out/steps.txt
s=$(date +%s); timeout 1500 python bench.py > $out/bench_default.json 2> $out/bench_default.err; echo "bench rc=$? $(( $(date +%s) - s ))s" >> $out/steps.txt
s=$(date +%s); timeout 1500 python bench.py --impl reference > $out/ref_default.json 2> $out/ref_default.err; echo "ref rc=$? $(( $(date +%s) - s ))s" >> $out/steps.txt
echo done >> $out/steps.txt
