#!/bin/bash
# Raw-edge H2D on two copy streams (BBTC_H2D_STREAMS=2): e2e A/B + host-input parity.
out=gpurun_out/${OUT:-r02kk}; mkdir -p $out
BBTC_H2D_STREAMS=2 timeout 1200 python -m pytest tests -q -m gpu -k "host or pairs or mapped or load or smoke or e2e" > $out/tests_2s.log 2>&1; echo "tests rc=$?" >> $out/steps.txt
for r in 1 2; do
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-ncu --e2e-steps 7 > $out/bench_1s_$r.json 2>> $out/err.txt
BBTC_H2D_STREAMS=2 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-ncu --e2e-steps 7 > $out/bench_2s_$r.json 2>> $out/err.txt
done
echo done >> $out/steps.txt
