#!/bin/bash
# Bit-row kernel: loads past a row's live part skipped (BBTC_DENSE_LIVE) — parity + A/B (+ dense ratio re-check).
out=gpurun_out/${OUT:-r02u}; mkdir -p $out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "dense or karate or rmat16 or probe_slots" > $out/tests_dense.log 2>&1; echo "tests rc=$?" >> $out/steps.txt
timeout 2400 python scripts/ab_variants.py rmat24:10,rmat24:12,orkut paper_2009_12457_b200/libbbtc.so build_ab/nolive/libbbtc.so "env:BBTC_DENSE_RATIO=3" "env:BBTC_DENSE_RATIO=2" > $out/ab.jsonl 2>> $out/err.txt
echo done >> $out/steps.txt
