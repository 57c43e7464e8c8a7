#!/bin/bash
# Phase 1 unified predicated round (BBTC_P1_UNIFIED) — parity + A/B against the previous loop.
out=gpurun_out/${OUT:-r02w}; mkdir -p $out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "not full_size" > $out/tests.log 2>&1; echo "tests rc=$?" >> $out/steps.txt
timeout 3000 python scripts/ab_variants.py rmat24:10,orkut,friendster paper_2009_12457_b200/libbbtc.so build_ab/p1old/libbbtc.so > $out/ab.jsonl 2>> $out/err.txt
echo done >> $out/steps.txt
