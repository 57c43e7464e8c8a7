#!/bin/bash
# Next-batch edge-id prefetch in the hash-only variant (BBTC_EDGE_PF) — friendster A/B + parity subset.
out=gpurun_out/${OUT:-r02z}; mkdir -p $out
BBTC_LIB=$PWD/build_ab/edgepf/libbbtc.so timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "not full_size and not counting and not bucket" > $out/tests_edgepf.log 2>&1; echo "tests rc=$?" >> $out/steps.txt
timeout 2400 python scripts/ab_variants.py friendster paper_2009_12457_b200/libbbtc.so build_ab/edgepf/libbbtc.so paper_2009_12457_b200/libbbtc.so build_ab/edgepf/libbbtc.so > $out/ab.jsonl 2>> $out/err.txt
echo done >> $out/steps.txt
