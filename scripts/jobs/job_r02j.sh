#!/bin/bash
# Band-option crash under memcheck; A/B of the L2 fetch granularity and cost-ruled bands.
out=gpurun_out/${OUT:-r02j}; mkdir -p $out
BBTC_BANDS=1 BBTC_BAND_BYTES=65536 timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python tests/gpu_child.py rmat:16:16:9 4 resident > $out/memcheck_bands.log 2>&1
echo "memcheck rc=$?" >> $out/steps.txt
BBTC_BANDS=1 BBTC_BAND_BYTES=65536 CUDA_LAUNCH_BLOCKING=1 timeout 600 python tests/gpu_child.py rmat:16:16:9 4 resident > $out/bands_blocking.log 2>&1
echo "blocking rc=$?" >> $out/steps.txt
timeout 2400 python scripts/ab_variants.py friendster,rmat24:10 paper_2009_12457_b200/libbbtc.so env:BBTC_L2_FETCH=32 env:BBTC_L2_FETCH=128 "env:BBTC_BANDS=cost;BBTC_TRACE=1" "env:BBTC_BANDS=cost;BBTC_BAND_BYTES=64e6" > $out/ab.jsonl 2>> $out/err.txt
echo done >> $out/steps.txt
