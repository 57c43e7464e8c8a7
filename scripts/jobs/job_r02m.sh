#!/bin/bash
# Bands with the lane-prefix fix (test + friendster A/B), hash bucket width A/B.
out=gpurun_out/${OUT:-r02m}; mkdir -p $out
BBTC_BANDS=1 BBTC_BAND_BYTES=65536 CUDA_LAUNCH_BLOCKING=1 timeout 300 python tests/gpu_child.py rmat:16:16:9 4 resident > $out/bands_blocking.log 2>&1; echo "bands rc=$?" >> $out/steps.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "bands" > $out/test_bands.log 2>&1; echo "test rc=$?" >> $out/steps.txt
timeout 3000 python scripts/ab_variants.py friendster,rmat24:10,orkut paper_2009_12457_b200/libbbtc.so build_ab/bw2/libbbtc.so build_ab/bw1/libbbtc.so "env:BBTC_BANDS=cost;BBTC_BAND_BYTES=64e6" "env:BBTC_BANDS=1;BBTC_BAND_BYTES=64e6" "env:BBTC_BANDS=cost;BBTC_BAND_BYTES=32e6;BBTC_BAND_RATIO=1" > $out/ab.jsonl 2>> $out/err.txt
echo done >> $out/steps.txt
