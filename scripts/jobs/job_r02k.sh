#!/bin/bash
# Bands crash bisect (HEAD with launch locations, r02h build, env toggles); prep traces; friendster band decisions.
out=gpurun_out/${OUT:-r02k}; mkdir -p $out
B="BBTC_BANDS=1 BBTC_BAND_BYTES=65536 CUDA_LAUNCH_BLOCKING=1"
env $B timeout 300 python tests/gpu_child.py rmat:16:16:9 4 resident > $out/head.log 2>&1; echo "head rc=$?" >> $out/steps.txt
env $B BBTC_LIB=$PWD/build_ab/r02h/libbbtc.so timeout 300 python tests/gpu_child.py rmat:16:16:9 4 resident > $out/r02h.log 2>&1; echo "r02h rc=$?" >> $out/steps.txt
env $B BBTC_DENSE_WALK=col timeout 300 python tests/gpu_child.py rmat:16:16:9 4 resident > $out/densecol.log 2>&1; echo "densecol rc=$?" >> $out/steps.txt
env $B BBTC_DENSE_BITS=1 timeout 300 python tests/gpu_child.py rmat:16:16:9 4 resident > $out/nodense.log 2>&1; echo "nodense rc=$?" >> $out/steps.txt
BBTC_TRACE=1 timeout 600 python scripts/trace_prep.py rmat24 10 5 > $out/trace_rmat24.log 2>&1; echo "trace rc=$?" >> $out/steps.txt
BBTC_TRACE=1 timeout 900 python scripts/trace_prep.py orkut 8 5 > $out/trace_orkut.log 2>&1
BBTC_TRACE=1 BBTC_BANDS=cost BBTC_BAND_BYTES=64e6 timeout 1200 python scripts/trace_prep.py friendster 4 1 > $out/trace_friendster_bands.log 2>&1; echo "trace2 rc=$?" >> $out/steps.txt
echo done >> $out/steps.txt
