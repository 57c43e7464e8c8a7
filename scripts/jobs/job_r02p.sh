#!/bin/bash
out=gpurun_out/${OUT:-r02p}; mkdir -p $out
BBTC_LIB=$PWD/build_ab/dbg/libbbtc.so BBTC_BANDS=1 BBTC_BAND_BYTES=65536 CUDA_LAUNCH_BLOCKING=1 timeout 300 python tests/gpu_child.py rmat:16:16:9 4 resident > $out/bands_dbg.log 2>&1; echo "bands rc=$?" >> $out/steps.txt
BBTC_TRACE=1 timeout 600 python scripts/trace_prep.py rmat24 10 5 > $out/trace_rmat24.log 2>&1
BBTC_TRACE=1 BBTC_CUB_STOCK=1 timeout 600 python scripts/trace_prep.py rmat24 10 5 > $out/trace_rmat24_stock.log 2>&1
BBTC_TRACE=1 timeout 900 python scripts/trace_prep.py friendster 4 2 > $out/trace_friendster.log 2>&1
BBTC_TRACE=1 BBTC_CUB_STOCK=1 timeout 900 python scripts/trace_prep.py friendster 4 2 > $out/trace_friendster_stock.log 2>&1
echo "trace rc=$?" >> $out/steps.txt
timeout 1200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-ncu > $out/bench_rmat24.json 2> $out/bench_rmat24.err; echo "bench rc=$?" >> $out/steps.txt
echo done >> $out/steps.txt
