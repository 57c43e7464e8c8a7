#!/bin/bash
out=gpurun_out/${OUT:-r02o}; mkdir -p $out
BBTC_LIB=$PWD/build_ab/dbg/libbbtc.so BBTC_BANDS=1 BBTC_BAND_BYTES=65536 CUDA_LAUNCH_BLOCKING=1 timeout 300 python tests/gpu_child.py rmat:16:16:9 4 resident > $out/bands_dbg.log 2>&1; echo "bands rc=$?" >> $out/steps.txt
timeout 900 scripts/micro/sorttune > $out/sorttune.log 2>&1; echo "sorttune rc=$?" >> $out/steps.txt
echo done >> $out/steps.txt
