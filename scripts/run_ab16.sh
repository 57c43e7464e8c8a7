#!/bin/bash
out=gpurun_out/r1z10; mkdir -p $out
BBTC_DENSE_BITS=16384 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "dense" > $out/gpu_tests.log 2>&1
for db in 8192 16384; do
for r in 2 3 4 6; do
  BBTC_DENSE_BITS=$db BBTC_DENSE_RATIO=$r timeout 300 python scripts/p_sweep.py rmat24 16 12 | sed "s/^{/{\"v\": \"db$db-r$r\", /" >> $out/ab.jsonl
done
done
echo done
