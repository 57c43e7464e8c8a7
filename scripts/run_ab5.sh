#!/bin/bash
out=gpurun_out/r1r; mkdir -p $out
for x in 1 2; do
for db in 2048 0 1024 4096; do
  BBTC_DENSE_BITS=$db timeout 300 python scripts/p_sweep.py rmat24 16 | sed "s/^{/{\"v\": \"dense$db\", /" >> $out/ab.jsonl
done
done
echo done
