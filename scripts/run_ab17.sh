#!/bin/bash
out=gpurun_out/r1z11; mkdir -p $out
for db in 2048 8192; do
  BBTC_DENSE_BITS=$db timeout 300 python scripts/p_sweep.py orkut 8 4 | sed "s/^{/{\"v\": \"db$db\", /" >> $out/ab.jsonl
done
timeout 300 python scripts/p_sweep.py rmat24 12 14 16 | sed "s/^{/{\"v\": \"default\", /" >> $out/ab.jsonl
timeout 300 python scripts/p_sweep.py rmat16 4 8 16 | sed "s/^{/{\"v\": \"default\", /" >> $out/ab.jsonl
echo done
