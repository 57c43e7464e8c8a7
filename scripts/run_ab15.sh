#!/bin/bash
out=gpurun_out/r1z9; mkdir -p $out
for db in 2048 4096 8192; do
for r in 4 8; do
  BBTC_DENSE_BITS=$db BBTC_DENSE_RATIO=$r timeout 300 python scripts/p_sweep.py rmat24 16 | sed "s/^{/{\"v\": \"db$db-r$r\", /" >> $out/ab.jsonl
done
done
for ips in 256 384 768; do
  BBTC_ITEMS_PER_SLOT=$ips timeout 300 python scripts/p_sweep.py rmat24 16 | sed "s/^{/{\"v\": \"ips$ips\", /" >> $out/ab.jsonl
done
echo done
