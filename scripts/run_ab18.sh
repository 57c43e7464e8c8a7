#!/bin/bash
out=gpurun_out/r1z12; mkdir -p $out
for x in 1 2; do
for v in cur d5 d6; do
  BBTC_LIB=abl/libbbtc_$v.so timeout 300 python scripts/p_sweep.py rmat24 12 | sed "s/^{/{\"v\": \"$v\", /" >> $out/ab.jsonl
done
done
echo done
