#!/bin/bash
out=gpurun_out/r1z3; mkdir -p $out
for x in 1 2; do
for v in cur nopf; do
  BBTC_LIB=abl/libbbtc_$v.so timeout 300 python scripts/p_sweep.py friendster 4 | sed "s/^{/{\"v\": \"$v\", /" >> $out/ab.jsonl
  BBTC_DENSE_RATIO=2 BBTC_LIB=abl/libbbtc_$v.so timeout 300 python scripts/p_sweep.py rmat24 12 16 | sed "s/^{/{\"v\": \"$v-ratio2\", /" >> $out/ab.jsonl
  BBTC_DENSE_RATIO=4 BBTC_LIB=abl/libbbtc_$v.so timeout 300 python scripts/p_sweep.py rmat24 16 | sed "s/^{/{\"v\": \"$v-ratio4\", /" >> $out/ab.jsonl
done
done
echo done
