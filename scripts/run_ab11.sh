#!/bin/bash
out=gpurun_out/r1z4; mkdir -p $out
for x in 1 2; do
for r in 4 8 16 32; do
  BBTC_DENSE_RATIO=$r timeout 300 python scripts/p_sweep.py rmat24 12 16 | sed "s/^{/{\"v\": \"ratio$r\", /" >> $out/ab.jsonl
done
done
echo done
