#!/bin/bash
out=gpurun_out/r1q; mkdir -p $out
for x in 1 2; do
for v in bm2 ml2 ml8; do
  for cfg in rmat24 orkut; do
    BBTC_LIB=abl/libbbtc_$v.so timeout 300 python scripts/p_sweep.py $cfg $(python -c "import inputs;print(inputs.CONFIGS['$cfg'].p)") | sed "s/^{/{\"v\": \"$v\", /" >> $out/ab.jsonl
  done
done
for r in 2 4; do
  BBTC_DENSE_RATIO=$r BBTC_LIB=abl/libbbtc_bm2.so timeout 300 python scripts/p_sweep.py rmat24 16 | sed "s/^{/{\"v\": \"bm2-ratio$r\", /" >> $out/ab.jsonl
done
done
echo done
