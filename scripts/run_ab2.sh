#!/bin/bash
# A/B of count-kernel builds (BBTC_LIB) on rmat24 and orkut: count time per variant.
out=gpurun_out/r1l; mkdir -p $out
for x in 1 2; do
for v in base pf; do
  for cfg in rmat24 orkut; do
    BBTC_LIB=abl/libbbtc_$v.so timeout 300 python scripts/p_sweep.py $cfg $(python -c "import inputs;print(inputs.CONFIGS['$cfg'].p)") | sed "s/^{/{\"v\": \"$v\", /" >> $out/ab.jsonl
  done
done
done
echo done
