#!/bin/bash
out=gpurun_out/r1w; mkdir -p $out
for x in 1 2; do
for ips in 24 12 48 96; do
  for cfg in rmat24 orkut; do
    BBTC_ITEMS_PER_SLOT=$ips timeout 300 python scripts/p_sweep.py $cfg $(python -c "import inputs;print(inputs.CONFIGS['$cfg'].p)") | sed "s/^{/{\"v\": \"ips$ips\", /" >> $out/ab.jsonl
  done
done
for c in 4 6 8; do
  BBTC_CTAS_PER_SM=$c timeout 300 python scripts/p_sweep.py rmat24 16 | sed "s/^{/{\"v\": \"ctas$c\", /" >> $out/ab.jsonl
done
done
echo done
