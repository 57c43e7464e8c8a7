#!/bin/bash
out=gpurun_out/r1z16; mkdir -p $out
for x in 1 2; do
for ips in 384 768 1536; do
  for cfg in rmat24 orkut; do
    BBTC_ITEMS_PER_SLOT=$ips timeout 300 python scripts/p_sweep.py $cfg $(python -c "import inputs;print(inputs.CONFIGS['$cfg'].p)") | sed "s/^{/{\"v\": \"ips$ips\", /" >> $out/ab.jsonl
  done
done
done
echo done
