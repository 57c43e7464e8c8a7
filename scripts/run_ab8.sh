#!/bin/bash
out=gpurun_out/r1x; mkdir -p $out
for ips in 96 192 384 768 1536; do
  for cfg in rmat24 orkut friendster; do
    BBTC_ITEMS_PER_SLOT=$ips timeout 300 python scripts/p_sweep.py $cfg $(python -c "import inputs;print(inputs.CONFIGS['$cfg'].p)") | sed "s/^{/{\"v\": \"ips$ips\", /" >> $out/ab.jsonl
  done
done
echo done
