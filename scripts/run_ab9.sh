#!/bin/bash
out=gpurun_out/r1z2; mkdir -p $out
for x in 1 2; do
for v in cur pbm nopf; do
  for cfg in rmat24 orkut; do
    BBTC_LIB=abl/libbbtc_$v.so timeout 300 python scripts/p_sweep.py $cfg $(python -c "import inputs;print(inputs.CONFIGS['$cfg'].p)") | sed "s/^{/{\"v\": \"$v\", /" >> $out/ab.jsonl
  done
done
for db in 1024 4096; do
  BBTC_DENSE_BITS=$db timeout 300 python scripts/p_sweep.py rmat24 16 | sed "s/^{/{\"v\": \"dense$db\", /" >> $out/ab.jsonl
done
for r in 0.5 2; do
  BBTC_DENSE_RATIO=$r timeout 300 python scripts/p_sweep.py rmat24 16 | sed "s/^{/{\"v\": \"ratio$r\", /" >> $out/ab.jsonl
done
done
timeout 600 python scripts/p_sweep.py rmat24 12 20 24 | sed "s/^{/{\"v\": \"psweep\", /" >> $out/ab.jsonl
echo done
