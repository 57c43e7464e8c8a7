#!/bin/bash
out=gpurun_out/r1z14; mkdir -p $out
for v in perbyte abs; do
  for cfg in friendster rmat24 orkut; do
    if [ $v = abs ]; then export BBTC_PEEL_ABS=1; else unset BBTC_PEEL_ABS; fi
    timeout 600 python scripts/stream_probe.py $cfg 2>&1 | grep '"copy_streams": 2' | sed "s/^{/{\"v\": \"$v\", /" >> $out/s.jsonl
  done
done
echo done
