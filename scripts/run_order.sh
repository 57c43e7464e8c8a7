#!/bin/bash
out=gpurun_out/r1h; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x -k "dense_and_sparse or streaming or out_of_core" > $out/gpu_tests.log 2>&1
for cfg in rmat24 friendster; do
for o in greedy exec; do
  BBTC_STREAM_ORDER=$o timeout 600 python scripts/stream_probe.py $cfg 2>&1 | grep '"copy_streams": 2' | sed "s/^/{\"order\": \"$o\"} /" >> $out/order_$cfg.jsonl
done
done
