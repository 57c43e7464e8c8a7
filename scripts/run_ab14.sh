#!/bin/bash
out=gpurun_out/r1z8; mkdir -p $out
BBTC_STREAM_ORDER=peel timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "streaming or dense_and_sparse" > $out/gpu_tests.log 2>&1
for v in greedy peel; do
  for cfg in friendster rmat24 orkut; do
    BBTC_STREAM_ORDER=$v timeout 600 python scripts/stream_probe.py $cfg 2>&1 | grep '"copy_streams": 2' | sed "s/^{/{\"v\": \"$v\", /" >> $out/s.jsonl
  done
done
echo done
