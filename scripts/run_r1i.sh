#!/bin/bash
out=gpurun_out/r1i; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x -k "dense_and_sparse or streaming or out_of_core or graph_load" > $out/gpu_tests_quick.log 2>&1
for cfg in rmat24 friendster; do
  timeout 600 python scripts/stream_probe.py $cfg 2>&1 | grep '"copy_streams": 2' >> $out/stream_$cfg.jsonl
done
timeout 1800 python -m pytest tests -m gpu -q -x > $out/gpu_tests.log 2>&1
