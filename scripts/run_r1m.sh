#!/bin/bash
out=gpurun_out/r1m; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x -k "dense_and_sparse or streaming or out_of_core or graph_load" > $out/gpu_tests_quick.log 2>&1
timeout 600 python scripts/stream_probe.py rmat24 2>&1 | grep '"copy_streams": 2' >> $out/stream_rmat24.jsonl
timeout 600 python scripts/ooc_sweep.py rmat24 0.25 0.5 0.75 >> $out/ooc_rmat24.jsonl 2>&1
timeout 900 python scripts/stream_probe.py friendster 2>&1 | grep '"copy_streams": 2' >> $out/stream_friendster.jsonl
