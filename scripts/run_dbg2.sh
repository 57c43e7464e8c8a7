#!/bin/bash
out=gpurun_out/dbg2; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "packed or rmat16 or dense_and_sparse or streaming or out_of_core or auto_p" > $out/gpu_tests.log 2>&1
timeout 300 python scripts/stream_probe.py rmat24 > $out/s_rmat24.jsonl 2> $out/s_rmat24.err
timeout 600 python scripts/stream_probe.py friendster > $out/s_friendster.jsonl 2> $out/s_friendster.err
echo done
