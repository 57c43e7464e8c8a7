#!/bin/bash
out=gpurun_out/r1z15; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py -q -x -k "streaming or dense_and_sparse or out_of_core or auto_p or two_ranks" > $out/gpu_tests.log 2>&1
for v in first last; do
  for cfg in rmat24 orkut; do
    if [ $v = last ]; then export BBTC_DENSE_LAST=1; else unset BBTC_DENSE_LAST; fi
    timeout 600 python scripts/stream_probe.py $cfg 2>&1 | grep '"copy_streams": 2' | sed "s/^{/{\"v\": \"$v\", /" >> $out/s.jsonl
  done
done
echo done
