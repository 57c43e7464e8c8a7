#!/bin/bash
out=gpurun_out/r1z7; mkdir -p $out
BBTC_LIB=abl/libbbtc_ver.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "streaming or dense_and_sparse or out_of_core" > $out/gpu_tests.log 2>&1
for v in cur ver; do
  for cfg in friendster rmat24; do
    BBTC_LIB=abl/libbbtc_$v.so timeout 600 python scripts/stream_probe.py $cfg 2>&1 | grep '"copy_streams": 2' | sed "s/^{/{\"v\": \"$v\", /" >> $out/s.jsonl
  done
  BBTC_LIB=abl/libbbtc_$v.so timeout 300 python scripts/p_sweep.py rmat24 16 | sed "s/^{/{\"v\": \"$v\", /" >> $out/ab.jsonl
done
echo done
