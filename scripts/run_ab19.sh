#!/bin/bash
out=gpurun_out/r1z13; mkdir -p $out
BBTC_LIB=abl/libbbtc_lh.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "rmat16 or random_graphs or karate or dense_rows or huge_part" > $out/gpu_tests.log 2>&1
for x in 1 2; do
for v in cur lh; do
  for cfg in rmat24 orkut friendster; do
    BBTC_LIB=abl/libbbtc_$v.so timeout 300 python scripts/p_sweep.py $cfg $(python -c "import inputs;print(inputs.CONFIGS['$cfg'].p)") | sed "s/^{/{\"v\": \"$v\", /" >> $out/ab.jsonl
  done
done
done
echo done
