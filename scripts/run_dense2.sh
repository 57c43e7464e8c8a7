for r in 0 0.5 1 2 4; do
  BBTC_DENSE_RATIO=$r timeout 300 python scripts/dense_sweep.py rmat24 16 2048,4096 | sed "s/^{/{\"ratio\": $r, /" >> gpurun_out/dense2_rmat24.jsonl
done
for p in 12 20 24 28 32; do
  timeout 400 python scripts/dense_sweep.py rmat24 $p 0,2048,4096 >> gpurun_out/dense2_rmat24.jsonl
done
echo done
