# A/B: p_sweep on rmat24 with the old library, the new one, and the new one without bitmaps
for x in 1 2; do
BBTC_LIB=abl/libbbtc_old.so timeout 300 python scripts/p_sweep.py rmat24 16 | sed 's/^{/{"v": "old", /' >> gpurun_out/ab_bitmap.jsonl
timeout 300 python scripts/p_sweep.py rmat24 16 | sed 's/^{/{"v": "new", /' >> gpurun_out/ab_bitmap.jsonl
BBTC_NO_BITMAP=1 timeout 300 python scripts/p_sweep.py rmat24 16 | sed 's/^{/{"v": "new-nobitmap", /' >> gpurun_out/ab_bitmap.jsonl
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "rmat16 or dense or random_graphs or karate or many_parts" > gpurun_out/ab_tests.log 2>&1
echo done
