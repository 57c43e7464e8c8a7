#!/bin/bash
out=gpurun_out/${OUT:-ab5}; mkdir -p $out
timeout 2400 python scripts/ab_variants.py rmat24:10,orkut,friendster paper_2009_12457_b200/libbbtc.so build_ab/lw2/libbbtc.so build_ab/lw3/libbbtc.so build_ab/lwall/libbbtc.so build_ab/rpbm/libbbtc.so > $out/ab_kernel.jsonl 2>> $out/err.txt
for ips in 192 768; do BBTC_ITEMS_PER_SLOT=$ips timeout 900 python scripts/ab_variants.py rmat24:10,orkut paper_2009_12457_b200/libbbtc.so | sed "s/^{/{\"items_per_slot\": $ips, /" >> $out/ab_items.jsonl 2>> $out/err.txt; done
echo done >> $out/steps.txt
BBTC_DENSE_NOKEEP=1 timeout 900 python scripts/ab_variants.py rmat24:10,rmat24:12,orkut paper_2009_12457_b200/libbbtc.so > $out/ab_dense_nokeep.jsonl 2>> $out/err.txt
timeout 900 python scripts/ab_variants.py rmat24:10,rmat24:12,orkut paper_2009_12457_b200/libbbtc.so > $out/ab_dense_keep.jsonl 2>> $out/err.txt
timeout 1200 python -m pytest tests -m gpu -q -x -k "dense or karate or rmat16_p_grid or full_size or row_bands" > $out/tests.log 2>&1
echo done2 >> $out/steps.txt
for bb in 16e6 32e6 64e6; do BBTC_BANDS=1 BBTC_BAND_BYTES=$bb timeout 1500 python scripts/ab_variants.py friendster,orkut paper_2009_12457_b200/libbbtc.so | sed "s/^{/{\"band_bytes\": $bb, /" >> $out/ab_bands.jsonl 2>> $out/err.txt; done
timeout 900 python -m pytest tests -m gpu -q -x -k "row_bands" > $out/tests_bands.log 2>&1
echo done3 >> $out/steps.txt
