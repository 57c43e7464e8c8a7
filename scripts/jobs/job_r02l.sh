#!/bin/bash
# Bands-crash bisect over library builds; A/B of phase-1 depth / rolling prefetch; friendster per-task times.
out=gpurun_out/${OUT:-r02l}; mkdir -p $out
B="BBTC_BANDS=1 BBTC_BAND_BYTES=65536 CUDA_LAUNCH_BLOCKING=1"
for v in bis_f80c68e bis_2a437ff bis_8e1bf6a bis_ec6a2e9 bis_8a14f4a bis_6a4db70 bis_b277141 r02h; do
  env $B BBTC_LIB=$PWD/build_ab/$v/libbbtc.so timeout 300 python tests/gpu_child.py rmat:16:16:9 4 resident > $out/bis_$v.log 2>&1; echo "$v rc=$?" >> $out/steps.txt
done
env $B BBTC_DENSE_WALK=col BBTC_LIB=$PWD/build_ab/r02h/libbbtc.so timeout 300 python tests/gpu_child.py rmat:16:16:9 4 resident > $out/r02h_densecol.log 2>&1; echo "r02h densecol rc=$?" >> $out/steps.txt
timeout 2400 python scripts/ab_variants.py friendster,rmat24:10,orkut paper_2009_12457_b200/libbbtc.so build_ab/pfnext/libbbtc.so build_ab/d8/libbbtc.so build_ab/pfd8/libbbtc.so > $out/ab.jsonl 2>> $out/err.txt
echo "ab rc=$?" >> $out/steps.txt
timeout 1500 python scripts/study_f4.py estim friendster 4 > $out/estim_friendster_p4.jsonl 2>> $out/err.txt
echo done >> $out/steps.txt
