#!/bin/bash
# Source-level ncu capture of the list kernel (k_count<1,1>) on rmat24.
out=gpurun_out/r1k; mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_count -s 0 -c 1 -o $out/prof_list_rmat24 python scripts/profile_count.py rmat24 > $out/ncu_list.log 2>&1
ncu -i $out/prof_list_rmat24.ncu-rep --page source --csv --print-source cuda > $out/src_cuda.csv 2> $out/src_cuda.err
ncu -i $out/prof_list_rmat24.ncu-rep --page details --csv > $out/details.csv 2>&1
ls -la $out
