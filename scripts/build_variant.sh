#!/bin/bash
# Build an A/B variant of libbbtc.so with extra nvcc defines into build_ab/<name>/libbbtc.so
#   scripts/build_variant.sh min6 -DBBTC_MIN_CTAS=6
name=$1; shift
out=build_ab/$name; mkdir -p $out
NV="/usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-fvisibility=hidden -Iinclude --expt-relaxed-constexpr"
C=paper_2009_12457_b200/csrc
$NV "$@" -c $C/count.cu -o $out/count.o -Xptxas -v 2> $out/count.ptxas.txt &
$NV "$@" -c $C/prep.cu -o $out/prep.o &
$NV "$@" -x cu -c $C/capi.cpp -o $out/capi.o &
$NV "$@" -x cu -c $C/io.cpp -o $out/io.o &
$NV "$@" -x cu -c $C/cpu.cpp -o $out/cpu.o &
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libbbtc.so $out/capi.o $out/io.o $out/cpu.o $out/prep.o $out/count.o -cudart static -lpthread
rm -f $out/*.o
echo $out/libbbtc.so
