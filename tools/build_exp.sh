#!/bin/sh
# Timing-experiment builds of libedak (wrong results by design): $1 = flags
set -e
cd "$(dirname "$0")/.."
OUT=build/exp_$2
mkdir -p $OUT
for f in capi l96 l96_ops sweep_tile circ circ_os blas lmp_gemm small cholinv jacobi_cluster pcg pcg_small peak; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC $1 -c paper_2605_23571_b200/csrc/$f.cu -o $OUT/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libedak.so $OUT/*.o -lcudart
