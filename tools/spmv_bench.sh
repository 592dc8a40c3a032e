#!/bin/bash
# builds and runs the level-0 SpMV microbenchmark (diagnostics)
set -e
cd "$(dirname "$0")"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -lineinfo \
  -I../include --expt-relaxed-constexpr -o /tmp/spmv_bench spmv_bench.cu
/tmp/spmv_bench "$@"
