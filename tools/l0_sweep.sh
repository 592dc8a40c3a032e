#!/bin/bash
# builds the level-0 size sweep (diagnostics) into tools/bin; run on the GPU box
set -e
cd "$(dirname "$0")"
mkdir -p bin
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -lineinfo \
  -I../include --expt-relaxed-constexpr -o bin/l0_sweep l0_sweep.cu
