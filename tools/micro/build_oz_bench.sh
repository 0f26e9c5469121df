#!/bin/bash
# Builds tools/micro/oz_bench against the in-tree library.
cd "$(dirname "$0")"
C=../../paper_2408_04440_b200/csrc
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -I$C -I../../include \
  -o oz_bench oz_bench.cu -L../../paper_2408_04440_b200/lib -lsphemu_gpu -lcuda \
  -Xlinker -rpath='$ORIGIN/../../paper_2408_04440_b200/lib'
