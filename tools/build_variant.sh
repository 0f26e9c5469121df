#!/bin/bash
# Builds a variant of the library with extra nvcc defines for tc_gemm.cu:
#   tools/build_variant.sh NAME -DSPH_TC_RING2=4 ...   -> variants/NAME/libsphemu_gpu.so
set -e
cd "$(dirname "$0")/../paper_2408_04440_b200/csrc"
name=$1; shift
NCCL_DIR=$(python3 -c "import nvidia.nccl as m; print(list(m.__path__)[0])")
out=../../variants/$name
mkdir -p $out
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr \
  -I../../include -I$NCCL_DIR/include "$@" -c tc_gemm.cu -o $out/tc_gemm.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libsphemu_gpu.so ../lib/obj/chol.o $out/tc_gemm.o \
  ../lib/obj/sht.o ../lib/obj/emulate.o -lcudart -lcuda -L$NCCL_DIR/lib -l:libnccl.so.2 -Xlinker --disable-new-dtags \
  -Xlinker -rpath=$NCCL_DIR/lib
echo "built $out/libsphemu_gpu.so"
