#!/bin/bash
# Build an A/B variant of the library with a different gemm_tc.cu (or -D flags) into build/variants/<name>.so
# usage: tools/build_variant.sh <name> <gemm_tc.cu path> [nvcc -D flags...]
set -e
name=$1; src=$2; shift 2
mkdir -p build/variants
objs=$(ls build/obj/*.o | grep -v gemm_tc)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -Ipaper_2604_10152_b200/csrc "$@" -c "$src" -o build/variants/$name.gemm_tc.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/$name.so \
  $objs build/variants/$name.gemm_tc.o -lcudart_static -ldl -lpthread -lrt
