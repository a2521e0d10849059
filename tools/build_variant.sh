#!/bin/bash
# Build an A/B variant of the library with one .cu file replaced (or rebuilt with -D flags) into build/variants/<name>.so
# usage: tools/build_variant.sh <name> <path of the .cu to swap in> [nvcc -D flags...]
set -e
name=$1; src=$2; shift 2
mkdir -p build/variants
base=$(basename $src .cu); objs=$(ls build/obj/*.o | grep -v "/$base\.")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -Ipaper_2604_10152_b200/csrc "$@" -c "$src" -o build/variants/$name.$base.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/$name.so \
  $objs build/variants/$name.$base.o -lcudart_static -ldl -lpthread -lrt
