#!/bin/bash
# Build an A/B variant of the library with .cu files replaced (or rebuilt with -D flags) into build/variants/<name>.so
# usage: tools/build_variant.sh <name> "<path of a .cu to swap in> [more .cu paths]" [nvcc -D flags...]
set -e
name=$1; srcs=$2; shift 2
mkdir -p build/variants
objs=$(ls build/obj/*.o)
vobjs=""
for src in $srcs; do
  base=$(basename $src .cu); objs=$(echo "$objs" | grep -v "/$base\.")
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -Ipaper_2604_10152_b200/csrc "$@" -c "$src" -o build/variants/$name.$base.o
  vobjs="$vobjs build/variants/$name.$base.o"
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/$name.so \
  $objs $vobjs -lcudart_static -ldl -lpthread -lrt
