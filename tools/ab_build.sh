#!/bin/bash
# A/B library build: tools/ab_build.sh <dir> <source.cu> <extra nvcc flags...>
# recompiles one translation unit with extra flags into <dir>/libclifford_b200.so
# (load it with CL_LIB_PATH=<dir>/libclifford_b200.so)
set -e
cd "$(dirname "$0")/.."
dir=$1; src=$2; shift 2
python -m paper_2507_01040_b200.build > /dev/null
mkdir -p $dir/obj
cp paper_2507_01040_b200/lib/obj/*.o $dir/obj/
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -Iinclude "$@" -c paper_2507_01040_b200/csrc/$src -o $dir/obj/$src.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $dir/libclifford_b200.so $dir/obj/*.o -lcudart_static -ldl -lrt -lpthread
echo built $dir/libclifford_b200.so
