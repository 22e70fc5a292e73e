#!/usr/bin/env bash
# Variant build: tools/variant_build.sh NAME SOURCE.cu [-D...] compiles one
# csrc/ source with extra flags and links tools/var_build/NAME/libslra_cuda.so
# from it and the regular objects of the other sources (run a probe with
# LD_LIBRARY_PATH pointing there). Measurement helper.
set -e
name=$1; src=$2; shift 2
cd "$(dirname "$0")/../paper_1611_01391_b200"
OUT=../tools/var_build/$name
mkdir -p $OUT
base=$(basename $src .cu)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../include "$@" \
  -c csrc/$src -o $OUT/$base.o
objs=$(ls build/*.o | grep -v -e host_ -e py_slra -e "/$base.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libslra_cuda.so $objs $OUT/$base.o \
  -L/usr/local/cuda/lib64 -lcudart
