#!/usr/bin/env bash
# Phase-timestamp build of libslra_cuda.so (lsr_cluster.cu with -DSLRA_CHOL_PROF)
# into tools/prof_build/chol/lib; probe: tools/chol_probe.py. Not shipped.
set -e
cd "$(dirname "$0")/../paper_1611_01391_b200"
OUT=../tools/prof_build/chol
mkdir -p $OUT/lib
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../include \
  -DSLRA_CHOL_PROF -c csrc/lsr_cluster.cu -o $OUT/lsr_cluster_prof.o
objs=$(ls build/*.o | grep -v -e host_ -e py_slra -e '/lsr_cluster.o')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/lib/libslra_cuda.so $objs $OUT/lsr_cluster_prof.o \
  -L/usr/local/cuda/lib64 -lcudart
