#!/usr/bin/env bash
# Phase-timing build of libslra_cuda.so (cross_approx.cu with -DSLRA_PHASE_PROF)
# into tools/prof_build/lib; run a probe with LD_LIBRARY_PATH pointing there
# (the binding's RUNPATH yields to it). Not shipped, not used by tests/bench.
set -e
cd "$(dirname "$0")/../paper_1611_01391_b200"
OUT=../tools/prof_build
mkdir -p $OUT/lib
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../include \
  -DSLRA_PHASE_PROF -c csrc/cross_approx.cu -o $OUT/cross_approx_prof.o
objs=$(ls build/*.o | grep -v -e host_ -e py_slra -e '/cross_approx.o')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/lib/libslra_cuda.so $objs $OUT/cross_approx_prof.o \
  -L/usr/local/cuda/lib64 -lcudart
