#!/usr/bin/env bash
# Phase-timing build of libslra_cuda.so (cholqr.cu with -DSLRA_CQC_PROF: CTA 0
# of problem 0 prints clock64 deltas per phase) into tools/prof_build/lib; run
# with LD_LIBRARY_PATH pointing there. Not shipped, not used by tests/bench.
set -e
cd "$(dirname "$0")/../paper_1611_01391_b200"
OUT=../tools/prof_build
mkdir -p $OUT/lib
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../include \
  -DSLRA_CQC_PROF -c csrc/cholqr.cu -o $OUT/cholqr_prof.o
objs=$(ls build/*.o | grep -v -e host_ -e py_slra -e '/cholqr.o')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/lib/libslra_cuda.so $objs $OUT/cholqr_prof.o \
  -L/usr/local/cuda/lib64 -lcudart
