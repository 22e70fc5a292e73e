#!/usr/bin/env bash
# Variant builds of stream_dmma.cu (tn_skinny stage rows / stages / CTAs per
# SM as -D macros) into tools/var_build/<name>/libslra_cuda.so; run a probe
# with LD_LIBRARY_PATH pointing at one. Measurement helper.
set -e
cd "$(dirname "$0")/../paper_1611_01391_b200"
build() {  # name, flags...
  local name=$1; shift
  local OUT=../tools/var_build/$name
  mkdir -p $OUT
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../include "$@" \
    -c csrc/stream_dmma.cu -o $OUT/stream_dmma.o
  objs=$(ls build/*.o | grep -v -e host_ -e py_slra -e '/stream_dmma.o')
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libslra_cuda.so $objs $OUT/stream_dmma.o \
    -L/usr/local/cuda/lib64 -lcudart
}
build tk32ns3 -DSLRA_TN_TK=32 -DSLRA_TN_NS=3 &
build tk64ns2 -DSLRA_TN_TK=64 -DSLRA_TN_NS=2 &
build tk32ns2c3 -DSLRA_TN_TK=32 -DSLRA_TN_NS=2 -DSLRA_TN_CTAS=3 &
build tk32ns3c3 -DSLRA_TN_TK=32 -DSLRA_TN_NS=3 -DSLRA_TN_CTAS=3 &
wait
