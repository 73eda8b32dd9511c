#!/bin/bash
# Build a side variant of libspecmoe.so with extra -D flags (debug/trace builds).
# usage: tools/build_variant.sh <out.so> -DFLAG ...
set -e
OUT=$1; shift
TMP=$(mktemp -d)
cd "$(dirname "$0")/.."
for f in c_api ops gemm_tc moe_tc attention engine decode prefill streamer ep xfer tcode; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -I include -I paper_2508_21706_b200/csrc "$@" -c paper_2508_21706_b200/csrc/$f.cu -o $TMP/$f.o &
done
g++ -O3 -mavx2 -mfma -std=c++17 -fPIC -pthread -I paper_2508_21706_b200/csrc -c paper_2508_21706_b200/csrc/cpu_attn.cpp \
  -o $TMP/cpu_attn.o &
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$OUT" $TMP/*.o \
  -Xcompiler -pthread
rm -rf $TMP
echo "built $OUT"
