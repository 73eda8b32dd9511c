#!/bin/bash
# Build a side variant of libspecmoe.so with extra -D flags (debug/trace builds).
# usage: tools/build_variant.sh <out.so> -DFLAG ...
set -e
OUT=$1; shift
TMP=$(mktemp -d)
cd "$(dirname "$0")/.."
for f in c_api ops gemm_tc attention engine ep; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -I include -I paper_2508_21706_b200/csrc "$@" -c paper_2508_21706_b200/csrc/$f.cu -o $TMP/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$OUT" $TMP/*.o
rm -rf $TMP
echo "built $OUT"
