#!/bin/bash
# Build libspecmoe.so with some csrc files taken from another git revision
# (same-box A/B timing: SPECMOE_LIB=<out.so> selects it).
# usage: tools/build_rev.sh <out.so> <rev> <file.cu|file.cuh> ...
set -e
OUT=$1; REV=$2; shift 2
cd "$(dirname "$0")/.."
TMP=$(mktemp -d)
cp -r paper_2508_21706_b200/csrc "$TMP/src"
for f in "$@"; do git show "$REV:paper_2508_21706_b200/csrc/$f" > "$TMP/src/$f"; done
for f in c_api ops gemm_tc moe_tc attention engine decode prefill streamer ep xfer tcode; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -I include -I "$TMP/src" -c "$TMP/src/$f.cu" -o "$TMP/$f.o" &
done
g++ -O3 -mavx2 -mfma -std=c++17 -fPIC -pthread -I "$TMP/src" -c "$TMP/src/cpu_attn.cpp" -o "$TMP/cpu_attn.o" &
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$OUT" "$TMP"/*.o \
  -Xcompiler -pthread
rm -rf "$TMP"
echo "built $OUT ($REV: $*)"
