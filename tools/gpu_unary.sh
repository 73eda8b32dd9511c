#!/bin/bash
# unary link code: kernel tests, engine tests, decoder microbench, ncu of the decoder
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -k "codec or compressed" -q 2>&1 | tail -8
timeout 300 python tools/kbench.py codec 2>&1 | tail -3 | tee gpurun_out/unary_kbench.jsonl
timeout 600 ncu --set full --clock-control none -k regex:unary_decode -c 1 --import-source on \
  -o gpurun_out/unary_decode -f python tools/kbench.py codec > gpurun_out/unary_ncu.log 2>&1
tail -2 gpurun_out/unary_ncu.log
