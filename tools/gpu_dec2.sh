#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_gpu_streamer.py tests/test_gpu_ep.py -k "codec or compressed or streamer or ep_" -q 2>&1 | tail -4
timeout 300 python tools/kbench.py codec 2>&1 | tail -2 | tee gpurun_out/unary_kbench2.jsonl
timeout 600 ncu --set full --clock-control none -k regex:unary_decode -c 1 --import-source on -o gpurun_out/unary_decode2 -f python tools/kbench.py codec > gpurun_out/unary_ncu2.log 2>&1; tail -1 gpurun_out/unary_ncu2.log
