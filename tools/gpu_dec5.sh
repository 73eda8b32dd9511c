#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_gpu_streamer.py -k "codec or compressed or streamer or cache" -q 2>&1 | tail -2
timeout 300 python tools/kbench.py codec 2>&1 | tail -1
