timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_gpu_ep.py -q -x -k "codec or compressed or ep_loop" > gpurun_out/pytest_codec.log 2>&1; echo "codec rc=$?"; tail -4 gpurun_out/pytest_codec.log
timeout 300 python tools/kbench.py codec
