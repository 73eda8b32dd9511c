set -x
timeout 300 python tools/dbg_prefill.py mid 4 100 > gpurun_out/dbg_mid.log 2>&1; echo "mid rc=$?"; tail -5 gpurun_out/dbg_mid.log
timeout 600 /usr/local/cuda/bin/compute-sanitizer --print-limit 5 python tools/dbg_prefill.py mid 4 100 > gpurun_out/dbg_mid_san.log 2>&1; echo "san rc=$?"; head -60 gpurun_out/dbg_mid_san.log
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/pytest_kern.log 2>&1; echo "kern rc=$?"; tail -25 gpurun_out/pytest_kern.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log
