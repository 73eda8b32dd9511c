set -x
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/pytest_decode.log 2>&1; echo "decode rc=$?"
tail -30 gpurun_out/pytest_decode.log
timeout 300 build/refsuites/test_verify_engine > gpurun_out/cpp_verify_engine.log 2>&1; echo "cpp rc=$?"; tail -30 gpurun_out/cpp_verify_engine.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
