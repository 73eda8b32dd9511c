timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -x -k "codec or compressed" > gpurun_out/pytest_codec.log 2>&1; echo "codec rc=$?"; tail -20 gpurun_out/pytest_codec.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --compress --no-cpu-baseline --steps 3 > gpurun_out/bench_comp.log 2>&1; echo "bench rc=$?"; grep metric gpurun_out/bench_comp.log | tail -1 | cut -c1-2500
