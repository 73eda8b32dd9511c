timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; grep metric gpurun_out/bench.log | tail -1 | cut -c1-600
bash tools/prof_r01c.sh > /dev/null 2>&1; echo "prof done"
