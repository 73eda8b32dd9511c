timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_t10.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest_t10.log
