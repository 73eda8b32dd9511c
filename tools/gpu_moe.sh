timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k fused_moe > gpurun_out/pytest_moe.log 2>&1; echo "moe rc=$?"; tail -15 gpurun_out/pytest_moe.log
timeout 600 python tools/kbench.py gemm --splits > gpurun_out/kbench_moe.jsonl 2>&1; grep -i "grouped" gpurun_out/kbench_moe.jsonl
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
