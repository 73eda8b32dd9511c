SMO_MOE_VARIANT=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k fused_moe > gpurun_out/pytest_moe.log 2>&1; echo "moe v1 rc=$?"; tail -3 gpurun_out/pytest_moe.log
for v in 0 1; do for sp in 1 2 4; do SMO_MOE_VARIANT=$v SMO_MOE_SPLITS=$sp timeout 300 python tools/kbench.py gemm 2>&1 | grep "fused" | sed "s/^/v$v s$sp /"; done; done
