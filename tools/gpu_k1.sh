timeout 900 python -m pytest tests/test_gpu_kernels.py -q > gpurun_out/pytest_k1.log 2>&1; echo "rc=$?"; tail -5 gpurun_out/pytest_k1.log
timeout 600 python tools/dbg_prefill.py mixtral 32 1024 > gpurun_out/dbg_mx1.log 2>&1; echo "mx 32x1024 rc=$?"; grep -v CUDAEvent gpurun_out/dbg_mx1.log | tail -4
timeout 600 python tools/kbench.py gemm --splits > gpurun_out/kbench_gemm.jsonl 2>&1; cat gpurun_out/kbench_gemm.jsonl
timeout 600 python tools/kbench.py attn > gpurun_out/kbench_attn.jsonl 2>&1; cat gpurun_out/kbench_attn.jsonl
