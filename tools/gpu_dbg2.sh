set -x
timeout 600 python tools/dbg_prefill.py mixtral 32 1024 > gpurun_out/dbg_mx1.log 2>&1; echo "mx 32x1024 rc=$?"; grep -v CUDAEvent gpurun_out/dbg_mx1.log | tail -5
timeout 600 python tools/dbg_prefill.py mixtral 4 1024 > gpurun_out/dbg_mx2.log 2>&1; echo "mx 4x1024 rc=$?"; grep -v CUDAEvent gpurun_out/dbg_mx2.log | tail -5
timeout 600 python tools/dbg_prefill.py mixtral 32 100 > gpurun_out/dbg_mx3.log 2>&1; echo "mx 32x100 rc=$?"; grep -v CUDAEvent gpurun_out/dbg_mx3.log | tail -5
