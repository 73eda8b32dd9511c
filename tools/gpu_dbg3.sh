set -x
SMO_PREFILL_CHECK=1 timeout 900 python tools/dbg_prefill.py mixtral 32 1024 > gpurun_out/dbg_mx_chk.log 2>&1; echo "rc=$?"; grep -v CUDAEvent gpurun_out/dbg_mx_chk.log | head -40
timeout 600 python tools/dbg_prefill.py mixtral 16 1024 > gpurun_out/dbg_mx16.log 2>&1; echo "16 rc=$?"; grep -v CUDAEvent gpurun_out/dbg_mx16.log | head -3
timeout 600 python tools/dbg_prefill.py mixtral 8 1024 > gpurun_out/dbg_mx8.log 2>&1; echo "8 rc=$?"; grep -v CUDAEvent gpurun_out/dbg_mx8.log | head -3
