#!/bin/bash
# ncu evidence for round 1 (run under gpurun, 1 GPU). Outputs in gpurun_out/.
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$NCU --metrics gpu__time_duration.sum --clock-control none -s 460 -c 440 --csv --log-file gpurun_out/launches_r01.csv $B > gpurun_out/ncu_launch_bench.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:verify_attention -s 40 -c 1 -o gpurun_out/attn_r01 $B > gpurun_out/ncu_attn.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:gemm_tc -s 200 -c 3 -o gpurun_out/gemm_r01 $B > gpurun_out/ncu_gemm.log 2>&1
ls -la gpurun_out
