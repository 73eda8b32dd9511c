#!/bin/bash
# ncu evidence for round 1 (run under gpurun, 1 GPU). Outputs in gpurun_out/.
# Launch counts: engine creation ~930 fills, one warm-up step ~486 launches.
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$NCU --metrics gpu__time_duration.sum --clock-control none -s 1420 -c 490 --csv --log-file gpurun_out/launches_r01.csv $B > gpurun_out/ncu_launch_bench.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:verify_attention -s 33 -c 1 -o gpurun_out/attn_r01 $B > gpurun_out/ncu_attn.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:gemm_tc -s 130 -c 4 -o gpurun_out/gemm_r01 $B > gpurun_out/ncu_gemm.log 2>&1
python tools/kbench.py all --sweep > gpurun_out/kbench_r01.jsonl 2>&1
ls -la gpurun_out
