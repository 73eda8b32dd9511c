#!/bin/bash
# ncu evidence, round 1 third capture (fused K4-MoE in the step). Run under gpurun, 1 GPU.
NCU=/usr/local/cuda/bin/ncu
export SMO_PROFILE_TIMED=1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-decode"
$NCU --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01c.csv $B > gpurun_out/ncu_launch_bench.log 2>&1
$NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:verify_attention -c 1 -o gpurun_out/attn_r01c $B > gpurun_out/ncu_attn.log 2>&1
$NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:moe_fused -c 1 -o gpurun_out/gemm_r01c $B > gpurun_out/ncu_gemm.log 2>&1
python tools/kbench.py all > gpurun_out/kbench_r01c.jsonl 2>&1
ls -la gpurun_out
