#!/bin/bash
# ncu evidence, round 1 final capture: the default (coded-transfer) bench step. Run under gpurun, 1 GPU.
NCU=/usr/local/cuda/bin/ncu
export SMO_PROFILE_TIMED=1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-decode"
$NCU --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01e.csv $B > gpurun_out/ncu_launch_bench.log 2>&1
$NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:moe_fused -c 1 -o gpurun_out/gemm_r01e $B > gpurun_out/ncu_gemm.log 2>&1
$NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:expert_decode -c 1 -o gpurun_out/codec_r01e $B > gpurun_out/ncu_codec.log 2>&1
python tools/kbench.py codec > gpurun_out/kbench_codec.jsonl 2>&1
ls -la gpurun_out
