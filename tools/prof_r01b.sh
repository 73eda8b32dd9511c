#!/bin/bash
# ncu evidence for round 1, second capture (current kernels). Run under gpurun, 1 GPU.
# bench.py brackets its timed steps with cudaProfilerStart/Stop when
# SMO_PROFILE_TIMED=1, so --profile-from-start off captures exactly the timed step.
NCU=/usr/local/cuda/bin/ncu
export SMO_PROFILE_TIMED=1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$NCU --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01b.csv $B > gpurun_out/ncu_launch_bench.log 2>&1
$NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:verify_attention -c 1 -o gpurun_out/attn_r01b $B > gpurun_out/ncu_attn.log 2>&1
$NCU --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tc -c 4 -o gpurun_out/gemm_r01b $B > gpurun_out/ncu_gemm.log 2>&1
python tools/kbench.py all --sweep > gpurun_out/kbench_r01b.jsonl 2>&1
ls -la gpurun_out
