NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none --import-source on -k regex:moe_fused -c 1 -o gpurun_out/moe_r01 python tools/kbench.py gemm > gpurun_out/ncu_moe.log 2>&1
$NCU -i gpurun_out/moe_r01.ncu-rep --page details --csv > gpurun_out/moe_r01_details.csv 2>&1
ls -la gpurun_out/moe_r01*
