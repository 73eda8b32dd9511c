timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/kbench.py gemm 2>&1 | grep fused
timeout 1200 python bench.py --no-cpu-baseline --no-decode --steps 3 > gpurun_out/bench_c.log 2>&1; echo "bench rc=$?"; grep metric gpurun_out/bench_c.log | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['frac'], d['expert_roofline']['frac'], d['stage_seconds_last_step'], d['gpu_launches'])"
