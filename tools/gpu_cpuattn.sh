timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --no-decode --attn-cpu --steps 3 > gpurun_out/bench_cpuattn.log 2>&1; echo "bench rc=$?"; grep metric gpurun_out/bench_cpuattn.log | cut -c1-1500
