set -x
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_dec.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/bench_dec.log
