#!/bin/bash
# r01h: the unary link code in the bench step — full GPU tests, smoke, bench
# (N=1 default + reference arm), launch list and one --set full capture of the
# unary decoder inside the timed step.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_h.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_h.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_h.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_h.log
timeout 1200 python bench.py > gpurun_out/bench_h.log 2>&1; echo "bench rc=$?"; grep metric gpurun_out/bench_h.log | tail -1 | cut -c1-300
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_h.log 2>&1; echo "ref rc=$?"; grep metric gpurun_out/bench_ref_h.log | tail -1 | cut -c1-200
SMO_PROFILE_TIMED=1 timeout 900 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01h.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-decode > /dev/null 2>&1; echo "ncu launches done"
SMO_PROFILE_TIMED=1 timeout 900 /usr/local/cuda/bin/ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:unary_decode -c 1 -o gpurun_out/codec_r01h -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-decode > gpurun_out/ncu_codec_h.log 2>&1; echo "ncu full rc=$?"
