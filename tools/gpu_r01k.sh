#!/bin/bash
# r01k: final decoder version in the bench step — GPU tests, smoke, bench, reference arm, launch list,
# --set full of the unary decoder inside the timed step
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01k.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_r01k.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01k.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_r01k.log
timeout 1200 python bench.py > gpurun_out/bench_r01k.log 2>&1; echo "bench rc=$?"; grep metric gpurun_out/bench_r01k.log | tail -1 | cut -c1-160
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_r01k.log 2>&1; echo "ref rc=$?"; grep metric gpurun_out/bench_ref_r01k.log | tail -1 | cut -c1-160
SMO_PROFILE_TIMED=1 timeout 900 /usr/local/cuda/bin/ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01k.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-decode > /dev/null 2>&1; echo "ncu launches done"
SMO_PROFILE_TIMED=1 timeout 900 /usr/local/cuda/bin/ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:unary_decode -c 1 -o gpurun_out/codec_r01k -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-decode > gpurun_out/ncu_codec_r01k.log 2>&1; echo "ncu full rc=$?"
