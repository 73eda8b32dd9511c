#!/bin/bash
# round-end validation: every GPU test, smoke, the default bench line and the reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_final.log
timeout 1200 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?"; grep metric gpurun_out/bench_final.log | tail -1 | cut -c1-200
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_final.log 2>&1; echo "ref rc=$?"; grep metric gpurun_out/bench_ref_final.log | tail -1 | cut -c1-160
