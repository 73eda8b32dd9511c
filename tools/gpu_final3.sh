timeout 600 python -m pytest tests/test_gpu_engine.py -q -x -k compressed > gpurun_out/pytest_c.log 2>&1; echo "c rc=$?"; tail -2 gpurun_out/pytest_c.log
timeout 1200 python bench.py --no-cpu-baseline --no-decode --steps 3 > gpurun_out/bench_c.log 2>&1; echo "bench rc=$?"; grep metric gpurun_out/bench_c.log | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']); print(d['expert_roofline']['frac'], d['stage_seconds_last_step'])"
SMO_PROFILE_TIMED=1 /usr/local/cuda/bin/ncu --profile-from-start off --set full --clock-control none -k regex:expert_decode -c 1 -o gpurun_out/codec_r01f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-decode > gpurun_out/ncu_codec.log 2>&1; echo "ncu rc=$?"
