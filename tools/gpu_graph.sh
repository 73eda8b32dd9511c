timeout 600 python -m pytest tests/test_gpu_decode.py -q -x > gpurun_out/pytest_dec.log 2>&1; echo "dec rc=$?"; tail -25 gpurun_out/pytest_dec.log
timeout 600 python tools/decode_bench.py > gpurun_out/decode_bench.jsonl 2>&1; cat gpurun_out/decode_bench.jsonl | tail -5
