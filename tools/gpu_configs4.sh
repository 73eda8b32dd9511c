#!/bin/bash
# every BASELINE config with the default (unary) link code; rest of the GPU tests
mkdir -p gpurun_out
rm -f gpurun_out/configs_final_r01.jsonl
for args in "--cache-gb 5.25" "--k 4" "--model dsv2-lite --cache-gb 5.25" "--model qwen2-57b --cache-gb 5.25" "--model mixtral-8x22b --alias 8 --steps 3" "--batch 1 --k 4 --moe-batching one" "--model dsv2-lite --batch 1 --k 4 --moe-batching one" "--attn-cpu --steps 3"; do
  echo "== $args"
  timeout 1200 python bench.py --no-cpu-baseline --no-decode $args > gpurun_out/cfg.log 2>&1; echo "rc=$?"
  grep '"metric"' gpurun_out/cfg.log | tail -1 >> gpurun_out/configs_final_r01.jsonl
done
timeout 900 python tools/spec_decode_bench.py > gpurun_out/spec_final.jsonl 2>gpurun_out/spec_final.err; echo "spec rc=$?"; tail -1 gpurun_out/spec_final.jsonl | cut -c1-300
