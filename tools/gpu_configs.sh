# BASELINE configs 2 (hot cache 5.25 GB, k=4), 4 (fine-grained + shared expert) and
# 5's model on one GPU (Mixtral-8x22B; 8 aliased pinned layers, bytes unchanged)
mkdir -p gpurun_out
for args in "--cache-gb 5.25" "--k 4" "--model dsv2-lite --cache-gb 5.25" "--model qwen2-57b --cache-gb 5.25" "--model mixtral-8x22b --alias 8 --steps 3"; do
  echo "== $args"
  timeout 1200 python bench.py --no-cpu-baseline --no-decode $args > gpurun_out/cfg.log 2>&1; echo "rc=$?"
  grep '"metric"' gpurun_out/cfg.log | tail -1 >> gpurun_out/configs_r01.jsonl
  grep -v CUDAEvent gpurun_out/cfg.log | tail -2 | cut -c1-400
done
