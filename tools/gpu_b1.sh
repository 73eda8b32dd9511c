timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
rm -f gpurun_out/batch_one_r01.jsonl
for args in "--batch 1 --k 4" "--batch 1 --k 4 --moe-batching one" "--model dsv2-lite --batch 1 --k 4" "--model dsv2-lite --batch 1 --k 4 --moe-batching one" "--model qwen2-57b --batch 1 --k 4 --moe-batching one" "--batch 4 --k 4 --moe-batching one"; do
  echo "== $args"
  timeout 900 python bench.py --no-cpu-baseline --no-decode --steps 3 $args > gpurun_out/b1.log 2>&1; echo "rc=$?"
  grep '"metric"' gpurun_out/b1.log | tail -1 >> gpurun_out/batch_one_r01.jsonl
  grep -v CUDAEvent gpurun_out/b1.log | grep -v metric | tail -2 | cut -c1-300
done
