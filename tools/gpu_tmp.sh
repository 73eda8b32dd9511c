ls /sys/devices/system/node/ | head; nvidia-smi topo -m 2>/dev/null | head -5; numactl -H 2>/dev/null | head -3
Q="--steps 5 --warmup 3 --no-cpu-baseline --no-decode --no-raw --no-e2e"
timeout 900 python bench.py $Q 2>&1 | grep '"metric"' > gpurun_out/bench_numa_t11.json; python -c "
import json; d=json.load(open('gpurun_out/bench_numa_t11.json')); print(round(d['value'],1), d['config']['host_numa_node'], d['h2d']['achieved_gbs'])"
SMO_HOST_NUMA=-1 timeout 900 python bench.py $Q 2>&1 | grep '"metric"' > gpurun_out/bench_nonuma_t11.json; python -c "
import json; d=json.load(open('gpurun_out/bench_nonuma_t11.json')); print(round(d['value'],1), d['config']['host_numa_node'], d['h2d']['achieved_gbs'])"
