"""Phase-0 box probe: host RAM, cores, PCIe H2D/D2H bandwidth (pinned), topology.
Writes gpurun_out/probe_box.json. Not part of the product path."""
import json, os, subprocess, time
import torch

def sh(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)

out = {"nproc": os.cpu_count(), "free": sh("free -g"), "lscpu": sh("lscpu | head -30"),
       "topo": sh("nvidia-smi topo -m"), "smi": sh("nvidia-smi --query-gpu=name,pcie.link.gen.max,pcie.link.width.max,pcie.link.gen.current,memory.total --format=csv"),
       "numa": sh("numactl -H 2>/dev/null | head -5"), "ulimit_l": sh("ulimit -l")}
dev = torch.device("cuda:0")
props = torch.cuda.get_device_properties(0)
out["sm_count"] = props.multi_processor_count
res = {}
for mb in [16, 64, 256, 1024, 2048]:
    n = mb << 20
    t0 = time.time()
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    pin_s = time.time() - t0
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(s):
            d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(2, min(20, (4 << 30) // n))
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(reps):
            d.copy_(h, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    h2d = n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(reps):
            h.copy_(d, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    d2h = n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
    res[mb] = {"h2d_gbs": h2d, "d2h_gbs": d2h, "pin_alloc_s": pin_s}
    del h, d
out["pcie"] = res
# two concurrent H2D streams on 1 GiB chunks
n = 1 << 30
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True); h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device=dev); d2 = torch.empty(n, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.time()
for _ in range(4):
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
torch.cuda.synchronize()
out["h2d_2streams_gbs"] = 8 * n / (time.time() - t0) / 1e9
# big pinned alloc timing (8 GiB)
t0 = time.time()
try:
    big = torch.empty(8 << 30, dtype=torch.uint8, pin_memory=True)
    out["pin_8g_s"] = time.time() - t0
    del big
except Exception as e:
    out["pin_8g_err"] = str(e)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k in ("nproc", "sm_count", "pcie", "h2d_2streams_gbs", "pin_8g_s")}, indent=1))
print(out["free"]); print(out["smi"]); print(out["topo"])
