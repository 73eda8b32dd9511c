"""RoPE + K/V append A/B at the verify shape (b=32, n=9, Mixtral heads): device
time (CUDA events, L2 flushed) and bit differences against the library's other
kernel. Run twice: SMO_ROPE_V1=0 / 1; outputs saved to /tmp/rope_<v>.pt."""
import os, sys, json
sys.path.insert(0, "tools")
import torch, kbench
from paper_2508_21706_b200 import ops
dev = torch.device("cuda:0")
b, n, nq, nkv, d, s = 32, 9, 32, 8, 128, 1024
g = torch.Generator(device=dev).manual_seed(5)
qkv = ((torch.rand((b * n, (nq + 2 * nkv) * d), generator=g, device=dev) * 2 - 1)).to(torch.bfloat16)
pre = torch.full((b,), s, dtype=torch.int32, device=dev) - torch.arange(b, dtype=torch.int32, device=dev) * 7
s_max = s + n + 64
kc = torch.zeros((b, nkv, s_max, d), dtype=torch.bfloat16, device=dev)
vc = torch.zeros_like(kc)
run = lambda: ops.rope_append(qkv, pre, None, b, n, nq, nkv, d, kc, vc, 1e6)
q = run()
t = kbench.timeit(run)
v = os.environ.get("SMO_ROPE_V1", "0")
torch.save({"q": q.cpu(), "k": kc.cpu(), "v": vc.cpu()}, f"/tmp/rope_{v}.pt")  # (large: kept off gpurun_out)
print(json.dumps({"rope_v1": v, "us": round(t * 1e6, 2)}))
