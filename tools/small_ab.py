"""Per-layer small kernels at the verify shape (T=288, h=4096): RMSNorm and the
router, device time via kbench.timeit (L2 flushed) — same-box A/B with SPECMOE_LIB."""
import sys, json
sys.path.insert(0, "tools")
import torch, kbench
from paper_2508_21706_b200 import ops
dev = torch.device("cuda:0")
T, h = 288, 4096
x = torch.randn((T, h), device=dev)
gain = torch.ones(h, dtype=torch.bfloat16, device=dev)
res = {"rmsnorm": round(kbench.timeit(lambda: ops.rmsnorm(x, gain, 1e-5)) * 1e6, 2)}
xb = x.to(torch.bfloat16)
w = (torch.rand((8, h), device=dev) * 0.02).to(torch.bfloat16)
res["router"] = round(kbench.timeit(lambda: ops.router_topk(xb, w, 2)) * 1e6, 2)
k = 2
y = torch.randn((T * k, h), device=dev)
pos = torch.randperm(T * k, device=dev).to(torch.int32)
wts = torch.rand((T, k), device=dev)
resid = torch.randn((T, h), device=dev)
res["combine"] = round(kbench.timeit(lambda: ops.unpermute_combine_(resid, y, pos, wts)) * 1e6, 2)
ids = torch.randint(0, 8, (T, 2), device=dev, dtype=torch.int32)
res["permute"] = round(kbench.timeit(lambda: ops.permute(ids, 8)) * 1e6, 2)
res["permute+gather"] = round(kbench.timeit(lambda: ops.permute(ids, 8, xb)) * 1e6, 2)
print(json.dumps(res))
