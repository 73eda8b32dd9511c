"""Router (K2) A/B at the verify shape: T=288 tokens, h=4096, 8 experts top-2
(and DSV2-Lite's 64 experts top-6); device time from kbench.timeit (L2 flushed)."""
import sys, json
sys.path.insert(0, "tools")
import torch, kbench
from paper_2508_21706_b200 import ops
dev = torch.device("cuda:0")
res = {}
for T, h, E, k in ((288, 4096, 8, 2), (288, 2048, 64, 6)):
    g = torch.Generator(device=dev).manual_seed(T + E)
    x = ((torch.rand((T, h), generator=g, device=dev) * 2 - 1)).to(torch.bfloat16)
    w = ((torch.rand((E, h), generator=g, device=dev) * 2 - 1) * 0.02).to(torch.bfloat16)
    t = kbench.timeit(lambda: ops.router_topk(x, w, k))
    res[f"E{E}"] = round(t * 1e6, 2)
print(json.dumps(res))
