"""Dense-projection GEMM timings at the verify step's shapes (QKV, O-proj +
residual, a 32-token QKV, a K = 14336 fp32 projection); one line per run,
prefixed by $TAG — for same-box A/Bs (e.g. SMO_GEMM_CSPLIT=0 vs default)."""
import sys, os
sys.path.insert(0, "tools")
import kbench, torch
from paper_2508_21706_b200 import ops, _lib as L
dev = torch.device("cuda:0")
tag = os.environ.get("TAG", "")
res = []
for (T, K, N, epi, nm) in ((288, 4096, 6144, L.EPI_BF16, "qkv"), (288, 4096, 4096, L.EPI_F32_ADD, "o"),
                           (32, 4096, 6144, L.EPI_BF16, "qkv32"), (288, 14336, 4096, L.EPI_F32, "down")):
    x = (torch.rand((T, K), device=dev) * 2 - 1).to(torch.bfloat16)
    w = (torch.rand((N, K), device=dev) * 2 - 1).to(torch.bfloat16)
    out = torch.zeros((T, N), dtype=torch.float32 if epi in (L.EPI_F32_ADD, L.EPI_F32) else torch.bfloat16, device=dev)
    t = kbench.timeit(lambda: ops.gemm(x, w, epilogue=epi, out=out))
    res.append(f"{nm}:{t*1e6:.1f}")
T, K, V = 288, 4096, 32000
x = (torch.rand((T, K), device=dev) * 2 - 1).to(torch.bfloat16)
w = (torch.rand((V, K), device=dev) * 2 - 1).to(torch.bfloat16)
t = kbench.timeit(lambda: ops.gemm(x, w, epilogue=L.EPI_ARGMAX))
res.append(f"lmhead:{t*1e6:.1f}")
print(tag, " ".join(res), flush=True)
