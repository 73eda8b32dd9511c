"""Debug: K1 timeline of CTA 0 (needs build/libspecmoe_trace.so, -DSMO_ATTN_TRACE)."""
import ctypes as C, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["SPECMOE_LIB"] = os.path.join(ROOT, "build", "libspecmoe_trace.so")
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch
import kbench
from paper_2508_21706_b200 import _lib as L, ops
lib = L.load()
b, n, s = (int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (32, 9, 1024)
nq, nkv, d = 32, 8, 128
print(kbench.attn(b, n, s))
buf = np.zeros((3, 4096), np.uint64); cnt = np.zeros(3, np.int32)
lib.smo_debug_attn_trace(buf.ctypes.data_as(C.c_void_p), cnt.ctypes.data_as(C.c_void_p))  # clear
dev = torch.device("cuda:0")
q = torch.randn((b * n, nq, d), device=dev).to(torch.bfloat16)
kc = torch.randn((b, nkv, s + 80, d), device=dev).to(torch.bfloat16)
vc = torch.randn((b, nkv, s + 80, d), device=dev).to(torch.bfloat16)
mask = torch.tensor([(1 << (i + 1)) - 1 for i in range(n)] * b, dtype=torch.int64, device=dev)
pre = torch.full((b,), s, dtype=torch.int32, device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ops.verify_attention(q, kc, vc, mask, pre, s)
e1.record()
torch.cuda.synchronize()
print('traced call (includes workspace alloc):', e0.elapsed_time(e1) * 1e3, 'us')
lib.smo_debug_attn_trace(buf.ctypes.data_as(C.c_void_p), cnt.ctypes.data_as(C.c_void_p))
t0 = min(int(buf[r][0] >> 8) for r in range(3) if cnt[r])
names = {0: "prod", 1: "mma", 2: "soft"}
for r in range(3):
    nn = min(int(cnt[r]), 4096)
    evs = [(int(x >> 8) - t0, int(x & 255)) for x in buf[r][:nn]]
    print(names[r], nn, " ".join(f"{c}@{t/1000:.2f}" for t, c in evs[:80]))
    print("   ...", " ".join(f"{c}@{t/1000:.2f}" for t, c in evs[-12:]))
