"""Does a kernel that follows a long GPU idle gap run slower? K1 at the
config-2 verify shape timed back-to-back vs after 35 ms of host-side idle
(the per-layer wait for the link in the offloaded step)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.argv = ["kbench"]
import kbench as K  # noqa: E402
from paper_2508_21706_b200 import ops  # noqa: E402

b, n, s = 32, 9, 1024
s_max = s + n + 64
dev = K.dev
g = torch.Generator(device=dev).manual_seed(1)
q = (torch.rand((b * n, 32, 128), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
kc = (torch.rand((b, 8, s_max, 128), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
vc = (torch.rand((b, 8, s_max, 128), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
mask = torch.tensor([(1 << (i + 1)) - 1 for i in range(n)] * b, dtype=torch.int64, device=dev)
pre = torch.full((b,), s, dtype=torch.int32, device=dev)
import ctypes  # noqa: E402

CB = ctypes.CFUNCTYPE(None, ctypes.c_void_p)


def _sleep35(_):
    time.sleep(0.035)


sleep_cb = CB(_sleep35)
cudart = ctypes.CDLL("libcudart.so") if os.path.exists("/usr/local/cuda/lib64/libcudart.so") else None
if cudart is None:
    import glob
    cudart = ctypes.CDLL(glob.glob("/usr/local/cuda/lib64/libcudart.so*")[0])
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    ops.verify_attention(q, kc, vc, mask, pre, s)  # warm
    torch.cuda.synchronize()
    for idle in (False, True):
        ts = []
        for rep in range(12):
            events = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(1)]
            torch.cuda.synchronize()
            flush = torch.empty(1 << 28, dtype=torch.uint8, device=dev)
            flush.zero_()  # GPU busy while the host enqueues the rest
            if idle:  # stream blocked for 35 ms on a host function: GPU idle, K1 already enqueued behind it
                cudart.cudaLaunchHostFunc(ctypes.c_void_p(stream.cuda_stream), sleep_cb, None)
            e0, e1 = events[0]
            e0.record(stream)
            ops.verify_attention(q, kc, vc, mask, pre, s)
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        print(json.dumps({"kernel": "K1 b=32 n=9 s=1024 (launch pre-enqueued)", "after_35ms_idle": idle,
                          "median_us": ts[len(ts) // 2], "min_us": ts[0]}))
