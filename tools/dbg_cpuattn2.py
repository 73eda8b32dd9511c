"""CPU vs GPU placement: prefill then decode steps; compare caches/histories."""
import dataclasses
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_21706_b200.engine import TINY, VerifyEngine  # noqa: E402

s = dataclasses.replace(TINY, seed=0x5EED + 7, lm_scale=8.0, router_scale=4.0, draft_layers=1, draft_inter=512)
b = 3
rng = np.random.default_rng(11)
prompts = [rng.integers(0, s.vocab, size=L).astype(np.int32) for L in [70, 33, 5]]
res = {}
f = lambda a: (a.astype(np.uint32) << 16).view(np.float32)  # noqa: E731
for cpu in (False, True):
    e = VerifyEngine(s, max_batch=b, max_verify=6, max_seq=256, debug=True, attn_cpu=cpu)
    nxt = e.prefill(prompts)
    kc = [e.debug_tensor("k_cache", l, (b, s.n_kv_heads, 256, s.head_dim), np.uint16) for l in range(2)]
    e.decode_step(0)
    h0 = e.decode_read(b, 16)
    e.decode_step(4, np.tile(np.arange(4, dtype=np.int32), (b, 1)))
    h1 = e.decode_read(b, 16)
    t = e.debug_tensor("attn", 0, (b * 5, s.n_q_heads, s.head_dim), np.uint16)
    res[cpu] = (nxt, kc, h0, h1, t)
    e.close()
print("next", res[False][0], res[True][0])
for l in range(2):
    for r, L in enumerate([70, 33, 5]):
        a, c = f(res[False][1][l][r, :, :L]), f(res[True][1][l][r, :, :L])
        print("layer", l, "req", r, "kc max diff", float(np.max(np.abs(a - c))))
print("hist after k=0", res[False][2][0][:, :3].tolist(), res[True][2][0][:, :3].tolist(), res[False][2][2], res[True][2][2])
print("hist after k=4", res[False][3][0][:, :6].tolist(), res[True][3][0][:, :6].tolist(), res[False][3][2], res[True][3][2])
print("attn L0 decode diff", float(np.max(np.abs(f(res[False][4]) - f(res[True][4])))))
