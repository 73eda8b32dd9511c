"""CPU vs GPU attention placement on the tiny model: same verify inputs,
compare per-layer attention outputs and targets."""
import dataclasses
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_21706_b200.engine import TINY, VerifyEngine  # noqa: E402

s = dataclasses.replace(TINY, seed=0x5EED + 7, lm_scale=8.0, router_scale=4.0)
b, n = 3, 5
pre = np.array([70, 33, 5], np.int32)
tok = np.random.default_rng(1).integers(0, s.vocab, size=(b, n)).astype(np.int32)
res = {}
for cpu in (False, True):
    e = VerifyEngine(s, max_batch=b, max_verify=6, max_seq=256, debug=True, attn_cpu=cpu)
    e.fill_prefix(pre)
    r = e.verify(tok, pre)
    res[cpu] = (r, [e.debug_tensor("attn", l, (b * n, s.n_q_heads, s.head_dim), np.uint16) for l in range(2)],
                [e.debug_tensor("q", l, (b * n, s.n_q_heads, s.head_dim), np.uint16) for l in range(2)],
                [e.debug_tensor("k_cache", l, (b, s.n_kv_heads, 256, s.head_dim), np.uint16) for l in range(2)])
    e.close()
f = lambda a: (a.astype(np.uint32) << 16).view(np.float32)  # noqa: E731
for l in range(2):
    for nm, i in (("attn", 1), ("q", 2), ("kc", 3)):
        a, c = f(res[False][i][l]), f(res[True][i][l])
        print(l, nm, "max abs diff", float(np.nanmax(np.abs(a - c))), "nan", int(np.isnan(c).sum()))
print("targets gpu", res[False][0].target.ravel()[:10], "\ntargets cpu", res[True][0].target.ravel()[:10])
print("acc", res[False][0].acc_len, res[True][0].acc_len)
