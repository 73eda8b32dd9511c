import sys, os, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests'); sys.path.insert(0, '/root/repo/oracle')
from test_gpu_kernels import _attn_case, _u16
import oracle_py as O
from paper_2508_21706_b200 import ops
cuda = torch.device('cuda:0')
for (b, n, nq, nkv, d, prefix, tree) in [(1,24,32,8,128,[3000],True),(1,24,32,8,128,[3000],False),(1,24,32,8,128,[100],False),(1,17,32,8,128,[100],False),(2,32,32,8,128,[1000,200],False),(1,24,32,8,64,[3000],False)]:
    s_max = max(prefix) + n + 64
    q, kc, vc, mask, pre, bits = _attn_case(torch, cuda, b, n, nq, nkv, d, prefix, s_max, tree, seed=b * 31 + n)
    out = ops.verify_attention(q, kc, vc, mask, pre, max(prefix))
    ref = np.zeros((b * n, nq, d), np.uint16)
    O.lib().orc_verify_attention(O._ptr(_u16(q)), O._ptr(_u16(kc)), O._ptr(_u16(vc)), O._ptr(bits), O._ptr(np.array(prefix, np.int32)), b, n, nq, nkv, d, s_max, O._ptr(ref))
    got = out.float().cpu().numpy(); exp = O.bf16_to_f32(ref).reshape(got.shape)
    err = np.abs(got-exp).reshape(b, n, nkv, nq//nkv, d).max(axis=(0,4))  # [n, nkv, g]
    rows = (err > 1e-2)
    print((b,n,d,prefix,tree), 'maxerr', err.max(), 'bad (i,hh) rows:', sorted(set((i*(nq//nkv)+h) for i,k,h in zip(*np.nonzero(rows))))[:40])
