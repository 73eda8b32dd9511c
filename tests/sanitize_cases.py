"""Workloads for the compute-sanitizer tier (tests/test_gpu_sanitizer.py).

Each case is small enough to finish in seconds under memcheck / racecheck /
synccheck and still launches the hand-written protocols the sanitizer should
see: K1 (stream-K split-KV with the in-kernel last-CTA merge over
workspace counters), K4-MoE (cross-CTA release/acquire on per-expert
counters, cooperative launch), the K5 unary codec, router/permute/combine,
greedy accept, and the expert-parallel loopback exchange.

    python tests/sanitize_cases.py verify|kernels|attn|moe|ep|coded|draft
"""
import dataclasses
import math
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def case_verify():
    from paper_2508_21706_b200.engine import TINY, VerifyEngine
    s = dataclasses.replace(TINY, seed=0x5EED + 1, lm_scale=8.0, router_scale=4.0)
    b, n = 4, 5
    prefix = np.array([300, 17, 64, 1], np.int32)
    tokens = np.random.default_rng(1).integers(0, s.vocab, size=(b, n)).astype(np.int32)
    for comp in (False, True):
        eng = VerifyEngine(s, max_batch=b, max_verify=n, max_seq=512, compress_experts=comp, micro_batches=2)
        eng.fill_prefix(prefix)
        eng.verify(tokens, prefix)
        eng.close()


def case_kernels():
    case_attn()
    case_moe()


def case_attn():
    from paper_2508_21706_b200 import ops
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(3)
    # K1: one request, 16 rows, long prefix -> several CTAs split the KV and merge
    b, n, nq, nkv, d, p = 1, 16, 32, 8, 128, 3000
    s_max = p + n + 64
    q = (torch.rand((b * n, nq, d), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
    kc = (torch.rand((b, nkv, s_max, d), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
    vc = (torch.rand((b, nkv, s_max, d), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
    mask = torch.tensor([(1 << (i + 1)) - 1 for i in range(n)], dtype=torch.int64, device=dev)
    pre = torch.tensor([p], dtype=torch.int32, device=dev)
    ops.verify_attention(q, kc, vc, mask, pre, p)
    torch.cuda.synchronize()


def case_moe():
    from paper_2508_21706_b200 import ops
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(4)
    # K4-MoE: several token tiles per expert, down split in 2
    T, E, k, h, hi = 300, 4, 2, 256, 256
    x = (torch.rand((T, h), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
    blk = 3 * h * hi
    pool = ((torch.rand((E * blk,), generator=g, device=dev) * 2 - 1) * math.sqrt(3.0 / h)).to(torch.bfloat16)
    ids = torch.topk(torch.randn((T, E), generator=g, device=dev), k, dim=1).indices.to(torch.int32).contiguous()
    off, perm, pos, xp = ops.permute(ids, E, x)
    ops.moe_experts(xp, off, pool, h=h, h_i=hi, n_expert=E, w_block_stride=blk * 2, w_pool_blocks=E, splits=2)
    # K5 unary codec round trip
    w = torch.empty(1024 * 64, dtype=torch.bfloat16, device=dev)
    ops.fill_uniform_(w, 0x5EED, 99, 0.02)
    code, _ = ops.expert_encode(w, 1)
    assert torch.equal(ops.expert_decode(code, w.numel(), 1).view(torch.int16), w.view(torch.int16))
    torch.cuda.synchronize()


def case_coded():
    """T2 / T3 tile codes: GPU encoder + decoder round trip, and K4-MoE decoding them in
    shared memory (bulk copies into a code ring, 16 decoder warps,
    fence.proxy.async + mbarriers, paired down stages) on ragged groups."""
    from paper_2508_21706_b200 import ops
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(5)
    T, E, k, h, hi = 150, 4, 2, 256, 384
    blk = 3 * h * hi
    blks = []
    for e in range(E):
        b = torch.empty(blk, dtype=torch.bfloat16, device=dev)
        ops.fill_uniform_(b, 0x5EED, 500 + e, math.sqrt(3.0 / h))
        blks.append(b)
    codes = [ops.tcode_encode(b, h, hi) for b in blks]
    assert torch.equal(ops.tcode_decode(codes[0], h, hi).view(torch.int16), blks[0].view(torch.int16))
    w_code = torch.tensor([c.data_ptr() for c in codes], dtype=torch.int64, device=dev)
    x = (torch.rand((T, h), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
    ids = torch.topk(torch.randn((T, E), generator=g, device=dev), k, dim=1).indices.to(torch.int32).contiguous()
    off, perm, pos, xp = ops.permute(ids, E, x)
    h1, y1 = ops.moe_experts_coded(xp, off, w_code, h=h, h_i=hi, n_expert=E)
    h0, y0 = ops.moe_experts(xp, off, torch.cat(blks), h=h, h_i=hi, n_expert=E, w_block_stride=blk * 2,
                             w_pool_blocks=E, splits=y1.shape[0])
    assert torch.equal(y0.view(torch.int32), y1.view(torch.int32))
    # T3: encoder + decoder, and K4-MoE decoding it (escape lists patched after a __syncwarp)
    codes3 = [ops.tcode_encode(b, h, hi, fmt=3) for b in blks]
    assert torch.equal(ops.tcode_decode(codes3[1], h, hi, fmt=3).view(torch.int16), blks[1].view(torch.int16))
    w_code3 = torch.tensor([c.data_ptr() for c in codes3], dtype=torch.int64, device=dev)
    h3, y3 = ops.moe_experts_coded(xp, off, w_code3, h=h, h_i=hi, n_expert=E, fmt=3)
    assert torch.equal(y0.view(torch.int32), y3.view(torch.int32))
    torch.cuda.synchronize()


def case_draft():
    """Drafter CPU part: host-resident drafter K/V, host-pool attention released
    and awaited through device-polled flags in mapped memory."""
    from paper_2508_21706_b200.engine import TINY, VerifyEngine
    s = dataclasses.replace(TINY, seed=0x5EED + 5, draft_layers=1, draft_inter=512)
    rng = np.random.default_rng(2)
    prompts = [list(rng.integers(0, s.vocab, size=L)) for L in (40, 17, 9)]
    eng = VerifyEngine(s, max_batch=3, max_verify=4, max_seq=128, draft_cpu_kv=True)
    eng.prefill(prompts)
    eng.set_draft_split(1)
    for _ in range(2):
        eng.decode_step(3)
    eng.decode_read(3, 32)
    eng.close()


def case_ep():
    from paper_2508_21706_b200.engine import TINY, EpGroup, VerifyEngine
    s = dataclasses.replace(TINY, seed=0x5EED + 3)
    P, B, N = 2, 4, 5
    prefix = np.array([300, 297, 200, 1], np.int32)
    tokens = np.random.default_rng(11).integers(0, s.vocab, size=(B, N)).astype(np.int32)
    grp = EpGroup.loopback(P)
    bl = B // P
    engines = [VerifyEngine(s, max_batch=bl, max_verify=N, max_seq=512, ep_rank=r, ep_size=P, ep_group=grp,
                            compress_experts=True) for r in range(P)]
    for r, e in enumerate(engines):
        e.fill_prefix(prefix[r * bl:(r + 1) * bl])
    streams = [torch.cuda.Stream() for _ in range(P)]
    errors = []

    def work(r):
        try:
            engines[r].verify(tokens[r * bl:(r + 1) * bl], prefix[r * bl:(r + 1) * bl], stream=streams[r].cuda_stream)
        except Exception as ex:
            errors.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for e in engines:
        e.close()
    grp.close()


if __name__ == "__main__":
    {"verify": case_verify, "kernels": case_kernels, "attn": case_attn, "moe": case_moe,
     "ep": case_ep, "coded": case_coded, "draft": case_draft}[sys.argv[1]]()
    print("case ok")
