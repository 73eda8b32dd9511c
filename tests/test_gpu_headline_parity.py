"""GPU parity at the shapes bench.py times (BASELINE config 2 — the headline —
and config 4), not only at the tiny config.

1. Mixtral-8x7B shape (h 4096, h_i 14336, 8 experts top-2, 32/8 heads x 128,
   V 32000), b=32, k=8 (n=9), prefix 1024, the bench's default unary-coded
   expert transfer: the engine reduced to 2 layers (every per-layer kernel and
   launch parameter is what the 32-layer bench runs), one verify step,
   teacher-forced stage parity on BOTH layers against the CPU oracle:
     router logits / top-k ids / permutation           bit-exact
     K1 attention                                      max-abs <= 2^-8 max|V|
     QKV+RoPE, O-proj+RMSNorm                          rel-RMS <= 5e-3 / 4e-3
     MoE + combine (fused K4-MoE, production split S)  rel-RMS <= 1e-2
     LM head logits                                    rel-RMS <= 1e-4
     argmax on margin-screened rows, accept/bonus      bit-exact
   and bit-identity with raw bf16 streaming.
2. The same at config 4 (DeepSeek-V2-Lite shape: 64 experts top-6 + shared).
3. Expert parallelism P=2 (loopback) at Mixtral dimensions: bit-identical to
   one GPU.
4. The unary codec on one full 352 MB Mixtral expert block (the engine's own
   procedural weights): bit-exact round trip, and the engine's host code is
   byte-identical to a fresh encode.
5. K4-MoE alone at 576 x 4096 x 14336 (T=288, top-2) with the production S
   vs fp32 torch.

Anchors: /root/reference/proj/include/moeplan/attention.hpp:117-156,
specdec.hpp:57-85, SURVEY.md §8(c) tolerances.
"""
import dataclasses
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

B, K_DRAFT, PREFIX = 32, 8, 1024
N = K_DRAFT + 1


def _close(got, exp, rel_rms, what):
    got = np.asarray(got, np.float64)
    exp = np.asarray(exp, np.float64)
    err = np.sqrt(np.mean((got - exp) ** 2) / max(1e-30, np.mean(exp ** 2)))
    assert err <= rel_rms, f"{what}: rel-RMS {err:.3e} > {rel_rms}"
    return err


def _prefix():
    # ragged like a live batch: most at the bench's 1024, a few shorter
    p = np.full(B, PREFIX, np.int32)
    p[1], p[5], p[17], p[30] = 1000, 513, 129, 1
    return p


def stage_parity(eng, om, oracle, tokens, prefix, s_max, moe_tol=1e-2):
    """Teacher-forced parity of every stage of every layer (each stage
    recomputed by the oracle from the GPU's own input to it). Returns the
    per-stage errors."""
    s = om.s
    b, n = tokens.shape
    T = b * n
    d, nq, nkv = s.head_dim, s.n_q_heads, s.n_kv_heads
    f32 = oracle.bf16_to_f32
    errs = {}
    x0 = eng.debug_tensor("x_in", 0, (T, s.hidden), np.float32)
    assert np.array_equal(x0, f32(om.embed()[tokens.ravel()]))
    pos = np.concatenate([prefix[r] + np.arange(n) for r in range(b)]).astype(np.int32)
    for l in range(s.n_layers):
        x_in = eng.debug_tensor("x_in", l, (T, s.hidden), np.float32)
        xn1 = eng.debug_tensor("xn1", l, (T, s.hidden), np.uint16)
        errs[f"L{l}.rmsnorm"] = _close(f32(xn1), f32(om.rmsnorm(x_in)), 4e-3, f"L{l} rmsnorm")
        q = eng.debug_tensor("q", l, (T, nq, d), np.uint16)
        qkv = oracle.f32_to_bf16(om.gemm(xn1, om.wqkv(l)))
        q_ref = om.rope(qkv[:, :nq * d], pos, nq).reshape(T, nq, d)
        errs[f"L{l}.qkv_rope"] = _close(f32(q), f32(q_ref), 5e-3, f"L{l} qkv+rope")
        kc = eng.debug_tensor("k_cache", l, (b, nkv, s_max, d), np.uint16)
        vc = eng.debug_tensor("v_cache", l, (b, nkv, s_max, d), np.uint16)
        kp = om.kv_prefix(l, 0, prefix, s_max)
        k_new = om.rope(qkv[:, nq * d:(nq + nkv) * d], pos, nkv).reshape(b, n, nkv, d)
        kg = np.stack([kc[r, :, prefix[r]:prefix[r] + n] for r in range(b)])  # [b, nkv, n, d]
        for r in range(b):
            assert np.array_equal(kc[r, :, :prefix[r]], kp[r, :, :prefix[r]]), f"L{l} prefix K row {r}"
        errs[f"L{l}.k_append"] = _close(f32(kg), f32(k_new.transpose(0, 2, 1, 3)), 5e-3, f"L{l} k append")
        attn = eng.debug_tensor("attn", l, (T, nq, d), np.uint16)
        mbits = np.tile(om.mask_bits(None, n), b)
        attn_ref = om.attention(q, kc, vc, mbits, prefix, n)
        vmax = float(np.abs(f32(vc)).max())
        aerr = float(np.abs(f32(attn) - f32(attn_ref)).max())
        # K1 max-abs <= 2^-8 * max|V| (K1 carries P as hi+lo bf16 planes)
        assert aerr <= 2 ** -8 * vmax, f"L{l} attention max-abs {aerr} > 2^-8 * {vmax}"
        errs[f"L{l}.attention_maxabs"] = aerr
        errs[f"L{l}.attention"] = _close(f32(attn), f32(attn_ref), 5e-3, f"L{l} attention")
        x_mid = x_in + om.gemm(attn.reshape(T, -1), om.wo(l))
        xn2 = eng.debug_tensor("xn2", l, (T, s.hidden), np.uint16)
        errs[f"L{l}.oproj_rmsnorm"] = _close(f32(xn2), f32(om.rmsnorm(x_mid)), 4e-3, f"L{l} o-proj+rmsnorm")
        lg = eng.debug_tensor("logits_r", l, (T, s.n_expert), np.float32)
        lg_ref = om.router_logits(xn2, l)
        assert np.array_equal(lg.view(np.uint32), lg_ref.view(np.uint32)), f"L{l} router logits"
        ids = eng.debug_tensor("ids", l, (T, s.top_k), np.int32)
        wts = eng.debug_tensor("weights", l, (T, s.top_k), np.float32)
        ids_ref, w_ref = om.topk(lg_ref)
        assert np.array_equal(ids, ids_ref), f"L{l} top-k ids"
        assert np.allclose(wts, w_ref, rtol=1e-5, atol=1e-6)
        off, perm, pos_p = om.permute(ids_ref)
        assert np.array_equal(eng.debug_tensor("offsets", l, (s.n_expert + 1,), np.int32), off), f"L{l} offsets"
        assert np.array_equal(eng.debug_tensor("pos", l, (T * s.top_k,), np.int32), pos_p), f"L{l} permutation"
        x_out = eng.debug_tensor("x_out", l, (T, s.hidden), np.float32)
        base = x_mid
        sh = om.shared(l)
        if sh is not None:
            Ysh = om.gemm(oracle.f32_to_bf16(_swiglu(om, xn2, sh)), sh[2])
            base = x_mid + Ysh
        ref_out = base + om.moe(xn2, l, ids, wts)
        # the expert contribution alone (x_out - x_mid) is what K4-MoE + combine produced
        errs[f"L{l}.moe_combine"] = _close(x_out - x_mid, ref_out - x_mid, moe_tol, f"L{l} moe+combine")
        errs[f"L{l}.x_out"] = _close(x_out, ref_out, moe_tol, f"L{l} x_out")
    x_last = eng.debug_tensor("x_out", s.n_layers - 1, (T, s.hidden), np.float32)
    xf = eng.debug_tensor("xf", -1, (T, s.hidden), np.uint16)
    errs["final_rmsnorm"] = _close(f32(xf), f32(om.rmsnorm(x_last)), 4e-3, "final rmsnorm")
    logits = eng.debug_tensor("logits", -1, (T, s.vocab), np.float32)
    lref = om.gemm(xf, om.lm_head())
    errs["lm_head"] = _close(logits, lref, 1e-4, "lm head")
    return errs, logits, lref


def _swiglu(om, xn, w):
    g = om.gemm(xn, w[0]).astype(np.float64)
    u = om.gemm(xn, w[1]).astype(np.float64)
    return (g / (1.0 + np.exp(-g)) * u).astype(np.float32)


def head_and_accept(oracle, res, tokens, logits, lref):
    """Argmax bit-exact on rows whose oracle top-1/top-2 margin exceeds 8x the
    observed max logit error; accept / bonus / keep equal the
    oracle's greedy accept (specdec.hpp:65-76) on the GPU's argmax targets."""
    b, n = tokens.shape
    T = b * n
    tgt = res.target.ravel()
    assert np.array_equal(tgt, np.argmax(logits, axis=1).astype(np.int32)), "fused argmax != argmax(logits)"
    err = float(np.abs(logits - lref).max())
    srt = np.sort(lref, axis=1)
    screened = (srt[:, -1] - srt[:, -2]) > 8 * err
    assert screened.sum() >= T // 2, f"only {screened.sum()} of {T} rows clear the margin screen"
    assert np.array_equal(tgt[screened], np.argmax(lref, axis=1)[screened].astype(np.int32))
    acc, bonus, keep = np.zeros(b, np.int32), np.zeros(b, np.int32), np.zeros(T, np.int32)
    oracle.lib().orc_greedy_accept(oracle._ptr(tokens), oracle._ptr(tgt.copy()), None, b, n, oracle._ptr(acc),
                                   oracle._ptr(bonus), oracle._ptr(keep))
    assert np.array_equal(res.acc_len, acc) and np.array_equal(res.bonus, bonus)
    assert np.array_equal(res.keep.ravel(), keep)
    return int(screened.sum())


def _planted_tokens(vocab, seed):
    """Random roots; request r's drafts copy part of a fixed chain so the
    accept kernel sees varied lengths only where the target agrees (greedy)."""
    return np.random.default_rng(seed).integers(0, vocab, size=(B, N)).astype(np.int32)


@pytest.mark.parametrize("model", ["mixtral-8x7b", "dsv2-lite"])
def test_headline_shape_stage_parity(cuda, oracle, model):
    import oracle_model
    from paper_2508_21706_b200.engine import DSV2_LITE, MIXTRAL_8X7B, VerifyEngine
    shape = dataclasses.replace(MIXTRAL_8X7B if model == "mixtral-8x7b" else DSV2_LITE, n_layers=2)
    prefix = _prefix()
    s_max = PREFIX + N + 64
    tokens = _planted_tokens(shape.vocab, 3)
    eng = VerifyEngine(shape, max_batch=B, max_verify=N, max_seq=s_max, debug=True, compress_experts=True)
    eng.fill_prefix(prefix)
    res = eng.verify(tokens, prefix)
    t = eng.last_times()
    raw = shape.n_layers * shape.n_expert * shape.expert_bytes
    assert t["h2d_raw_bytes"] == raw
    assert 0 < t["h2d_bytes"] < raw * 11 // 16  # coded: ~10.3 bits/weight crossed the link
    om = oracle_model.OracleModel(shape)
    errs, logits, lref = stage_parity(eng, om, oracle, tokens, prefix, s_max)
    screened = head_and_accept(oracle, res, tokens, logits, lref)
    # the coded transfer is lossless: a raw-bf16 engine gives the same bits
    x_last = eng.debug_tensor("x_out", shape.n_layers - 1, (B * N, shape.hidden), np.float32)
    eng.close()
    raw_eng = VerifyEngine(shape, max_batch=B, max_verify=N, max_seq=s_max, debug=True, compress_experts=False)
    raw_eng.fill_prefix(prefix)
    r2 = raw_eng.verify(tokens, prefix)
    x2 = raw_eng.debug_tensor("x_out", shape.n_layers - 1, (B * N, shape.hidden), np.float32)
    raw_eng.close()
    assert np.array_equal(x_last.view(np.uint32), x2.view(np.uint32))
    assert np.array_equal(res.target, r2.target) and np.array_equal(res.acc_len, r2.acc_len)
    print(model, "screened rows", screened, {k: float(f"{v:.3e}") for k, v in errs.items()})


def test_ep2_mixtral_dims_bit_identical(cuda):
    """Expert parallelism P=2 over the loopback transport at Mixtral
    dimensions (config 5's mechanism at the config-2 shape): each rank owns 4
    experts, streams only their coded blocks, and its requests' outputs equal
    a single-GPU engine's bit for bit (the same expert rows, same K order,
    same combine order)."""
    import threading

    import torch
    from paper_2508_21706_b200.engine import EpGroup, MIXTRAL_8X7B, VerifyEngine
    shape = dataclasses.replace(MIXTRAL_8X7B, n_layers=2)
    P, bl = 2, B // 2
    prefix = _prefix()
    s_max = PREFIX + N + 64
    tokens = _planted_tokens(shape.vocab, 5)
    grp = EpGroup.loopback(P)
    engines = [VerifyEngine(shape, max_batch=bl, max_verify=N, max_seq=s_max, debug=True, ep_rank=r, ep_size=P,
                            ep_group=grp, compress_experts=True) for r in range(P)]
    for r, e in enumerate(engines):
        e.fill_prefix(prefix[r * bl:(r + 1) * bl])
    streams = [torch.cuda.Stream() for _ in range(P)]
    results, errors = [None] * P, []

    def work(r):
        try:
            results[r] = engines[r].verify(tokens[r * bl:(r + 1) * bl], prefix[r * bl:(r + 1) * bl],
                                           stream=streams[r].cuda_stream)
        except Exception as ex:
            errors.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=900)
    assert not errors, errors
    t0 = engines[0].last_times()
    assert t0["h2d_raw_bytes"] == shape.n_layers * (shape.n_expert // P) * shape.expert_bytes
    mine = [[e.debug_tensor("x_out", l, (bl * N, shape.hidden), np.float32) for l in range(shape.n_layers)]
            for e in engines]
    for e in engines:
        e.close()
    grp.close()
    for r in range(P):
        ref = VerifyEngine(shape, max_batch=bl, max_verify=N, max_seq=s_max, debug=True, compress_experts=True)
        ref.fill_prefix(prefix[r * bl:(r + 1) * bl])
        want = ref.verify(tokens[r * bl:(r + 1) * bl], prefix[r * bl:(r + 1) * bl])
        assert np.array_equal(results[r].target, want.target), r
        assert np.array_equal(results[r].acc_len, want.acc_len) and np.array_equal(results[r].bonus, want.bonus)
        for l in range(shape.n_layers):
            full = ref.debug_tensor("x_out", l, (bl * N, shape.hidden), np.float32)
            assert np.array_equal(mine[r][l].view(np.uint32), full.view(np.uint32)), (r, l)
        ref.close()


def _mixtral_block(torch, cuda, h=4096, hi=14336, seed=0x5EED, layer=0, expert=0):
    """One [W1 | W3 | W2] expert block exactly as the engine generates it
    (DESIGN.md §3.1 tensor ids and scales)."""
    from paper_2508_21706_b200 import ops
    blk = torch.empty(3 * h * hi, dtype=torch.bfloat16, device=cuda)
    base = 1000 * (layer + 1) + 100 + 3 * expert
    ops.fill_uniform_(blk[:hi * h], seed, base, math.sqrt(3.0 / h))
    ops.fill_uniform_(blk[hi * h:2 * hi * h], seed, base + 1, math.sqrt(3.0 / h))
    ops.fill_uniform_(blk[2 * hi * h:], seed, base + 2, math.sqrt(3.0 / hi))
    return blk


def test_unary_codec_full_mixtral_block(cuda, oracle):
    """K5: one whole Mixtral expert block (176 M values, 352 MB) through the
    unary link code: bit-exact round trip; ~10.25 bits/weight; a numpy
    restatement of the format decodes sampled segments identically; and the
    code an engine keeps in pinned host memory for that block is the same
    bytes."""
    import torch
    from paper_2508_21706_b200 import ops
    from paper_2508_21706_b200.engine import MIXTRAL_8X7B, VerifyEngine
    import test_gpu_kernels as K
    x = _mixtral_block(torch, cuda)
    n = x.numel()
    code, ovf = ops.expert_encode(x, 1)
    assert not ovf
    bpw = code.numel() * 8 / n
    assert 10.0 < bpw < 10.5, bpw
    y = ops.expert_decode(code, n, 1)
    assert torch.equal(y.view(torch.int16), x.view(torch.int16))
    del y
    c = code.cpu().numpy()
    xs = x.view(torch.int16).cpu().numpy().view(np.uint16)
    segs = n // 1024
    for sgm, v in K._np_unary_decode(c, n, (0, 1, segs // 3, segs // 2 + 7, segs - 1)).items():
        assert np.array_equal(v, xs[sgm * 1024:(sgm + 1) * 1024]), sgm
    # the engine's own host-resident code of (layer 0, expert 0)
    shape = dataclasses.replace(MIXTRAL_8X7B, n_layers=1)
    eng = VerifyEngine(shape, max_batch=1, max_verify=1, max_seq=64, compress_experts=True)
    ptr, nbytes = eng.tensor_ptr("expert_host", 0, 0)
    import ctypes
    host = np.ctypeslib.as_array((ctypes.c_uint8 * code.numel()).from_address(ptr)).copy()
    eng.close()
    assert np.array_equal(host, c)


def test_fused_moe_mixtral_dims_vs_torch(cuda):
    """K4-MoE at the bench's exact launch: 576 (token, slot) rows (T=288,
    top-2) over 8 Mixtral experts (h 4096, h_i 14336) with the production
    down split S (splits=0 -> the kernel's waves model) vs fp32 torch."""
    import torch
    from paper_2508_21706_b200 import ops
    h, hi, E, k, T = 4096, 14336, 8, 2, B * N
    g = torch.Generator(device=cuda).manual_seed(41)
    x = (torch.rand((T, h), generator=g, device=cuda) * 2 - 1).to(torch.bfloat16)
    blk = 3 * h * hi
    pool = torch.empty(E * blk, dtype=torch.bfloat16, device=cuda)
    for e in range(E):
        pool[e * blk:(e + 1) * blk] = _mixtral_block(torch, cuda, expert=e)
    logits = torch.randn((T, E), generator=g, device=cuda)
    ids = torch.topk(logits, k, dim=1).indices.to(torch.int32).contiguous()
    off, perm, pos, xp = ops.permute(ids, E, x)
    hbuf, ys = ops.moe_experts(xp, off, pool, h=h, h_i=hi, n_expert=E, w_block_stride=blk * 2, w_pool_blocks=E,
                               splits=0)
    ysum = ys[0].clone()
    for s_ in range(1, ys.shape[0]):
        ysum += ys[s_]
    offs = off.cpu().tolist()
    for e in range(E):
        a, b = offs[e], offs[e + 1]
        assert b > a
        base = e * blk
        w1 = pool[base:base + hi * h].view(hi, h).float()
        w3 = pool[base + hi * h:base + 2 * hi * h].view(hi, h).float()
        w2 = pool[base + 2 * hi * h:base + blk].view(h, hi).float()
        X = xp[a:b].float()
        gg, uu = X @ w1.T, X @ w3.T
        H = (gg * torch.sigmoid(gg) * uu).to(torch.bfloat16)
        dh = (hbuf[a:b].float() - H.float()).abs().max().item()
        assert dh <= 2 ** -7 * max(1.0, H.float().abs().max().item()), (e, dh)
        Y = hbuf[a:b].float() @ w2.T
        dy = (ysum[a:b] - Y).abs().max().item()
        assert dy <= 1e-4 * max(1.0, Y.abs().max().item()), (e, dy)
        del w1, w3, w2
