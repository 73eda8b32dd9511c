"""Per-kernel microbench at BASELINE config-2/3 shapes (CUDA events, L2 flushed
between reps). Prints one JSON line per kernel with achieved GB/s vs the
measured HBM peak. Usage: python tools/kbench.py [attn|gemm|all] [--sweep]"""
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2508_21706_b200 import ops, _lib as L  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        # keep the GPU busy while the host enqueues the events and the launch,
        # so the events bracket device time only (not Python / launch latency)
        torch.cuda._sleep(200_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    ts.sort()
    return ts[len(ts) // 2]


def attn(b, n, s, nq=32, nkv=8, d=128, tree=False):
    s_max = s + n + 64
    g = torch.Generator(device=dev).manual_seed(1)
    q = (torch.rand((b * n, nq, d), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
    kc = (torch.rand((b, nkv, s_max, d), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
    vc = (torch.rand((b, nkv, s_max, d), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
    if tree:  # random draft tree per request: ancestor-or-self masks (attention.hpp:41-71)
        import numpy as np
        rng = np.random.default_rng(b * 1000 + n)
        bits = []
        for _ in range(b):
            par = [-1] + [int(rng.integers(0, i)) for i in range(1, n)]
            for i in range(n):
                m, cur = 0, i
                while cur >= 0:
                    m |= 1 << cur
                    cur = par[cur] if cur > 0 else -1
                bits.append(m)
    else:
        bits = [(1 << (i + 1)) - 1 for i in range(n)] * b
    mask = torch.tensor(bits, dtype=torch.int64, device=dev)
    pre = torch.full((b,), s, dtype=torch.int32, device=dev)
    out = torch.empty_like(q)
    # persistent, zeroed workspace (K1 leaves its pair counters at zero), as the engine keeps it
    a = L.AttnArgs(q=q.data_ptr(), k_cache=kc.data_ptr(), v_cache=vc.data_ptr(), mask=mask.data_ptr(),
                   prefix_len=pre.data_ptr(), out=out.data_ptr(), b=b, n=n, n_q=nq, n_kv=nkv, d=d, s_max=s_max,
                   max_prefix=s, workspace=None, workspace_bytes=0, block_table=None, max_pages=0, num_pages=0)
    import ctypes
    wsb = L.load().smo_verify_attention_workspace(ctypes.byref(a))
    ws = torch.zeros(max(16, wsb), dtype=torch.uint8, device=dev)
    a.workspace, a.workspace_bytes = ws.data_ptr(), wsb

    def run():
        L.check(L.load().smo_verify_attention(ctypes.byref(a), torch.cuda.current_stream().cuda_stream))
    t = timeit(run)
    if os.environ.get("KBENCH_B2B"):  # A/B: mean of 20 back-to-back launches (warm L2, no carve-out switch)
        t = timeit(lambda: [run() for _ in range(20)]) / 20
    byts = 2 * b * (s + n) * nkv * d * 2 + 2 * q.numel() * 2
    return {"kernel": "K1 verify_attention", "b": b, "n": n, "s": s, "mask": "tree" if tree else "chain",
            "us": t * 1e6, "GBs": byts / t / 1e9,
            "frac": byts / t / 1e9 / PEAK, "TFLOPs": 4 * b * n * (s + n) * nq * d / t / 1e12}


def gemm(T, K, N, epi=L.EPI_BF16, name="dense"):
    g = torch.Generator(device=dev).manual_seed(2)
    x = (torch.rand((T, K), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
    w = (torch.rand((N, K), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
    out = torch.zeros((T, N), dtype=torch.float32 if epi in (L.EPI_F32, L.EPI_F32_ADD) else torch.bfloat16, device=dev)
    t = timeit(lambda: ops.gemm(x, w, epilogue=epi, out=out))
    byts = N * K * 2 + T * K * 2 + T * N * out.element_size()
    return {"kernel": f"K4 gemm {name}", "T": T, "K": K, "N": N, "us": t * 1e6, "GBs": byts / t / 1e9,
            "frac": byts / t / 1e9 / PEAK, "TFLOPs": 2 * T * K * N / t / 1e12}


def moe(T=288, h=4096, hi=14336, E=8, k=2, split=0):
    g = torch.Generator(device=dev).manual_seed(3)
    x = (torch.rand((T, h), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
    blk = 3 * h * hi
    pool = (torch.rand((E * blk,), generator=g, device=dev) * 0.02).to(torch.bfloat16)
    ids = torch.stack([torch.randperm(E, generator=g, device=dev)[:k] for _ in range(T)]).to(torch.int32)
    off, perm, pos, xp = ops.permute(ids, E, x)
    hbuf = torch.empty((T * k, hi), dtype=torch.bfloat16, device=dev)
    y = torch.empty((T * k, h), dtype=torch.float32, device=dev)

    def up():
        ops.gemm(xp, pool, epilogue=L.EPI_SWIGLU, out=hbuf, w_up=pool[hi * h:], row_offsets=off, groups=E,
                 w_block_stride=blk * 2, w_pool_blocks=E, N=hi, max_rows_per_group=T, split_k=split)

    def down():
        ops.gemm(hbuf, pool[2 * hi * h:], epilogue=L.EPI_F32, out=y, row_offsets=off, groups=E,
                 w_block_stride=blk * 2, w_pool_blocks=E, N=h, max_rows_per_group=T, split_k=split)
    y4 = torch.empty((4, T * k, h), dtype=torch.float32, device=dev)
    scratch = torch.zeros(128, dtype=torch.int32, device=dev)
    widx = torch.arange(E, dtype=torch.int32, device=dev)

    def fused():
        L.check(L.load().smo_moe_experts(xp.data_ptr(), T * k, h, hi, E, off.data_ptr(), pool.data_ptr(), blk * 2, E,
                                         widx.data_ptr(), hbuf.data_ptr(), y4.data_ptr(), split, None,
                                         scratch.data_ptr(), torch.cuda.current_stream().cuda_stream))
    r = []
    for nm, fn, wb in (("swiglu gate/up", up, 2 * E * hi * h * 2), ("down", down, E * h * hi * 2),
                       ("fused moe (gate/up + down, one kernel)", fused, 3 * E * hi * h * 2)):
        if split and "fused" not in nm:
            continue
        t = timeit(fn)
        r.append({"kernel": f"K4 grouped {nm}" + (f" split {split}" if split else ""), "T": T, "E": E, "us": t * 1e6, "GBs": wb / t / 1e9,
                  "frac": wb / t / 1e9 / PEAK, "TFLOPs": (3 if "fused" in nm else 2 if "gate" in nm else 1) * 2 * T * k * h * hi / t / 1e12})
    return r


def codec(n=3 * 4096 * 14336, bits=3, dist="uniform"):
    """K5 codec on one Mixtral expert block: decode reads the code, writes bf16.
    dist: uniform (the engine's procedural init) or gaussian (trained-like)."""
    x = torch.empty(n, dtype=torch.bfloat16, device=dev)
    (ops.fill_normal_ if dist == "gaussian" else ops.fill_uniform_)(x, 0x5EED, 1100, math.sqrt(3.0 / 4096))
    code, ovf = ops.expert_encode(x, bits)
    assert not ovf
    out = torch.empty_like(x)
    t = timeit(lambda: L.check(L.load().smo_expert_decode(code.data_ptr(), n, bits, out.data_ptr(),
                                                          torch.cuda.current_stream().cuda_stream)))
    assert torch.equal(out.view(torch.int16), x.view(torch.int16))
    byts = code.numel() + 2 * n
    name = "unary" if bits == 1 else f"{bits}-bit"
    return {"kernel": f"K5 expert_decode ({name})", "dist": dist, "N": n, "bits_per_weight": code.numel() * 8 / n,
            "us": t * 1e6, "GBs": byts / t / 1e9, "frac": byts / t / 1e9 / PEAK, "TFLOPs": 0.0}


def moe_coded(T=288, h=4096, hi=14336, E=8, k=2, dist="uniform"):
    """K4-MoE on T2-coded experts (decode in shared memory) vs the bf16
    kernel and vs unary expansion + bf16 kernel (the round-1 pipeline), on
    the engine's procedural expert init (uniform or gaussian-like)."""
    g = torch.Generator(device=dev).manual_seed(3)
    x = (torch.rand((T, h), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
    blk = 3 * h * hi
    pool = torch.empty(E * blk, dtype=torch.bfloat16, device=dev)
    fill = ops.fill_normal_ if dist == "gaussian" else ops.fill_uniform_
    for e in range(E):
        b = pool[e * blk:(e + 1) * blk]
        fill(b[:hi * h], 0x5EED, 1100 + 3 * e, math.sqrt(3.0 / h))
        fill(b[hi * h:2 * hi * h], 0x5EED, 1101 + 3 * e, math.sqrt(3.0 / h))
        fill(b[2 * hi * h:], 0x5EED, 1102 + 3 * e, math.sqrt(3.0 / hi))
    codes = [ops.tcode_encode(pool[e * blk:(e + 1) * blk], h, hi) for e in range(E)]
    codes3 = [ops.tcode_encode(pool[e * blk:(e + 1) * blk], h, hi, fmt=3) for e in range(E)]
    w_code3 = torch.tensor([c.data_ptr() for c in codes3], dtype=torch.int64, device=dev)
    ucodes = [ops.expert_encode(pool[e * blk:(e + 1) * blk], 1)[0] for e in range(E)]
    w_code = torch.tensor([c.data_ptr() for c in codes], dtype=torch.int64, device=dev)
    ids = torch.stack([torch.randperm(E, generator=g, device=dev)[:k] for _ in range(T)]).to(torch.int32)
    off, perm, pos, xp = ops.permute(ids, E, x)
    hbuf = torch.empty((T * k, hi), dtype=torch.bfloat16, device=dev)
    y4 = torch.empty((4, T * k, h), dtype=torch.float32, device=dev)
    scratch = torch.zeros(128, dtype=torch.int32, device=dev)
    widx = torch.arange(E, dtype=torch.int32, device=dev)
    st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731

    def plain():
        L.check(L.load().smo_moe_experts(xp.data_ptr(), T * k, h, hi, E, off.data_ptr(), pool.data_ptr(), blk * 2, E,
                                         widx.data_ptr(), hbuf.data_ptr(), y4.data_ptr(), 0, None,
                                         scratch.data_ptr(), st()))

    def coded():
        L.check(L.load().smo_moe_experts_coded(xp.data_ptr(), T * k, h, hi, E, off.data_ptr(), w_code.data_ptr(),
                                               hbuf.data_ptr(), y4.data_ptr(), 0, None, scratch.data_ptr(), st()))

    def coded3():
        L.check(L.load().smo_moe_experts_coded3(xp.data_ptr(), T * k, h, hi, E, off.data_ptr(), w_code3.data_ptr(),
                                                hbuf.data_ptr(), y4.data_ptr(), 0, None, scratch.data_ptr(), st()))

    def unary_then_plain():
        for e in range(E):
            L.check(L.load().smo_expert_decode(ucodes[e].data_ptr(), blk, 1, pool[e * blk:].data_ptr(), st()))
        plain()
    cb = sum(c.numel() for c in codes)
    cb3 = sum(c.numel() for c in codes3)
    ub = sum(c.numel() for c in ucodes)
    act = T * k * h * 2 * 2 + T * k * hi * 2 * 2 + T * k * h * 4  # x rows (gate/up), H write + read, y
    r = []
    for nm, fn, byts, wb in (("bf16 weights", plain, E * blk * 2, E * blk * 2),
                             ("T2-coded weights, decoded in smem", coded, cb, cb),
                             ("T3-coded weights, decoded in smem", coded3, cb3, cb3),
                             ("unary expansion (8 launches) + bf16 kernel", unary_then_plain, ub + 2 * E * blk * 2, ub)):
        t = timeit(fn)
        r.append({"kernel": f"K4-MoE {nm}", "dist": dist, "T": T, "E": E, "us": t * 1e6,
                  "weight_bytes": wb, "bits_per_weight": wb * 8 / (E * blk), "GBs": byts / t / 1e9,
                  "frac": byts / t / 1e9 / PEAK, "GBs_incl_act": (byts + act) / t / 1e9,
                  "TFLOPs": 3 * 2 * T * k * h * hi / t / 1e12})
    return r


def tcode_dec(h=4096, hi=14336, dist="uniform"):
    """K5 tile code (T2) standalone expansion of one Mixtral expert block to bf16."""
    n = 3 * h * hi
    x = torch.empty(n, dtype=torch.bfloat16, device=dev)
    fill = ops.fill_normal_ if dist == "gaussian" else ops.fill_uniform_
    fill(x[:hi * h], 0x5EED, 1100, math.sqrt(3.0 / h))
    fill(x[hi * h:2 * hi * h], 0x5EED, 1101, math.sqrt(3.0 / h))
    fill(x[2 * hi * h:], 0x5EED, 1102, math.sqrt(3.0 / hi))
    code = ops.tcode_encode(x, h, hi)
    out = torch.empty_like(x)
    t = timeit(lambda: L.check(L.load().smo_tcode_decode(code.data_ptr(), h, hi, out.data_ptr(),
                                                         torch.cuda.current_stream().cuda_stream)))
    assert torch.equal(out.view(torch.int16), x.view(torch.int16))
    byts = code.numel() + 2 * n
    return {"kernel": "K5 tcode_decode (T2 tile code -> bf16)", "dist": dist, "N": n,
            "bits_per_weight": code.numel() * 8 / n, "us": t * 1e6, "GBs": byts / t / 1e9, "frac": byts / t / 1e9 / PEAK,
            "TFLOPs": 0.0}


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    res = []
    if what in ("attn", "all"):
        res.append(attn(32, 9, 1024))
        res.append(attn(32, 5, 1024))
        if "--sweep" in sys.argv:  # BASELINE config 3 / SURVEY.md §8(d): the full grid, chain and tree
            for s in (1024, 2048, 4096, 8192, 16384, 32768):
                for n in (1, 2, 4, 8, 16):
                    for b in (1, 4, 16, 32, 64):
                        for tree in ((False, True) if n > 2 else (False,)):
                            r = attn(b, n, s, tree=tree)
                            print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()}),
                                  flush=True)
                        torch.cuda.empty_cache()
            return
    if what == "attnsmall":  # latency end of config 3 (split-KV merge, launch floor)
        for b, n, s in ((1, 1, 1024), (1, 9, 1024), (4, 9, 1024), (1, 9, 4096), (1, 1, 32768), (16, 9, 1024),
                        (32, 9, 1024), (64, 16, 1024)):
            res.append(attn(b, n, s))
    if what in ("codec", "all"):
        res.append(codec(bits=3))
        res.append(codec(bits=1))
        res.append(codec(bits=1, dist="gaussian"))
    if what in ("tcode", "all"):
        res.append(tcode_dec())
        res.append(tcode_dec(dist="gaussian"))
        res.append(codec(bits=1))
    if what in ("moecoded", "all"):
        res += moe_coded()
        res += moe_coded(dist="gaussian")
    if what in ("gemm", "all"):
        res.append(gemm(288, 4096, 6144, name="qkv"))
        res.append(gemm(288, 4096, 4096, L.EPI_F32_ADD, name="o-proj (+residual)"))
        res.append(gemm(288, 4096, 32000, L.EPI_ARGMAX, name="lm-head argmax"))
        res += moe()
        if "--splits" in sys.argv:
            for sp in (1, 2, 4):
                res += moe(split=sp)
    for r in res:
        print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()}))


if __name__ == "__main__":
    main()
