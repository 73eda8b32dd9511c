"""Torch-tensor front end over the C-ABI kernels (K1-K6 and support ops).

Every function here launches sm_100a kernels from libspecmoe.so on the current
torch CUDA stream; tensors must be CUDA tensors. There is no CPU path: on a
machine without the library or a GPU these raise.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import _lib as L

_BF16 = torch.bfloat16


def _p(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _req(t: torch.Tensor, dtype, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name}: expected a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: expected a contiguous tensor")


def fill_uniform_(t: torch.Tensor, seed: int, tensor_id: int, scale: float, base: int = 0) -> torch.Tensor:
    """Procedural bf16 init, identical to the oracle's."""
    _req(t, _BF16, "fill_uniform_")
    L.check(L.load().smo_fill_uniform_bf16(_p(t), t.numel(), seed, tensor_id, base, scale, _stream()))
    return t


def fill_normal_(t: torch.Tensor, seed: int, tensor_id: int, scale: float, base: int = 0) -> torch.Tensor:
    """Trained-weight-like procedural init (c_api.h smo_fill_normal_bf16),
    identical to the oracle's orc_fill_normal_bf16."""
    _req(t, _BF16, "fill_normal_")
    L.check(L.load().smo_fill_normal_bf16(_p(t), t.numel(), seed, tensor_id, base, scale, _stream()))
    return t


def verify_attention(q, k_cache, v_cache, mask, prefix_len, max_prefix: int, out=None, block_table=None):
    """K1. q [b*n, n_q, d] bf16; caches [b, n_kv, s_max, d] bf16 — or, with
    block_table int32 [b, max_pages], page pools [num_pages, n_kv, 128, d];
    mask int64 [b*n] (bit j = draft j visible); prefix_len int32 [b].
    Returns out [b*n, n_q, d]."""
    T, n_q, d2 = q.shape
    if block_table is not None:
        _req(block_table, torch.int32, "block_table")
        b, max_pages = block_table.shape
        num_pages, n_kv, page, d = k_cache.shape
        if page != 128:
            raise ValueError("attention: pages hold 128 tokens")
        s_max = 128 * max_pages
    else:
        b, n_kv, s_max, d = k_cache.shape
        max_pages = num_pages = 0
    if d2 != d or T % b:
        raise ValueError("attention: shape mismatch")
    n = T // b
    for t, nm in ((q, "q"), (k_cache, "k_cache"), (v_cache, "v_cache")):
        _req(t, _BF16, nm)
    _req(mask, torch.int64, "mask")
    _req(prefix_len, torch.int32, "prefix_len")
    out = torch.empty_like(q) if out is None else out
    a = L.AttnArgs(q=q.data_ptr(), k_cache=k_cache.data_ptr(), v_cache=v_cache.data_ptr(), mask=mask.data_ptr(),
                   prefix_len=prefix_len.data_ptr(), out=out.data_ptr(), b=b, n=n, n_q=n_q, n_kv=n_kv, d=d,
                   s_max=s_max, max_prefix=int(max_prefix), workspace=None, workspace_bytes=0,
                   block_table=None if block_table is None else block_table.data_ptr(), max_pages=max_pages,
                   num_pages=num_pages)
    lib = L.load()
    ws_bytes = lib.smo_verify_attention_workspace(C.byref(a))
    if ws_bytes == C.c_size_t(-1).value:
        L.check(L.SMO_INVALID_ARG)
    # zero-filled: K1 keeps per-pair counters there (and leaves them at zero)
    ws = torch.zeros(max(16, ws_bytes), dtype=torch.uint8, device=q.device) if ws_bytes else None
    if ws is not None:
        a.workspace = ws.data_ptr()
        a.workspace_bytes = ws_bytes
    L.check(lib.smo_verify_attention(C.byref(a), _stream()))
    return out


def cpu_verify_attention(q, k_cache, v_cache, mask, prefix_len, threads: int = 0):
    """Host verification attention (AttentionPlacement::CPU)
    on numpy arrays: q uint16(bf16) [b*n, n_q, d], caches [b, n_kv, s_max, d],
    mask uint64 [b*n], prefix_len int32 [b]. Returns bf16 bits [b*n, n_q, d]."""
    import numpy as np
    b, n_kv, s_max, d = k_cache.shape
    T, n_q, _ = q.shape
    arrs = [np.ascontiguousarray(x) for x in (q, k_cache, v_cache)]
    m = np.ascontiguousarray(mask, np.uint64)
    pre = np.ascontiguousarray(prefix_len, np.int32)
    out = np.zeros((T, n_q, d), np.uint16)
    vp = lambda a: a.ctypes.data  # noqa: E731
    a = L.AttnArgs(q=vp(arrs[0]), k_cache=vp(arrs[1]), v_cache=vp(arrs[2]), mask=vp(m), prefix_len=vp(pre),
                   out=vp(out), b=b, n=T // b, n_q=n_q, n_kv=n_kv, d=d, s_max=s_max, max_prefix=int(pre.max()))
    L.check(L.load().smo_cpu_verify_attention(C.byref(a), threads))
    return out


def moe_experts(x_perm, offsets, pool, *, h: int, h_i: int, n_expert: int, w_block_stride: int,
                w_pool_blocks: int, w_index=None, splits: int = 0):
    """K4-MoE (one persistent kernel): x_perm bf16 [rows, h] grouped by
    offsets int32 [E+1]; pool = base of [W1 | W3 | W2] blocks. Returns
    (h_out bf16 [rows, h_i], y f32 [S, rows, h]); the down projection is
    y.sum(0) taken in slice order (S = splits, 0 = the kernel's choice)."""
    _req(x_perm, _BF16, "x_perm")
    rows = x_perm.shape[0]
    dev = x_perm.device
    if w_index is None:
        w_index = torch.arange(n_expert, dtype=torch.int32, device=dev)
    hout = torch.empty((rows, h_i), dtype=_BF16, device=dev)
    y = torch.empty((splits or 4, rows, h), dtype=torch.float32, device=dev)
    scratch = torch.zeros(128, dtype=torch.int32, device=dev)
    used = C.c_int32(0)
    L.check(L.load().smo_moe_experts(_p(x_perm), rows, h, h_i, n_expert, _p(offsets), _p(pool), w_block_stride,
                                     w_pool_blocks, _p(w_index), _p(hout), _p(y), splits, C.byref(used), _p(scratch),
                                     _stream()))
    return hout, y[:used.value]


def moe_experts_coded(x_perm, offsets, w_code, *, h: int, h_i: int, n_expert: int, splits: int = 0, fmt: int = 2):
    """K4-MoE on tile-coded experts (fmt 2: T2, 3: T3): w_code = int64 device
    tensor [E] of code block addresses (tcode_encode outputs of that format).
    Same returns as moe_experts."""
    _req(x_perm, _BF16, "x_perm")
    rows = x_perm.shape[0]
    dev = x_perm.device
    hout = torch.empty((rows, h_i), dtype=_BF16, device=dev)
    y = torch.empty((splits or 4, rows, h), dtype=torch.float32, device=dev)
    scratch = torch.zeros(80, dtype=torch.int32, device=dev)
    used = C.c_int32(0)
    fn = L.load().smo_moe_experts_coded3 if fmt == 3 else L.load().smo_moe_experts_coded
    L.check(fn(_p(x_perm), rows, h, h_i, n_expert, _p(offsets), _p(w_code), _p(hout), _p(y), splits, C.byref(used),
               _p(scratch), _stream()))
    return hout, y[:used.value]


def tcode_encode(block, h: int, h_i: int, fmt: int = 2):
    """T2 (fmt 2) or T3 (fmt 3) tile code of one expert block [W1 | W3 | W2]
    (bf16, device): uint8 device tensor trimmed to the bytes used (16-B
    aligned storage)."""
    _req(block, _BF16, "block")
    assert block.numel() == 3 * h * h_i and fmt in (2, 3)
    code = torch.empty(int(L.load().smo_tcode_max_bytes(h, h_i)), dtype=torch.uint8, device=block.device)
    n = C.c_uint64(0)
    fn = L.load().smo_tcode3_encode if fmt == 3 else L.load().smo_tcode_encode
    L.check(fn(_p(block), h, h_i, _p(code), C.byref(n), _stream()))
    return code[:n.value]


def tcode_decode(code, h: int, h_i: int, fmt: int = 2):
    """Inverse of tcode_encode: the bf16 block [W1 | W3 | W2] (3 h h_i values)."""
    out = torch.empty(3 * h * h_i, dtype=_BF16, device=code.device)
    fn = L.load().smo_tcode3_decode if fmt == 3 else L.load().smo_tcode_decode
    L.check(fn(_p(code), h, h_i, _p(out), _stream()))
    return out


def expert_encode(x, bits: int = 3):
    """Lossless code of a bf16 tensor (numel % 1024 == 0) with `bits`-bit
    exponent codes (bits = 1: the variable-length unary code): returns
    (uint8 code, overflow) — overflow means a segment needed > 32 escapes
    (retry with 4 bits or keep the tensor raw); unary never overflows and its
    code is trimmed to the bytes used."""
    _req(x, _BF16, "x")
    n = x.numel()
    code = torch.empty(int(L.load().smo_expert_code_bytes(n, bits)), dtype=torch.uint8, device=x.device)
    ovf = torch.zeros(1, dtype=torch.int32, device=x.device)
    L.check(L.load().smo_expert_encode(_p(x), n, bits, _p(code), _p(ovf), _stream()))
    if bits == 1:
        code = code[:int(L.load().smo_expert_coded_size(_p(code), n, bits))]
    return code, bool(ovf.item())


def expert_decode(code, n: int, bits: int = 3):
    """Inverse of expert_encode: n bf16 values."""
    out = torch.empty(n, dtype=_BF16, device=code.device)
    L.check(L.load().smo_expert_decode(_p(code), n, bits, _p(out), _stream()))
    return out


def router_topk(x, w_router, k: int, want_logits: bool = False):
    """K2. x [T, h] bf16, w_router [E, h] bf16 -> ids int32 [T,k], weights f32 [T,k] (, logits)."""
    _req(x, _BF16, "x")
    _req(w_router, _BF16, "w_router")
    T, h = x.shape
    E = w_router.shape[0]
    ids = torch.empty((T, k), dtype=torch.int32, device=x.device)
    wts = torch.empty((T, k), dtype=torch.float32, device=x.device)
    logits = torch.empty((T, E), dtype=torch.float32, device=x.device) if want_logits else None
    L.check(L.load().smo_router_topk(_p(x), _p(w_router), T, h, E, k, _p(logits), _p(ids), _p(wts), _stream()))
    return (ids, wts, logits) if want_logits else (ids, wts)


def permute(ids, n_expert: int, x=None):
    """K3. ids [T,k] int32 -> offsets [E+1], perm [T*k], pos [T*k] (, x_perm [T*k, h])."""
    _req(ids, torch.int32, "ids")
    T, k = ids.shape
    dev = ids.device
    offsets = torch.empty(n_expert + 1, dtype=torch.int32, device=dev)
    perm = torch.empty(T * k, dtype=torch.int32, device=dev)
    pos = torch.empty(T * k, dtype=torch.int32, device=dev)
    xp = None
    h = 0
    if x is not None:
        _req(x, _BF16, "x")
        h = x.shape[1]
        xp = torch.empty((T * k, h), dtype=_BF16, device=dev)
    L.check(L.load().smo_permute(_p(ids), T, k, n_expert, _p(x), h, _p(offsets), _p(perm), _p(pos), _p(xp),
                                 _stream()))
    return offsets, perm, pos, xp


def unpermute_combine_(residual, y_perm, pos, weights):
    """K3 combine: residual[t] += sum_j weights[t,j] * y_perm[pos[t*k+j]] (in place)."""
    _req(residual, torch.float32, "residual")
    _req(y_perm, torch.float32, "y_perm")
    T, h = residual.shape
    k = weights.shape[1]
    L.check(L.load().smo_unpermute_combine(_p(y_perm), _p(pos), _p(weights), T, k, h, _p(residual), _stream()))
    return residual


def gemm(x, w, *, epilogue=L.EPI_BF16, out=None, w_up=None, row_offsets=None, w_index=None,
         groups: int = 1, w_block_stride: int = 0, w_pool_blocks: int = 1, N: Optional[int] = None,
         max_rows_per_group: Optional[int] = None, split_k: int = 0):
    """K4 (tcgen05). out[t, n] = x[t] . W_g[n] for the rows of group g.
    Dense: w [N, K]. Grouped: w is a pool base pointer tensor and N must be given."""
    _req(x, _BF16, "x")
    rows, K = x.shape
    if N is None:
        N = w.shape[0]
    dev = x.device
    amax_v = amax_i = None
    if epilogue == L.EPI_ARGMAX:
        amax_v = torch.empty((rows, N // 128), dtype=torch.float32, device=dev)
        amax_i = torch.empty((rows, N // 128), dtype=torch.int32, device=dev)
    elif out is None:
        dt = _BF16 if epilogue in (L.EPI_BF16, L.EPI_SWIGLU) else torch.float32
        out = torch.zeros((rows, N), dtype=dt, device=dev)
    a = L.GemmArgs(x=x.data_ptr(), rows=rows, K=K, N=N, groups=groups,
                   row_offsets=None if row_offsets is None else row_offsets.data_ptr(),
                   max_rows_per_group=max_rows_per_group or rows, w=w.data_ptr(),
                   w_up=None if w_up is None else w_up.data_ptr(), w_block_stride=w_block_stride,
                   w_pool_blocks=w_pool_blocks, w_index=None if w_index is None else w_index.data_ptr(),
                   epilogue=epilogue, out=None if out is None else out.data_ptr(),
                   ldo=0 if out is None else out.shape[-1],
                   argmax_val=None if amax_v is None else amax_v.data_ptr(),
                   argmax_idx=None if amax_i is None else amax_i.data_ptr(), split_k=split_k)
    ws_bytes = L.load().smo_gemm_workspace(C.byref(a))
    if ws_bytes == C.c_size_t(-1).value:
        L.check(L.SMO_INVALID_ARG)
    ws = torch.empty(max(16, ws_bytes), dtype=torch.uint8, device=dev) if ws_bytes else None
    if ws is not None:
        a.workspace, a.workspace_bytes = ws.data_ptr(), ws_bytes
    L.check(L.load().smo_gemm(C.byref(a), _stream()))
    if epilogue == L.EPI_ARGMAX:
        return amax_v, amax_i
    return out


def rmsnorm(x, gain, eps: float):
    _req(x, torch.float32, "x")
    y = torch.empty(x.shape, dtype=_BF16, device=x.device)
    L.check(L.load().smo_rmsnorm(_p(x), _p(gain), x.shape[0], x.shape[1], eps, _p(y), _stream()))
    return y


def embed(tokens, table):
    _req(tokens, torch.int32, "tokens")
    x = torch.empty((tokens.numel(), table.shape[1]), dtype=torch.float32, device=tokens.device)
    L.check(L.load().smo_embed(_p(tokens), _p(table), tokens.numel(), table.shape[1], _p(x), _stream()))
    return x


def rope_append(qkv, prefix_len, parent, b, n, n_q, n_kv, d, k_cache, v_cache, theta):
    q = torch.empty((b * n, n_q, d), dtype=_BF16, device=qkv.device)
    L.check(L.load().smo_rope_append(_p(qkv), _p(prefix_len), _p(parent), b, n, n_q, n_kv, d, k_cache.shape[2],
                                     theta, _p(q), _p(k_cache), _p(v_cache), _stream()))
    return q


def argmax_reduce(val, idx):
    rows, parts = val.shape
    t = torch.empty(rows, dtype=torch.int32, device=val.device)
    L.check(L.load().smo_argmax_reduce(_p(val), _p(idx), rows, parts, _p(t), _stream()))
    return t


def argmax_rows(logits):
    _req(logits, torch.float32, "logits")
    rows, V = logits.shape
    t = torch.empty(rows, dtype=torch.int32, device=logits.device)
    L.check(L.load().smo_argmax_rows(_p(logits), rows, V, _p(t), _stream()))
    return t


def greedy_accept(tokens, target, b: int, n: int, parent=None):
    """K6. tokens/target int32 [b*n] -> acc_len [b], bonus [b], keep [b*n]."""
    dev = tokens.device
    acc = torch.empty(b, dtype=torch.int32, device=dev)
    bonus = torch.empty(b, dtype=torch.int32, device=dev)
    keep = torch.empty(b * n, dtype=torch.int32, device=dev)
    L.check(L.load().smo_greedy_accept(_p(tokens), _p(target), _p(parent), b, n, _p(acc), _p(bonus), _p(keep),
                                       _stream()))
    return acc, bonus, keep


def kv_rollback(k_caches, v_caches, prefix_len, acc_len, keep, b, n):
    """Tree KV compaction over all layers; returns kv_len [b] = prefix + acc + 1."""
    dev = prefix_len.device
    n_kv, s_max, d = k_caches[0].shape[1:]
    kp = torch.tensor([t.data_ptr() for t in k_caches], dtype=torch.int64, device=dev)
    vp = torch.tensor([t.data_ptr() for t in v_caches], dtype=torch.int64, device=dev)
    kv_len = torch.empty(b, dtype=torch.int32, device=dev)
    L.check(L.load().smo_kv_rollback(_p(kp), _p(vp), len(k_caches), _p(prefix_len), _p(acc_len), _p(keep), b, n,
                                     n_kv, d, s_max, _p(kv_len), _stream()))
    return kv_len


class ExpertStreamer:
    """K5 expert streamer handle (smo_streamer_*): blocks in pinned host
    memory -> double-buffered HBM slots on a copy-engine stream, hot-expert
    cache, coded blocks expanded on the consumer stream.

    host_blocks: list (layer-major, n_layers * n_experts) of pinned uint8 CPU
    tensors — raw bf16 blocks of `block_bytes`, or K5 codes (then `codes`
    gives 1 / 3 / 4 per block). The caller keeps them alive."""

    def __init__(self, host_blocks, n_layers: int, n_experts: int, block_bytes: int, codes=None,
                 hbm_slots: int = 2, cache_bytes: int = 0, device: int = 0):
        n = n_layers * n_experts
        assert len(host_blocks) == n
        for t in host_blocks:
            assert t.is_pinned(), "streamer: host blocks must be pinned"
        self._ptrs = (C.c_void_p * n)(*[t.data_ptr() for t in host_blocks])
        self._bytes = (C.c_uint64 * n)(*[t.numel() * t.element_size() for t in host_blocks])
        self._codes = (C.c_int32 * n)(*(codes if codes is not None else [0] * n))
        a = L.StreamerArgs(n_layers=n_layers, n_experts=n_experts, block_bytes=block_bytes,
                           host_blocks=C.cast(self._ptrs, C.c_void_p), host_bytes=C.cast(self._bytes, C.c_void_p),
                           host_codes=C.cast(self._codes, C.c_void_p), hbm_slots=hbm_slots,
                           cache_bytes=cache_bytes, device=device)
        self.handle = C.c_void_p()
        L.check(L.load().smo_streamer_create(C.byref(a), C.byref(self.handle)))
        self.n_experts, self.block_bytes = n_experts, block_bytes

    def enqueue_layer(self, layer: int, active=None):
        buf = None
        if active is not None:
            buf = (C.c_uint8 * self.n_experts)(*[1 if x else 0 for x in active])
        L.check(L.load().smo_streamer_enqueue_layer(self.handle, layer, buf))

    def wait_layer(self, layer: int, stream=None):
        L.check(L.load().smo_streamer_wait_layer(self.handle, layer, stream if stream is not None else _stream()))

    def release_layer(self, layer: int, stream=None):
        L.check(L.load().smo_streamer_release_layer(self.handle, layer, stream if stream is not None else _stream()))

    def expert_ptr(self, layer: int, expert: int) -> int:
        p = C.c_void_p()
        L.check(L.load().smo_streamer_expert_ptr(self.handle, layer, expert, C.byref(p)))
        return p.value

    def ready_event(self, layer: int) -> int:
        ev = C.c_void_p()
        L.check(L.load().smo_streamer_expert_ready_event(self.handle, layer, C.byref(ev)))
        return ev.value

    def close(self):
        if getattr(self, "handle", None):
            L.load().smo_streamer_destroy(self.handle)
            self.handle = None
