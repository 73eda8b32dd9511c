"""VerifyEngine: Python handle over smo_engine_* (the measured verify step).

Mirrors the additive engine API of SURVEY.md §8(b): construct from a model
shape + options, `verify(batch)` runs one speculative verification step
(the reference's target DAG, pipeline.hpp:147-206, realised on CUDA streams)
and returns the greedy accept result; `last_times()` returns the measured
stage durations in the reference's IterationBreakdown vocabulary
(report.hpp:27-37).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib as L


@dataclass
class ModelShape:
    hidden: int
    inter: int
    n_expert: int
    top_k: int
    n_layers: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    vocab: int
    rope_theta: float = 1e6
    rms_eps: float = 1e-5
    seed: int = 0x5EED
    lm_scale: float = 1.0
    router_scale: float = 1.0
    shared_inter: int = 0  # always-on shared expert (config 4), resident in HBM
    draft_layers: int = 0  # drafter depth (DraftModelSpec.n_layers); 0: no drafter
    draft_inter: int = 0   # drafter dense SwiGLU width
    expert_init: int = 0   # 0: uniform (default), 1: gaussian-like trained weights (L.INIT_GAUSSIAN)

    @property
    def expert_bytes(self) -> int:
        return 3 * self.hidden * self.inter * 2

    def to_c(self) -> L.ModelConfig:
        return L.ModelConfig(self.hidden, self.inter, self.n_expert, self.top_k, self.n_layers, self.n_q_heads,
                             self.n_kv_heads, self.head_dim, self.vocab, self.rope_theta, self.rms_eps, self.seed,
                             self.lm_scale, self.router_scale, self.shared_inter, self.draft_layers,
                             self.draft_inter, self.expert_init)


# BASELINE.json configs
TINY = ModelShape(hidden=512, inter=1792, n_expert=8, top_k=2, n_layers=2, n_q_heads=8, n_kv_heads=2,
                  head_dim=64, vocab=32000)
MIXTRAL_8X7B = ModelShape(hidden=4096, inter=14336, n_expert=8, top_k=2, n_layers=32, n_q_heads=32,
                          n_kv_heads=8, head_dim=128, vocab=32000)
MIXTRAL_8X22B = ModelShape(hidden=6144, inter=16384, n_expert=8, top_k=2, n_layers=56, n_q_heads=48,
                           n_kv_heads=8, head_dim=128, vocab=32000)
# BASELINE config 4: DeepSeek-V2-Lite-shaped fine-grained MoE (64 routed experts
# top-6 + 2 shared experts of 1408 = one shared SwiGLU of 2816); GQA stands in
# for MLA (not in the reference model).
DSV2_LITE = ModelShape(hidden=2048, inter=1408, n_expert=64, top_k=6, n_layers=26, n_q_heads=16, n_kv_heads=4,
                       head_dim=128, vocab=102400, shared_inter=2816)
# Qwen2-57B-A14B-shaped: 64 experts top-8 + shared expert 20480
QWEN2_57B = ModelShape(hidden=3584, inter=2560, n_expert=64, top_k=8, n_layers=28, n_q_heads=28, n_kv_heads=4,
                       head_dim=128, vocab=151552, shared_inter=20480)


class EpGroup:
    """Expert-parallel transport (smo_ep_group): NCCL across processes, or an
    in-process loopback group for P engines on one device."""

    def __init__(self, handle, size: int = 0):
        self.handle = handle
        self.size = size

    @staticmethod
    def loopback(ep_size: int) -> "EpGroup":
        h = C.c_void_p()
        L.check(L.load().smo_ep_loopback_create(ep_size, C.byref(h)))
        return EpGroup(h, ep_size)

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        L.check(L.load().smo_nccl_unique_id(buf))
        return bytes(buf)

    @staticmethod
    def nccl(unique_id: bytes, nranks: int, rank: int) -> "EpGroup":
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        L.check(L.load().smo_ep_nccl_create(buf, nranks, rank, C.byref(h)))
        return EpGroup(h, nranks)

    BARRIER_FN = C.CFUNCTYPE(None, C.c_void_p)

    @staticmethod
    def workspace_bytes(P: int, T: int, k: int, h: int, E: int, C: int) -> int:
        return int(L.load().smo_ep_workspace(P, T, k, h, E, C))

    def dispatch(self, rank: int, x, ids, n_expert: int, capacity: int, workspace, stream: int = 0):
        """smo_ep_dispatch: x bf16 [T,h], ids int32 [T,k] (device tensors) ->
        (xl bf16 [P*C,h], offsets_l int32 [E/P+1], back int32 [P*C],
        pos_ep int32 [T*k]); collective over the group."""
        import torch
        T, h = x.shape
        k = ids.shape[1]
        P = self.size
        xl = torch.empty((P * capacity, h), dtype=torch.bfloat16, device=x.device)
        offsets_l = torch.empty(n_expert // P + 1, dtype=torch.int32, device=x.device)
        back = torch.empty(P * capacity, dtype=torch.int32, device=x.device)
        pos_ep = torch.empty(T * k, dtype=torch.int32, device=x.device)
        L.check(L.load().smo_ep_dispatch(self.handle, rank, x.data_ptr(), ids.data_ptr(), T, k, h, n_expert, capacity,
                                         xl.data_ptr(), offsets_l.data_ptr(), back.data_ptr(), pos_ep.data_ptr(),
                                         workspace.data_ptr(), stream))
        return xl, offsets_l, back, pos_ep

    def combine(self, rank: int, yl, back, offsets_l, pos_ep, weights, x, n_expert: int, capacity: int, workspace,
                stream: int = 0):
        """smo_ep_combine: x fp32 [T,h] += sum_j weights[t,j] * expert output."""
        T, h = x.shape
        k = weights.numel() // T
        L.check(L.load().smo_ep_combine(self.handle, rank, yl.data_ptr(), back.data_ptr(), offsets_l.data_ptr(),
                                        pos_ep.data_ptr(), weights.data_ptr(), T, k, h, n_expert, capacity,
                                        x.data_ptr(), workspace.data_ptr(), stream))

    @staticmethod
    def ipc(nranks: int, rank: int, slot_bytes: int, all_gather, barrier) -> "EpGroup":
        """Peer-memory transport over CUDA IPC (no NCCL): `all_gather(bytes)`
        returns every rank's bytes in rank order and `barrier()` synchronises
        the ranks (e.g. torch.distributed over gloo)."""
        lib = L.load()
        blob = (C.c_uint8 * int(lib.smo_ep_ipc_handle_bytes()))()
        h = C.c_void_p()
        L.check(lib.smo_ep_ipc_create(nranks, rank, slot_bytes, C.byref(h), blob))
        allb = b"".join(all_gather(bytes(blob)))
        buf = (C.c_uint8 * len(allb)).from_buffer_copy(allb)
        cb = EpGroup.BARRIER_FN(lambda _ctx: barrier())
        L.check(lib.smo_ep_ipc_connect(h, buf, C.cast(cb, C.c_void_p), None))
        g = EpGroup(h, nranks)
        g._keep = cb  # the callback must outlive the group
        return g

    @staticmethod
    def ipc_slot_bytes(shape: "ModelShape", max_batch: int, max_verify: int) -> int:
        """Mailbox slot that fits the engine's dispatch and combine blocks, a
        whole number of fp32 rows so the engine can use direct (peer-store)
        dispatch / combine into it."""
        rows = max_batch * max_verify * shape.top_k
        row = shape.hidden * 4
        dispatch = rows * shape.hidden * 2 + 16 + 4 * shape.n_expert
        return max(rows, -(-dispatch // row)) * row

    def close(self):
        if getattr(self, "handle", None):
            L.load().smo_ep_group_destroy(self.handle)
            self.handle = None


@dataclass
class VerifyResult:
    acc_len: np.ndarray
    bonus: np.ndarray
    keep: np.ndarray
    target: np.ndarray


class VerifyEngine:
    def __init__(self, shape: ModelShape, *, max_batch: int, max_verify: int, max_seq: int, hbm_slots: int = 2,
                 expert_cache_bytes: int = 0, host_alias_layers: int = 0, device: int = 0, debug: bool = False,
                 ep_rank: int = 0, ep_size: int = 1, ep_group: Optional["EpGroup"] = None, kv_pages: int = 0,
                 attn_cpu: bool = False, batch_one: bool = False, compress_experts: int = 0,
                 micro_batches: int = 1, draft_cpu_kv: bool = False):
        self.shape = shape
        self.max_batch, self.max_verify, self.max_seq = max_batch, max_verify, max_seq
        if ep_size > 1 and ep_group is None:
            raise ValueError("ep_size > 1 needs an EpGroup (nccl or loopback)")
        if ep_group is not None:
            ep_size = max(1, ep_size)
        self._group = ep_group  # keep the transport alive as long as the engine
        opt = L.EngineOptions(max_batch, max_verify, max_seq, hbm_slots, int(expert_cache_bytes),
                              host_alias_layers, device, L.ENGINE_DEBUG if debug else 0, ep_rank, ep_size,
                              None if ep_group is None else ep_group.handle, kv_pages, int(attn_cpu),
                              int(batch_one), int(compress_experts), int(micro_batches), int(draft_cpu_kv))
        cfg = shape.to_c()
        h = C.c_void_p()
        L.check(L.load().smo_engine_create(C.byref(cfg), C.byref(opt), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            L.load().smo_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_micro_batches(self, m: int) -> None:
        """Hyperparameters.m for the next steps (stage-major micro-batches)."""
        L.check(L.load().smo_engine_set_micro_batches(self._h, int(m)))

    def layer_times(self):
        """Measured per-layer timeline of the last step: (m, array [L, 4 + 6m])
        (c_api.h smo_engine_layer_times)."""
        lib = L.load()
        m = C.c_int32(0)
        L.check(lib.smo_engine_last_micro_batches(self._h, C.byref(m)))
        out = np.zeros((self.shape.n_layers, 4 + 6 * m.value))
        L.check(lib.smo_engine_layer_times(self._h, out.ctypes.data_as(C.c_void_p), out.size))
        return m.value, out

    def fill_prefix(self, prefix_len) -> None:
        p = np.ascontiguousarray(prefix_len, np.int32)
        L.check(L.load().smo_engine_fill_prefix(self._h, p.ctypes.data_as(C.c_void_p), p.size))

    def verify(self, tokens, prefix_len, parent=None, stream: Optional[int] = None) -> VerifyResult:
        """One verify step from HOST arrays (the e2e path): tokens [b, n] int32
        (column 0 = root), prefix_len [b]; parent [b, n] (tree) or None (chain)."""
        tok = np.ascontiguousarray(tokens, np.int32)
        b, n = tok.shape
        pre = np.ascontiguousarray(prefix_len, np.int32)
        par = None if parent is None else np.ascontiguousarray(parent, np.int32)
        vp = lambda a: None if a is None else a.ctypes.data_as(C.c_void_p)  # noqa: E731
        acc = np.zeros(b, np.int32)
        bonus = np.zeros(b, np.int32)
        keep = np.zeros(b * n, np.int32)
        target = np.zeros(b * n, np.int32)
        inp = L.VerifyBatch(b, n, vp(tok), vp(par), vp(pre), 0)
        out = L.VerifyOutput(vp(acc), vp(bonus), vp(keep), vp(target), 0)
        L.check(L.load().smo_engine_verify(self._h, C.byref(inp), C.byref(out), C.c_void_p(stream or 0)))
        return VerifyResult(acc, bonus, keep.reshape(b, n), target.reshape(b, n))

    def verify_device(self, tokens, prefix_len, acc, bonus, parent=None, keep=None, target=None,
                      stream: Optional[int] = None) -> None:
        """Device-resident variant (torch CUDA tensors); asynchronous."""
        b, n = tokens.shape
        p = lambda t: None if t is None else C.c_void_p(t.data_ptr())  # noqa: E731
        inp = L.VerifyBatch(b, n, p(tokens), p(parent), p(prefix_len), 1)
        out = L.VerifyOutput(p(acc), p(bonus), p(keep), p(target), 1)
        L.check(L.load().smo_engine_verify(self._h, C.byref(inp), C.byref(out), C.c_void_p(stream or 0)))

    # ------------------------------------------------------------ decode loop
    def prefill(self, prompts, stream: Optional[int] = None) -> np.ndarray:
        """Run prompts (list of int sequences, or [b, L] array with all rows
        full) through the target and drafter; returns the greedy next token per
        request and sets the decode state (kv_len = prompt length)."""
        if isinstance(prompts, np.ndarray) and prompts.ndim == 2:
            seqs = [list(r) for r in prompts]
        else:
            seqs = [list(p) for p in prompts]
        b, lmax = len(seqs), max(len(p) for p in seqs)
        tok = np.zeros((b, lmax), np.int32)
        for r, p in enumerate(seqs):
            tok[r, :len(p)] = p
        ln = np.array([len(p) for p in seqs], np.int32)
        nxt = np.zeros(b, np.int32)
        L.check(L.load().smo_engine_prefill(self._h, tok.ctypes.data_as(C.c_void_p), ln.ctypes.data_as(C.c_void_p), b,
                                            lmax, nxt.ctypes.data_as(C.c_void_p), C.c_void_p(stream or 0)))
        return nxt

    def decode_begin(self, root, kv_len) -> None:
        r = np.ascontiguousarray(root, np.int32)
        k = np.ascontiguousarray(kv_len, np.int32)
        L.check(L.load().smo_engine_decode_begin(self._h, r.ctypes.data_as(C.c_void_p), k.ctypes.data_as(C.c_void_p),
                                                 r.size))

    def decode_step(self, k: int, drafts=None, stream: Optional[int] = None) -> None:
        """One draft -> verify -> accept -> commit iteration (asynchronous).
        drafts: None (drafter proposes) or [b, k] planted drafts."""
        d = None if drafts is None else np.ascontiguousarray(drafts, np.int32)
        L.check(L.load().smo_engine_decode_step(self._h, k, None if d is None else d.ctypes.data_as(C.c_void_p),
                                                C.c_void_p(stream or 0)))

    def decode_step_tree(self, tokens, parents, stream: Optional[int] = None) -> None:
        """One iteration with a planted draft tree: tokens [b, n-1] for nodes
        1..n-1, parents [b, n] (parents[:, 0] = -1, parents[:, i] < i)."""
        t = np.ascontiguousarray(tokens, np.int32)
        p = np.ascontiguousarray(parents, np.int32)
        L.check(L.load().smo_engine_decode_step_tree(self._h, p.shape[1], t.ctypes.data_as(C.c_void_p),
                                                     p.ctypes.data_as(C.c_void_p), C.c_void_p(stream or 0)))

    def decode_run(self, k: int, steps: int, graph: bool = False, stream: Optional[int] = None) -> None:
        """`steps` drafter-driven iterations (asynchronous); graph=True replays
        one captured CUDA graph per iteration (needs a non-default stream)."""
        L.check(L.load().smo_engine_decode_run(self._h, k, steps, int(graph), C.c_void_p(stream or 0)))

    def set_draft_split(self, gpu_requests: int) -> None:
        """Drafter GPU part = requests [0, gpu_requests), CPU part (host K/V,
        host-pool attention) = the rest; -1: all on the GPU (draft_cpu_kv)."""
        L.check(L.load().smo_engine_set_draft_split(self._h, int(gpu_requests)))

    def draft_split_times(self, max_steps: int = 64) -> np.ndarray:
        """[steps, 3] (GPU part, host attention, GPU after the join) seconds of
        the last decode step's drafter steps; empty if it ran without a split."""
        out = np.zeros(3 * max_steps, np.float64)
        n = C.c_int32(0)
        L.check(L.load().smo_engine_draft_split_times(self._h, out.ctypes.data_as(C.c_void_p), out.size, C.byref(n)))
        return out[:3 * n.value].reshape(n.value, 3)

    def decode_read(self, b: int, cap: int):
        """(committed [b, cap] -1 padded, n_committed [b], kv_len [b], root [b])"""
        com = np.zeros((b, cap), np.int32)
        n = np.zeros(b, np.int32)
        kv = np.zeros(b, np.int32)
        root = np.zeros(b, np.int32)
        vp = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        L.check(L.load().smo_engine_decode_read(self._h, vp(com), cap, vp(n), vp(kv), vp(root)))
        return com, n, kv, root

    def last_times(self) -> dict:
        t = L.StageTimes()
        L.check(L.load().smo_engine_last_times(self._h, C.byref(t)))
        return {k: getattr(t, k) for k, _ in L.StageTimes._fields_}

    def debug_tensor(self, name: str, layer: int, shape, dtype) -> np.ndarray:
        out = np.zeros(shape, dtype)
        L.check(L.load().smo_engine_debug_tensor(self._h, name.encode(), layer, out.ctypes.data_as(C.c_void_p),
                                                 out.nbytes))
        return out

    def tensor_ptr(self, name: str, layer: int = -1, expert: int = 0):
        p, nb = C.c_void_p(), C.c_size_t()
        L.check(L.load().smo_engine_tensor_ptr(self._h, name.encode(), layer, expert, C.byref(p), C.byref(nb)))
        return p.value, nb.value


def geometric_alpha(p: float, k: int) -> float:
    """alpha(k) = sum_{i<=k} p^i (config.hpp:77-89)."""
    return sum(p ** i for i in range(k + 1)) if p != 1.0 else float(k + 1)


def step_roofline(shape: ModelShape, b: int, n: int, prefix: int, h2d_gbs: float, hbm_gbs: float,
                  tflops: float, cached_blocks: int = 0, ep: int = 1, h2d_bytes: Optional[float] = None,
                  extra_hbm_bytes: float = 0.0) -> dict:
    """Binding roofline of one verify step: the slower of
    host-link bytes, HBM bytes and tensor peak (roofline.hpp:108-151), per
    GPU. `b` is the global batch; with expert parallelism over `ep` GPUs each
    streams and reads E/ep experts per layer and attends b/ep requests.
    h2d_bytes=None: the algorithmic H2D bytes of SURVEY.md §8(d) (bf16
    expert blocks, roofline.hpp:61-62); else the bytes actually streamed.
    extra_hbm_bytes: HBM traffic beyond the algorithmic bytes that the
    implementation chose to spend (the link codec's code read + bf16 write)."""
    s = shape
    T = b * n
    e_bytes = s.expert_bytes
    activated = s.n_expert  # large batch: every expert activates
    h2d = (s.n_layers * activated - cached_blocks) * e_bytes / ep
    if h2d_bytes is not None:  # the bytes actually streamed (BATCH_ONE selection, coded experts)
        h2d = h2d_bytes
    kv = 2 * (b / ep) * (prefix + n) * s.n_kv_heads * s.head_dim * 2
    dense = (s.hidden * (s.n_q_heads + 2 * s.n_kv_heads) * s.head_dim + s.n_q_heads * s.head_dim * s.hidden) * 2
    hbm = s.n_layers * (activated / ep * e_bytes + kv + dense) + s.vocab * s.hidden * 2 + extra_hbm_bytes
    flops = (s.n_layers * (2 * 3 * s.hidden * s.inter * T * s.top_k / ep + 2 * (T / ep) * dense / 2
                           + 4 * (b / ep) * n * (prefix + n) * s.n_q_heads * s.head_dim)
             + 2 * (T / ep) * s.hidden * s.vocab)
    t = {"h2d": h2d / (h2d_gbs * 1e9), "hbm": hbm / (hbm_gbs * 1e9), "tensor": flops / (tflops * 1e12)}
    bound = max(t, key=t.get)
    return {"bound": bound, "t_roof_s": t[bound], "h2d_bytes": h2d, "hbm_bytes": hbm, "flops": flops,
            "times": t, "fits": math.isfinite(t[bound])}
