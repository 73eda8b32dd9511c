"""Python mirror of the reference's attention API (attention.hpp:16-205).

Same names, argument meaning and error behaviour as `moeplan::`:
`Matrix`, `AttentionInstance`, `CompactMask` (+`chain`), `expand`, `compact`,
`mask_memory_savings`, `chunked_attention`, `naive_oracle`. Errors raise
ValueError (the reference's std::invalid_argument) with the reference's
messages. `chunked_attention` runs the fp64 operator on the GPU through
smo_chunked_attention_f64; the batched bf16 production path is
ops.verify_attention (K1). `naive_oracle` is the reference's own brute-force
cross-check (attention.hpp:158-203) and stays a small numpy routine, exactly
as the reference keeps it beside the operator.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


class Matrix:
    """Row-major dense fp64 matrix (attention.hpp:19-28)."""

    def __init__(self, rows: int = 0, cols: int = 0, data=None):
        self.rows, self.cols = int(rows), int(cols)
        self.data = np.zeros((self.rows, self.cols)) if data is None else np.array(data, dtype=np.float64).reshape(
            self.rows, self.cols)

    def at(self, r, c):
        return self.data[r, c]

    def set(self, r, c, v):
        self.data[r, c] = v


@dataclass
class AttentionInstance:
    """n draft queries over prefix_len previous tokens (attention.hpp:31-38)."""
    n: int = 0
    prefix_len: int = 0
    d: int = 0
    Q: Matrix = field(default_factory=Matrix)
    K: Matrix = field(default_factory=Matrix)
    V: Matrix = field(default_factory=Matrix)


class CompactMask:
    """n x n draft-draft visibility; prefix implicit (attention.hpp:41-58)."""

    def __init__(self, n: int = 0, visible=None):
        self.n = int(n)
        self.visible = np.zeros((self.n, self.n), dtype=bool) if visible is None else np.array(
            visible, dtype=bool).reshape(self.n, self.n)

    def at(self, i, j) -> bool:
        return bool(self.visible[i, j])

    def set(self, i, j, v: bool):
        self.visible[i, j] = bool(v)

    @staticmethod
    def chain(n: int) -> "CompactMask":
        return CompactMask(n, np.tril(np.ones((n, n), dtype=bool)))

    def bits(self) -> np.ndarray:
        """Row bitmasks as used by K1 (bit j = draft j visible)."""
        if self.n > 64:
            raise ValueError("attention: mask size mismatch")
        w = (np.uint64(1) << np.arange(self.n, dtype=np.uint64))
        return (self.visible.astype(np.uint64) * w).sum(axis=1).astype(np.uint64)


def expand(mask: CompactMask, prefix_len: int) -> np.ndarray:
    """Full n x (prefix_len+n) mask (attention.hpp:61-71)."""
    n = mask.n
    full = np.zeros((n, prefix_len + n), dtype=bool)
    full[:, :prefix_len] = True
    full[:, prefix_len:] = mask.visible
    return full


def compact(full, n: int, prefix_len: int) -> CompactMask:
    full = np.asarray(full, dtype=bool).reshape(n, prefix_len + n)
    return CompactMask(n, full[:, prefix_len:])


def mask_memory_savings(n: int, prefix_len: int) -> float:
    if n < 1:
        raise ValueError("mask_memory_savings: n >= 1")
    return float(prefix_len + n) / float(n)


def _check_shapes(inst: AttentionInstance):
    total = inst.prefix_len + inst.n
    if ((inst.Q.rows, inst.Q.cols) != (inst.n, inst.d) or (inst.K.rows, inst.K.cols) != (total, inst.d)
            or (inst.V.rows, inst.V.cols) != (total, inst.d)):
        raise ValueError("attention: shape mismatch")


def chunked_attention(inst: AttentionInstance, mask: CompactMask) -> Matrix:
    """moeplan::chunked_attention (attention.hpp:117-156), fp64, on the GPU."""
    _check_shapes(inst)
    n, p, d = inst.n, inst.prefix_len, inst.d
    Q = np.ascontiguousarray(inst.Q.data, np.float64)
    K = np.ascontiguousarray(inst.K.data, np.float64)
    V = np.ascontiguousarray(inst.V.data, np.float64)
    m = np.ascontiguousarray(mask.visible, np.uint8)
    out = np.zeros((n, d), np.float64)
    vp = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    L.check(L.load().smo_chunked_attention_f64(n, p, d, vp(Q), vp(K), vp(V), mask.n, vp(m), vp(out)))
    return Matrix(n, d, out)


def naive_oracle(inst: AttentionInstance, full_mask) -> Matrix:
    """The reference's brute-force cross-check (attention.hpp:161-203)."""
    _check_shapes(inst)
    for nm, M in (("Q", inst.Q), ("K", inst.K), ("V", inst.V)):
        if not np.all(np.isfinite(M.data)):
            raise ValueError(f"attention: non-finite {nm}")
    n, total = inst.n, inst.prefix_len + inst.n
    full = np.asarray(full_mask, dtype=bool).ravel()
    if full.size != n * total:
        raise ValueError("attention: full mask size mismatch")
    full = full.reshape(n, total)
    scale = 1.0 / np.sqrt(float(inst.d))
    out = np.zeros((n, inst.d))
    for i in range(n):
        s = np.array([float(np.dot(inst.Q.data[i], inst.K.data[j])) * scale for j in range(total)])
        s = np.where(full[i], s, -np.inf)
        mx = s.max() if total else -np.inf
        if mx == -np.inf:
            raise ValueError("attention: fully blocked query row")
        e = np.where(s == -np.inf, 0.0, np.exp(s - mx))
        den = e.sum()
        for j in range(total):
            w = e[j] / den
            if w != 0.0:
                out[i] += w * inst.V.data[j]
    return Matrix(n, inst.d, out)
