"""ctypes bindings for the CPU checker libraries.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py. The product package
(paper_2508_21706_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmoeplan_ref.so")

_P = np.ctypeslib.ndpointer
_d = C.c_double
_sz = C.c_size_t


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (+ _ref when /root/reference is present)."""
    subprocess.run(["make", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_trial_uniform.restype = C.c_double
        L.orc_trial_uniform.argtypes = [C.POINTER(C.c_uint64)]
        L.orc_chunked_attention.restype = C.c_int
        L.orc_chunked_attention.argtypes = [_sz, _sz, _sz, C.c_void_p, C.c_void_p, C.c_void_p, _sz, C.c_void_p, C.c_void_p]
        L.orc_naive_attention.restype = C.c_int
        L.orc_naive_attention.argtypes = [_sz, _sz, _sz, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_simulate_tokens.restype = C.c_int
        L.orc_simulate_tokens.argtypes = [C.c_void_p, _sz, C.c_int, C.c_int64, C.c_uint64, C.POINTER(_d), C.POINTER(_d)]
        L.orc_random_cases.restype = None
        L.orc_random_cases.argtypes = [C.c_uint64, C.c_uint64] + [C.c_void_p] * 5 + [C.POINTER(_sz)] * 3
        L.orc_fill_uniform_bf16.restype = None
        L.orc_fill_uniform_bf16.argtypes = [C.c_void_p, _sz, C.c_uint64, C.c_uint64, C.c_uint64, C.c_float]
        L.orc_fill_normal_bf16.restype = None
        L.orc_fill_normal_bf16.argtypes = [C.c_void_p, _sz, C.c_uint64, C.c_uint64, C.c_uint64, C.c_float]
        L.orc_rmsnorm.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_float, C.c_void_p]
        L.orc_gemm_xwt.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.orc_router_logits.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.orc_topk_softmax.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_permute.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_expert_swiglu.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_rope.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_float]
        L.orc_verify_attention.restype = C.c_int
        L.orc_verify_attention.argtypes = [C.c_void_p] * 5 + [C.c_int] * 6 + [C.c_void_p]
        L.orc_argmax_rows.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_greedy_accept.argtypes = [C.c_void_p] * 3 + [C.c_int, C.c_int] + [C.c_void_p] * 3
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The unmodified reference headers behind ref_shim.cpp (oracle/_ref)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_splitmix64.restype = C.c_uint64
        L.ref_splitmix64.argtypes = [C.c_uint64]
        L.ref_trial_stream.argtypes = [C.c_uint64, _sz, C.c_void_p]
        L.ref_mask_memory_savings.restype = C.c_double
        L.ref_mask_memory_savings.argtypes = [_sz, _sz]
        L.ref_chunked_attention.restype = C.c_int
        L.ref_chunked_attention.argtypes = [_sz, _sz, _sz, C.c_void_p, C.c_void_p, C.c_void_p, _sz, C.c_void_p, C.c_void_p]
        L.ref_naive_oracle.restype = C.c_int
        L.ref_naive_oracle.argtypes = [_sz, _sz, _sz, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_simulate_tokens.restype = C.c_int
        L.ref_simulate_tokens.argtypes = [C.c_void_p, _sz, C.c_int, C.c_int64, C.c_uint64, C.POINTER(_d), C.POINTER(_d)]
        L.ref_verify_layer_attention.restype = C.c_double
        L.ref_verify_layer_attention.argtypes = [C.c_void_p] * 5 + [C.c_int] * 7 + [C.c_void_p]
        _ref = L
    return _ref


# ---------------------------------------------------------------------------
# Thin numpy-level helpers

ERRORS = {1: "attention: shape mismatch", 2: "attention: non-finite Q",
          3: "attention: non-finite K", 4: "attention: non-finite V",
          5: "attention: mask size mismatch", 6: "attention: fully blocked query row"}


def chunked_attention(Q, K, V, mask):
    Q = np.ascontiguousarray(Q, np.float64)
    K = np.ascontiguousarray(K, np.float64)
    V = np.ascontiguousarray(V, np.float64)
    mask = np.ascontiguousarray(mask, np.uint8)
    n, d = Q.shape
    p = K.shape[0] - n
    out = np.zeros((n, d), np.float64)
    rc = lib().orc_chunked_attention(n, p, d, _ptr(Q), _ptr(K), _ptr(V), mask.shape[0], _ptr(mask), _ptr(out))
    if rc:
        raise ValueError(ERRORS[rc])
    return out


def naive_attention(Q, K, V, full):
    Q = np.ascontiguousarray(Q, np.float64)
    K = np.ascontiguousarray(K, np.float64)
    V = np.ascontiguousarray(V, np.float64)
    full = np.ascontiguousarray(full, np.uint8)
    n, d = Q.shape
    p = K.shape[0] - n
    out = np.zeros((n, d), np.float64)
    rc = lib().orc_naive_attention(n, p, d, _ptr(Q), _ptr(K), _ptr(V), _ptr(full), _ptr(out))
    if rc:
        raise ValueError(ERRORS[rc])
    return out


def random_cases(seed: int, count: int):
    """The `moeplan verify-attention --random seed count` instances."""
    L = lib()
    ql, kl, ml = _sz(), _sz(), _sz()
    L.orc_random_cases(seed, count, None, None, None, None, None, C.byref(ql), C.byref(kl), C.byref(ml))
    dims = np.zeros((count, 3), np.int64)
    q = np.zeros(ql.value); k = np.zeros(kl.value); v = np.zeros(kl.value)
    m = np.zeros(ml.value, np.uint8)
    L.orc_random_cases(seed, count, _ptr(dims), _ptr(q), _ptr(k), _ptr(v), _ptr(m), C.byref(ql), C.byref(kl), C.byref(ml))
    cases = []
    qo = ko = mo = 0
    for n, p, d in dims.tolist():
        t = p + n
        cases.append(dict(n=n, p=p, d=d,
                          Q=q[qo:qo + n * d].reshape(n, d),
                          K=k[ko:ko + t * d].reshape(t, d),
                          V=v[ko:ko + t * d].reshape(t, d),
                          mask=m[mo:mo + n * n].reshape(n, n)))
        qo += n * d; ko += t * d; mo += n * n
    return cases


def simulate_tokens(probs, k, trials, seed):
    probs = np.ascontiguousarray(probs, np.float64)
    mean, sd = _d(), _d()
    rc = lib().orc_simulate_tokens(_ptr(probs), probs.size, k, trials, seed, C.byref(mean), C.byref(sd))
    if rc:
        raise ValueError("simulate_tokens: " + ("trials >= 1" if rc == 1 else "probabilities length >= k"))
    return mean.value, sd.value


def bf16_to_f32(a):
    return (np.asarray(a, np.uint16).astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(a):
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    r[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)
    return r


def fill_uniform_bf16(count, seed, tensor_id, scale, base=0):
    out = np.empty(count, np.uint16)
    lib().orc_fill_uniform_bf16(_ptr(out), count, seed, tensor_id, base, scale)
    return out


def fill_normal_bf16(count, seed, tensor_id, scale, base=0):
    out = np.empty(count, np.uint16)
    lib().orc_fill_normal_bf16(_ptr(out), count, seed, tensor_id, base, scale)
    return out
