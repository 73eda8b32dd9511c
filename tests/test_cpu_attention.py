"""CPU tier: the host verification attention of the CPU placement
(smo_cpu_verify_attention — pure host code inside
libspecmoe.so, no GPU needed) against the oracle's restatement of
moeplan::chunked_attention (attention.hpp:117-156) on the same bf16 inputs.
Tolerance as K1: max-abs <= 2^-7 max|V|, rel-RMS <= 5e-3."""
import numpy as np
import pytest


def _case(oracle, b, n, nq, nkv, d, prefix, tree, seed):
    s_max = max(prefix) + n + 16
    rng = np.random.default_rng(seed)
    f = lambda *sh: oracle.f32_to_bf16(rng.uniform(-1, 1, size=sh).astype(np.float32))  # noqa: E731
    q, kc, vc = f(b * n, nq, d), f(b, nkv, s_max, d), f(b, nkv, s_max, d)
    bits = np.zeros(b * n, np.uint64)
    for r in range(b):
        par = [-1] + [int(rng.integers(0, i)) for i in range(1, n)] if tree else None
        for i in range(n):
            m, cur = 0, i
            if tree:
                while cur >= 0:
                    m |= 1 << cur
                    cur = -1 if cur == 0 else par[cur]
            else:
                m = (1 << (i + 1)) - 1
            bits[r * n + i] = m
    return q, kc, vc, bits, np.array(prefix, np.int32), s_max


@pytest.mark.parametrize("b,n,nq,nkv,d,prefix,tree", [
    (4, 5, 8, 2, 64, [1024, 1000, 3, 0], False),
    (2, 9, 32, 8, 128, [700, 131], True),
    (3, 1, 16, 16, 128, [127, 128, 129], False),
    (2, 32, 8, 2, 64, [0, 64], False),
])
def test_cpu_attention_vs_oracle(oracle, b, n, nq, nkv, d, prefix, tree):
    from paper_2508_21706_b200 import ops
    q, kc, vc, bits, pre, s_max = _case(oracle, b, n, nq, nkv, d, prefix, tree, seed=b + n)
    got = oracle.bf16_to_f32(ops.cpu_verify_attention(q, kc, vc, bits, pre, threads=4))
    ref = np.zeros((b * n, nq, d), np.uint16)
    rc = oracle.lib().orc_verify_attention(oracle._ptr(q), oracle._ptr(kc), oracle._ptr(vc), oracle._ptr(bits),
                                           oracle._ptr(pre), b, n, nq, nkv, d, s_max, oracle._ptr(ref))
    assert rc == 0
    exp = oracle.bf16_to_f32(ref)
    assert np.max(np.abs(got - exp)) <= 2 ** -7
    rel = np.sqrt(np.mean((got - exp) ** 2) / np.mean(exp ** 2))
    assert rel <= 5e-3, rel


def test_cpu_attention_errors():
    from paper_2508_21706_b200 import ops
    q = np.zeros((2, 4, 64), np.uint16)
    kc = np.zeros((1, 2, 8, 64), np.uint16)
    with pytest.raises(ValueError, match="shape mismatch"):
        ops.cpu_verify_attention(q, kc, kc, np.ones(2, np.uint64), np.array([7], np.int32))
