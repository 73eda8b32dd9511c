"""CPU tier: the K5 unary link format restated in numpy (tests/codec_ref.py)
— lossless round trips on the data kinds the engine meets, and known-answer
layouts that pin the byte format the GPU encoder must produce
(tests/test_gpu_kernels.py::test_expert_codec_unary_matches_numpy_encoder)."""
import numpy as np
import pytest

import codec_ref


def _bf16(f32: np.ndarray) -> np.ndarray:
    u = f32.astype(np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)  # round to nearest even


def _data(kind: str, n: int) -> np.ndarray:
    rng = np.random.default_rng(17)
    if kind == "uniform":  # the engine's expert init: U(-a, a), a = sqrt(3 / 4096)
        return _bf16((rng.random(n) * 2 - 1) * np.sqrt(3.0 / 4096))
    if kind == "normal":  # trained-weight-like, exact zeros and outliers
        x = rng.normal(0, 0.02, n)
        x[::997] = 0
        x[::4099] *= 64
        return _bf16(x)
    return rng.integers(0, 1 << 16, n).astype(np.uint16)  # every exponent: escapes, tiny bases


@pytest.mark.parametrize("kind", ["uniform", "normal", "wide"])
def test_unary_round_trip(kind):
    x = _data(kind, 1024 * 24)
    code = codec_ref.encode(x)
    assert codec_ref.total_bytes(code, x.size) == len(code)
    assert np.array_equal(codec_ref.decode(code, x.size), x)
    bpw = 8 * len(code) / x.size
    if kind == "uniform":
        assert 9.9 < bpw < 10.6, bpw  # the exponent entropy (~2 bits) + 8 bits of sign/mantissa
    if kind == "normal":
        assert bpw < 12.0, bpw  # below the 4-bit window code


def test_unary_known_answers():
    # one segment, every value 1.0 (exponent 127): j = 0 everywhere -> 1024
    # zero bits = 32 zero words, no escapes; table (16 B) + 1024 + 128 bytes
    x = np.full(1024, 0x3F80, np.uint16)
    code = codec_ref.encode(x)
    t = np.frombuffer(code[:16], np.uint8)
    assert int(t[:4].view("<u4")[0]) == 16 and t[4] == 127 and t[5] == 0 and int(t[6:8].view("<u2")[0]) == 32
    assert int(t[8:12].view("<u4")[0]) == 16 + 1024 + 128 == len(code)
    assert code[16:16 + 1024] == b"\0" * 1024 and code[16 + 1024:] == b"\0" * 128
    # halve every second value (exponent 126): j alternates 0, 1 -> codes "0", "10"
    y = x.copy()
    y[1::2] = 0x3F00
    c2 = codec_ref.encode(y)
    bits = np.unpackbits(np.frombuffer(c2[16 + 1024:], np.uint8)[:4][::-1])  # word 0, MSB first
    assert list(bits[:9]) == [0, 1, 0, 0, 1, 0, 0, 1, 0]
    assert np.array_equal(codec_ref.decode(c2, 1024), y)
    # an outlier 2^6 above the rest escapes (24 bits) instead of lengthening all codes
    z = x.copy()
    z[5] = 0x4280  # 64.0, exponent 133
    c3 = codec_ref.encode(z)
    t3 = np.frombuffer(c3[:8], np.uint8)
    assert t3[4] == 127 and t3[5] == 1
    assert np.array_equal(codec_ref.decode(c3, 1024), z)
