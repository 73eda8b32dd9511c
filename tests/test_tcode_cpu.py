"""CPU tier: the K5 tile code T2 restated in numpy (tests/tcode_ref.py) —
lossless round trips on the data kinds the engine meets, known-answer
layouts that pin the byte format the GPU encoder must produce
(tests/test_gpu_tcode.py), and the code sizes the link relies on."""
import numpy as np
import pytest

import tcode_ref as T
import oracle_py as O


def _mats(kind: str, h: int, hi: int):
    n = h * hi
    if kind == "uniform":  # the engine's expert init (engine.cu, fill_uniform)
        f = [O.fill_uniform_bf16(n, 7, 1101 + i, np.sqrt(3.0 / (h if i < 2 else hi))) for i in range(3)]
    elif kind == "gaussian":  # SMO_INIT_GAUSSIAN (fill_normal: Irwin-Hall + 1/1024 outliers x8)
        f = [O.fill_normal_bf16(n, 7, 1101 + i, np.sqrt(3.0 / (h if i < 2 else hi))) for i in range(3)]
    else:  # every bit pattern: escapes, literals, raw segments, tiny bases
        rng = np.random.default_rng(5)
        f = [rng.integers(0, 1 << 16, n).astype(np.uint16) for _ in range(3)]
        f[0][::7] = 0  # exact zeros (exponent 0: literals)
    return np.concatenate(f)


@pytest.mark.parametrize("kind", ["uniform", "gaussian", "wide"])
def test_tcode_round_trip(kind):
    h, hi = 256, 128
    x = _mats(kind, h, hi)
    code = T.encode_expert(x, h, hi)
    assert len(code) <= T.max_bytes(h, hi)
    assert np.array_equal(T.decode_expert(code, h, hi), x)
    bpw = 8 * len(code) / x.size
    if kind == "uniform":
        assert 10.2 < bpw < 10.7, bpw  # 8 + ~2.35 exponent bits + headers
    if kind == "gaussian":
        assert bpw < 11.1, bpw  # below the unary code on these weights (~11.45)


def _segment_tile(seg0: np.ndarray) -> np.ndarray:
    """A 128 x 64 matrix whose tile (0, 0) has segment 0 = seg0 and 1.0 elsewhere."""
    W = np.full((128, 64), 0x3F80, np.uint16)
    W[:16] = seg0.reshape(16, 64)
    return W


def test_tcode_known_answers():
    # every value 1.0 (exponent 127): E = 127, j = 0 -> all L1 codes 0, no
    # streams: header 32 + lo 8 x 1024 + L1 8 x 256 = 10272 bytes
    W = np.full((128, 64), 0x3F80, np.uint16)
    code = T.encode([W])
    toff = np.frombuffer(code[:16], "<u4")
    assert toff[0] == 16 and toff[1] == len(code) == 16 + 10272
    hdr = np.frombuffer(code[16:48], "<u4")
    assert np.all(hdr == (127 | ((10272 // 4) << 12)))
    assert not np.any(np.frombuffer(code[48:], np.uint8))  # lo = 0 (positive, zero mantissa), codes 0
    # segment 0: value 3 halved (j = 1) and value 17 at 2^-3 (j = 3: L1 code 3, level-2 code 0)
    s = np.full(1024, 0x3F80, np.uint16)
    s[3] = 0x3F00
    s[17] = 0x3E00
    code = T.encode([_segment_tile(s)])
    hdr = np.frombuffer(code[16:48], "<u4")
    assert hdr[0] == 127 | (2 << 8) | (2568 << 12) and hdr[1] == 127 | (2569 << 12)
    l1 = np.frombuffer(code[16 + 32 + 8192:16 + 32 + 8192 + 256], "<u4")
    # lane 0 word 0: value 3 = 2 q + 1 with q = 1 -> bits 16 + 2; word 1: value 17 = 16 + 2*0 + 1 -> bits 16
    assert l1[0] == 1 << 18 and l1[1] == 3 << 16 and not np.any(l1[2:])
    assert np.frombuffer(code[16 + 10272:16 + 10276], "<u4")[0] == 0  # level-2 code 0
    assert len(code) == 16 + 10288  # one stream word, padded to 16 B
    assert np.array_equal(T.decode(code, [(128, 64)])[0], _segment_tile(s))
    # an exact zero (exponent 0, j = 127): 3, 3, nibble 15 and a literal byte 0
    z = np.full(1024, 0x3F80, np.uint16)
    z[0] = 0
    code = T.encode([_segment_tile(z)])
    assert (int(np.frombuffer(code[16:20], "<u4")[0]) >> 8) & 0xF == 2 | 4 | 8
    st = np.frombuffer(code[16 + 10272:16 + 10284], "<u4")
    assert st.tolist() == [3, 15, 0]  # L2 word, L3 word, literal 0 padded to 4 bytes
    assert np.array_equal(T.decode(code, [(128, 64)])[0], _segment_tile(z))
    # incompressible tile -> raw: header word 0 = flags 1, the tile verbatim
    r = np.random.default_rng(1).integers(0, 1 << 16, (128, 64)).astype(np.uint16)
    code = T.encode([r])
    assert np.frombuffer(code[16:48], "<u4").tolist() == [1 << 8] + [0] * 7
    assert len(code) == 16 + 32 + 16384 and np.frombuffer(code[48:], "<u2").tolist() == r.ravel().tolist()
    assert np.array_equal(T.decode(code, [(128, 64)])[0], r)


def test_tcode_base_choice_prefers_fewer_bits():
    # one outlier 2^6 above the rest: E drops to the highest base that keeps
    # the bulk within level 1 (j = 2; ties prefer the higher E) and the
    # outlier becomes a 16-bit literal, instead of adding 6 to every j
    s = np.full(1024, 0x3F80, np.uint16)
    s[5] = 0x4280  # 64.0
    E, bits = T.choose_base(((s.astype(np.int64) >> 7) & 0xFF))
    assert E == 129 and bits == 2 * 1023 + 16


# ---------------------------------------------------------------- T3
import tcode3_ref as T3  # noqa: E402


@pytest.mark.parametrize("kind", ["uniform", "gaussian", "wide"])
def test_tcode3_round_trip(kind):
    h, hi = 256, 128
    x = _mats(kind, h, hi)
    code = T3.encode_expert(x, h, hi)
    assert len(code) <= T.max_bytes(h, hi)
    assert np.array_equal(T3.decode_expert(code, h, hi), x)
    bpw = 8 * len(code) / x.size
    if kind == "uniform":
        assert 11.0 < bpw < 11.4, bpw  # 8 + 3 + escapes (~1/128 x 24 bits) + headers


def test_tcode3_known_answers():
    # every value 1.0: E = 127, codes 0, no escapes: 32 + 8192 + 3072 = 11296 bytes
    W = np.full((128, 64), 0x3F80, np.uint16)
    code = T3.encode([W])
    assert np.frombuffer(code[:16], "<u4")[1] == len(code) == 16 + 11296
    assert np.all(np.frombuffer(code[16:48], "<u4") == (127 | ((11296 // 4) << 20)))
    # segment 0: value 3 halved (j = 1), value 30 at 2^-6 (j = 6, pair 15 even),
    # value 33 at 2^-7 (j = 7: escape, lane 1 pair 0 odd)
    s = np.full(1024, 0x3F80, np.uint16)
    s[3], s[30], s[33] = 0x3F00, 0x3C80, 0x3C00
    code = T3.encode([_segment_tile(s)])
    hdr = np.frombuffer(code[16:48], "<u4")
    assert hdr[0] == 127 | (1 << 9) | ((11296 // 4) << 20) and hdr[1] == 127 | ((11300 // 4) << 20)
    c3 = np.frombuffer(code[16 + 8224:16 + 8224 + 384], "<u4")
    # lane 0: pair 1 (values 2, 3) odd code 1 at bits 16 + 3; pair 15 even code 6 = 0b110: bits 15 of words 1, 2
    assert c3[0] == 1 << 19 and c3[1] == 1 << 15 and c3[2] == 1 << 15
    assert c3[3] == 7 << 16  # lane 1, pair 0 odd: the escape code
    assert np.frombuffer(code[16 + 11296:16 + 11298], "<u2")[0] == 33 and code[16 + 11298] == 120
    assert np.array_equal(T3.decode(code, [(128, 64)])[0], _segment_tile(s))
    # an exact zero: the segment maximum stays the base, the zero escapes
    z = np.full(1024, 0x3F80, np.uint16)
    z[0] = 0
    code = T3.encode([_segment_tile(z)])
    assert (int(np.frombuffer(code[16:20], "<u4")[0]) >> 9) & 0x7FF == 1
    assert np.array_equal(T3.decode(code, [(128, 64)])[0], _segment_tile(z))
    # a segment whose maximum exponent is below 7 (near-zero values) -> raw tile
    t = np.full(1024, 0x0080, np.uint16)  # exponent 1
    code = T3.encode([_segment_tile(t)])
    assert np.frombuffer(code[16:48], "<u4").tolist() == [1 << 8] + [0] * 7
    assert np.array_equal(T3.decode(code, [(128, 64)])[0], _segment_tile(t))
