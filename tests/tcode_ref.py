"""Test infrastructure: the K5 tile code ("T2", paper_2508_21706_b200/csrc/
tcode.cuh header) restated in numpy — encoder and decoder — so the byte layout
is pinned on the CPU tier and the GPU encoder is checked byte for byte.

The code is shaped for the expert kernel, which decodes it straight into
its shared-memory weight tiles (moe_tc.cu, moe_coded_kernel):

  block  = the matrices of one expert ([W1 | W3 | W2]: (h_i, h), (h_i, h),
           (h, h_i) row-major bf16), cut into tiles of 128 rows x 64 columns
           in (matrix, row tile, column tile) order — one tile is one
           k-block of the expert kernel's A operand.
           u32 toff[nt + 1] (byte offset of tile t from the block start,
           toff[nt] = total bytes), zero-padded to 16 B; then the tiles,
           each 16-B aligned.
  tile   = 8 segments of 16 rows x 64 columns (segment s = rows 16 s ..).
           u32 hdr[8]: E | flags << 8 | soff4 << 12 (flags: 1 the whole tile
           is raw, 2 some value of the segment leaves level 1, 4 some value
           reaches the nibble level, 8 literals; soff4 = the segment's
           stream offset from the tile start in 4-byte units), then
             lo[8][1024]  sign << 7 | mantissa of value v of segment s
             L1[8][256]   2-bit level-1 codes; the 32 values 32 L + i of
                          "lane" L of a segment sit in two u32 words at 8 L:
                          word w holds value 16 w + 2 q at bits [2 q, 2 q + 2)
                          and value 16 w + 2 q + 1 at bits [16 + 2 q, ..)
                          (q = 0..7) — two values per 16-bit half, so the
                          decoder forms bf16 pairs with one shift and mask
             streams      per segment, 4-byte aligned:
                          L2   u32 words of 2-bit fields, LSB first: the
                               level-2 codes of the values whose level-1 code
                               is 3 (value order)
                          L3   u32 words of 4-bit fields: the nibbles of the
                               values whose level-2 code is 3 (value order)
                          lit  exponent bytes of the values whose nibble is
                               15, zero-padded to 4 bytes
           zero padding to 16 B. A raw tile (flags 1 in hdr[0]; every other
           header word 0) is the header + its 128 x 64 bf16 values row-major.
  segment value order v = 64 r + c (row r, column c of the segment).
  Exponent e of a value, segment base E, j = E - e: j <= 2 is its level-1
  code; 3 <= j <= 5 codes 3, then j - 3; 6 <= j <= 20 codes 3, 3, then the
  nibble j - 6; any other value (e > E or j > 20) codes 3, 3, nibble 15 and
  its exponent byte as a literal (2, 4, 8, 16 bits). E = the segment maximum
  or up to 7 below it, never below 6, the fewest code bits wins (ties: the
  higher E; 6 when the maximum is below 6); a tile whose code would take
  more bytes than raw is stored raw.

For uniform-init weights (j geometric, p = 1/2) this is 2 + 2/8 + 4/64 ...
~2.35 bits per exponent (the unary code: 2.15); for gaussian-like weights
~2.7 (unary: 2.9). Lossless for every bf16 bit pattern."""
import numpy as np

TR, TC, SR = 128, 64, 16  # tile rows, tile columns, segment rows
SEG = SR * TC
RAW_BYTES = 2 * SEG


def _pad16(n: int) -> int:
    return (n + 15) & ~15


def _cost(j: np.ndarray) -> np.ndarray:
    """Code bits of each exponent offset j (2, 4, 8 or 16 for literals)."""
    return np.where((j >= 0) & (j <= 2), 2, np.where((j >= 3) & (j <= 5), 4,
                                                      np.where((j >= 6) & (j <= 20), 8, 16)))


def choose_base(e: np.ndarray):
    """(E, code bits) of a segment's exponents e (int array)."""
    emax = int(e.max())
    best, base = None, max(emax, 6)
    for c in range(8):
        b0 = emax - c
        if b0 < 6:  # E >= 6: the decoder forms E - c1 - c2 (<= 6) without a borrow
            break
        cost = int(np.sum(_cost(b0 - e)))
        if best is None or cost < best:
            best, base = cost, b0
    if best is None:
        best = int(np.sum(_cost(base - e)))
    return base, best


def _pack(fields: np.ndarray, width: int) -> bytes:
    per = 32 // width
    nw = (fields.size + per - 1) // per
    f = np.zeros(nw * per, np.uint32)
    f[:fields.size] = fields
    if not nw:
        return b""
    w = np.bitwise_or.reduce(f.reshape(nw, per) << (width * np.arange(per, dtype=np.uint32)), axis=1)
    return w.astype("<u4").tobytes()


def _l1_words(c1: np.ndarray) -> np.ndarray:
    """32 lanes x 2 u32 words from 1024 level-1 codes (value order)."""
    c = c1.reshape(32, 2, 8, 2).astype(np.uint32)  # lane, word, q, half
    sh = (2 * np.arange(8, dtype=np.uint32))[None, None, :, None] + np.array([0, 16], np.uint32)[None, None, None, :]
    return np.bitwise_or.reduce((c << sh).reshape(32, 2, 16), axis=2).reshape(64)


def encode_segment(v: np.ndarray):
    """(E, flags, lo bytes, L1 bytes, stream bytes) of one segment, v = 1024 bf16 (uint16) in value order."""
    v = np.asarray(v, np.uint16).astype(np.int64)
    e = (v >> 7) & 0xFF
    E, _ = choose_base(e)
    j = E - e
    lit = (j < 0) | (j > 20)
    c1 = np.where((j >= 0) & (j <= 2), j, 3)
    s2 = c1 == 3
    c2 = np.where((j >= 3) & (j <= 5), j - 3, 3)[s2]
    s3 = s2 & ~((j >= 3) & (j <= 5))
    nib = np.where(lit, 15, j - 6)[s3]
    lits = e[lit].astype(np.uint8).tobytes()
    lits += b"\0" * ((-len(lits)) % 4)
    lo = (((v >> 8) & 0x80) | (v & 0x7F)).astype(np.uint8)
    stream = _pack(c2.astype(np.uint32), 2) + _pack(nib.astype(np.uint32), 4) + lits
    flags = (2 if s2.any() else 0) | (4 if s3.any() else 0) | (8 if lit.any() else 0)
    return E, flags, lo.tobytes(), _l1_words(c1).astype("<u4").tobytes(), stream


def tile_segments(W: np.ndarray, nb: int, kb: int):
    """The 8 segments (1024 values each, value order) of tile (nb, kb) of W."""
    t = W[nb * TR:(nb + 1) * TR, kb * TC:(kb + 1) * TC]
    return [t[s * SR:(s + 1) * SR].reshape(SEG) for s in range(TR // SR)]


def encode_tile(W: np.ndarray, nb: int, kb: int) -> bytes:
    segs = [encode_segment(seg) for seg in tile_segments(W, nb, kb)]
    off = 32 + 8 * SEG + 8 * 256
    hdr, streams = [], []
    for E, flags, _, _, st in segs:
        hdr.append(E | (flags << 8) | ((off // 4) << 12))
        streams.append(st)
        off += len(st)
    body = np.array(hdr, "<u4").tobytes() + b"".join(x[2] for x in segs) + b"".join(x[3] for x in segs) + \
        b"".join(streams)
    body += b"\0" * (_pad16(len(body)) - len(body))
    raw = 32 + 2 * TR * TC
    if len(body) >= raw:  # incompressible: the header (flags 1) + the tile verbatim
        t = W[nb * TR:(nb + 1) * TR, kb * TC:(kb + 1) * TC]
        return np.array([1 << 8] + [0] * 7, "<u4").tobytes() + t.astype("<u2").tobytes()
    return body


def encode(mats) -> bytes:
    """Block code of a list of row-major bf16 (uint16) matrices."""
    tiles = []
    for W in mats:
        R, C = W.shape
        assert R % TR == 0 and C % TC == 0
        for nb in range(R // TR):
            for kb in range(C // TC):
                tiles.append(encode_tile(W, nb, kb))
    nt = len(tiles)
    tb = _pad16(4 * (nt + 1))
    off = np.zeros(nt + 1, np.int64)
    off[0] = tb
    for t, b in enumerate(tiles):
        off[t + 1] = off[t] + len(b)
    head = off.astype("<u4").tobytes()
    return head + b"\0" * (tb - len(head)) + b"".join(tiles)


def encode_expert(block: np.ndarray, h: int, hi: int) -> bytes:
    """[W1 | W3 | W2] of one expert, flat bf16 (uint16)."""
    b = np.asarray(block, np.uint16)
    m = h * hi
    return encode([b[:m].reshape(hi, h), b[m:2 * m].reshape(hi, h), b[2 * m:3 * m].reshape(h, hi)])


def _unpack(b: np.ndarray, n: int, width: int) -> np.ndarray:
    per = 32 // width
    nw = (n + per - 1) // per
    w = b[:4 * nw].view("<u4").astype(np.int64)
    f = (w[:, None] >> (width * np.arange(per))[None, :]) & ((1 << width) - 1)
    return f.reshape(-1)[:n], 4 * nw


def decode_segment(hw: int, lo: np.ndarray, l1: np.ndarray, rest: np.ndarray) -> np.ndarray:
    """1024 values of a coded segment from its header word, lo / L1 bytes and
    the tile bytes from its stream offset on; returns (values, stream bytes used)."""
    E, flags = hw & 0xFF, (hw >> 8) & 0xF
    lo = lo.astype(np.uint32)
    w = l1.view("<u4").reshape(32, 2).astype(np.int64)
    sh = (2 * np.arange(8))[None, None, :, None] + np.array([0, 16])[None, None, None, :]
    c1 = ((w[:, :, None, None] >> sh) & 3).reshape(SEG)
    j = c1.copy()
    s2 = np.flatnonzero(c1 == 3)
    assert bool(flags & 2) == bool(s2.size)
    c2, used2 = _unpack(rest, s2.size, 2)
    j[s2] += c2
    s3 = s2[c2 == 3]
    assert bool(flags & 4) == bool(s3.size)
    nib, used3 = _unpack(rest[used2:], s3.size, 4)
    j[s3] = 6 + nib
    sl = s3[nib == 15]
    assert bool(flags & 8) == bool(sl.size)
    e = (E - j) & 0xFF
    e[sl] = rest[used2 + used3:used2 + used3 + sl.size]
    used = used2 + used3 + ((sl.size + 3) & ~3)
    assert not np.any(rest[used2 + used3 + sl.size:used])
    return (((lo & 0x80) << 8) | (e.astype(np.uint32) << 7) | (lo & 0x7F)).astype(np.uint16), used


def decode_tile(tile: np.ndarray) -> np.ndarray:
    hdr = tile[:32].view("<u4")
    if hdr[0] & (1 << 8):
        assert tile.size == 32 + 2 * TR * TC and not np.any(hdr[1:]) and hdr[0] == 1 << 8
        return tile[32:].view("<u2").reshape(TR, TC).astype(np.uint16)
    out = np.empty((TR, TC), np.uint16)
    off = 32 + 8 * SEG + 8 * 256
    for s in range(8):
        assert int(hdr[s] >> 12) * 4 == off and not (hdr[s] >> 8) & 1
        v, used = decode_segment(int(hdr[s]), tile[32 + s * SEG:32 + (s + 1) * SEG],
                                 tile[32 + 8 * SEG + 256 * s:32 + 8 * SEG + 256 * (s + 1)], tile[off:])
        out[s * SR:(s + 1) * SR] = v.reshape(SR, TC)
        off += used
    assert tile.size == _pad16(off) and not np.any(tile[off:])
    return out


def decode(code: bytes, shapes) -> list:
    c = np.frombuffer(code, np.uint8)
    nt = sum((R // TR) * (C // TC) for R, C in shapes)
    toff = c[:4 * (nt + 1)].view("<u4").astype(np.int64)
    assert toff[0] == _pad16(4 * (nt + 1)) and toff[nt] == c.size
    out, t = [], 0
    for R, C in shapes:
        W = np.empty((R, C), np.uint16)
        for nb in range(R // TR):
            for kb in range(C // TC):
                W[nb * TR:(nb + 1) * TR, kb * TC:(kb + 1) * TC] = decode_tile(c[toff[t]:toff[t + 1]])
                t += 1
        out.append(W)
    return out


def decode_expert(code: bytes, h: int, hi: int) -> np.ndarray:
    W1, W3, W2 = decode(code, [(hi, h), (hi, h), (h, hi)])
    return np.concatenate([W1.ravel(), W3.ravel(), W2.ravel()])


def max_bytes(h: int, hi: int) -> int:
    """Capacity of an expert block's code (every segment raw)."""
    nt = 3 * (h * hi) // (TR * TC)
    return _pad16(4 * (nt + 1)) + nt * (32 + 2 * TR * TC)
