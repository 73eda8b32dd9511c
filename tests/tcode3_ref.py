"""Test infrastructure: the K5 tile code "T3" (paper_2508_21706_b200/csrc/
tcode.cuh) restated in numpy — encoder and decoder — so the byte layout is
pinned on the CPU tier and the GPU encoder is checked byte for byte.

T3 trades ~0.8 bits per weight against T2 for a decoder without per-lane
loops: every exponent is a fixed 3-bit code, the rare escapes (about 1/128
of uniform-init values) are a per-segment list of (position, exponent) the
decoder patches in parallel. It is the code for the case where the expert
kernel, not the host link, bounds the step (every block resident in the
coded hot cache).

  block  = as T2 (tcode_ref.py): [W1 | W3 | W2] cut into 128 x 64 tiles in
           (matrix, row tile, column tile) order; u32 toff[nt + 1], zero-padded
           to 16 B; the tiles, each 16-B aligned.
  tile   = 8 segments of 16 rows x 64 columns.
           u32 hdr[8]: E | nesc << 9 | eoff4 << 20 (nesc escapes of segment s,
           their list at byte 4 * eoff4 of the tile); bit 8 of hdr[0] marks a
           raw tile (every other header word 0, then 128 x 64 bf16 row-major)
             lo[8][1024]   sign << 7 | mantissa (as T2)
             C3[8][32][3]  3-bit codes: "lane" L of a segment owns values
                           32 L .. 32 L + 31 (row L / 2, columns 32 (L % 2) ..);
                           pair k = values 2k, 2k+1 of the lane, k < 15: word
                           k / 5 bits [3 (k % 5), +3) (even) and [16 + 3 (k % 5),
                           +3) (odd); pair 15: bit b of the even / odd code at
                           bit 15 / 31 of word b
             escapes       per segment: u16 pos[nesc] (value order), u8
                           exponent[nesc], zero-padded to 4 B
           zero padding to 16 B.
  value  j = E - e: code j for 0 <= j <= 6, else 7 and an escape entry.
  E      the segment maximum or up to 7 below it, >= 7, with the fewest
         escapes (ties: the higher E). A tile with a segment whose maximum is
         below 7, more than 1023 escapes in a segment, or whose code would not
         be smaller than raw is stored raw."""
import numpy as np

from tcode_ref import SEG, SR, TC, TR, _pad16, tile_segments

CODE_OFF = 32 + 8 * SEG          # 8224
ESC_OFF = CODE_OFF + 8 * 32 * 12  # 11296: first escape list
RAW = 32 + 2 * TR * TC


def choose_base(e: np.ndarray):
    """E of a segment's exponents (None: the tile goes raw)."""
    emax = int(e.max())
    best, base = None, None
    for c in range(8):
        b0 = emax - c
        if b0 < 7:
            break
        j = b0 - e
        n = int(np.sum((j < 0) | (j > 6)))
        if best is None or n < best:
            best, base = n, b0
    return base


def _lane_words(code: np.ndarray) -> np.ndarray:
    """32 lanes x 3 u32 words from 1024 codes (value order)."""
    c = code.reshape(32, 16, 2).astype(np.uint32)  # lane, pair, even/odd
    w = np.zeros((32, 3), np.uint32)
    for k in range(15):
        wi, j = divmod(k, 5)
        w[:, wi] |= (c[:, k, 0] << (3 * j)) | (c[:, k, 1] << (16 + 3 * j))
    for b in range(3):
        w[:, b] |= (((c[:, 15, 0] >> b) & 1) << 15) | (((c[:, 15, 1] >> b) & 1) << 31)
    return w.reshape(96)


def _codes(words: np.ndarray) -> np.ndarray:
    w = words.reshape(32, 3).astype(np.int64)
    c = np.zeros((32, 16, 2), np.int64)
    for k in range(15):
        wi, j = divmod(k, 5)
        c[:, k, 0] = (w[:, wi] >> (3 * j)) & 7
        c[:, k, 1] = (w[:, wi] >> (16 + 3 * j)) & 7
    for b in range(3):
        c[:, 15, 0] |= ((w[:, b] >> 15) & 1) << b
        c[:, 15, 1] |= ((w[:, b] >> 31) & 1) << b
    return c.reshape(SEG)


def encode_tile(W: np.ndarray, nb: int, kb: int) -> bytes:
    segs = tile_segments(W, nb, kb)
    hdr, lo, codes, escs = [], [], [], []
    off = ESC_OFF
    raw = False
    for v in segs:
        v = np.asarray(v, np.uint16).astype(np.int64)
        e = (v >> 7) & 0xFF
        E = choose_base(e)
        if E is None:
            raw = True
            break
        j = E - e
        esc = (j < 0) | (j > 6)
        pos = np.flatnonzero(esc)
        if pos.size > 1023:
            raw = True
            break
        lst = pos.astype("<u2").tobytes() + e[esc].astype(np.uint8).tobytes()
        lst += b"\0" * ((-len(lst)) % 4)
        hdr.append(E | (pos.size << 9) | ((off // 4) << 20))
        lo.append((((v >> 8) & 0x80) | (v & 0x7F)).astype(np.uint8).tobytes())
        codes.append(_lane_words(np.where(esc, 7, j)).astype("<u4").tobytes())
        escs.append(lst)
        off += len(lst)
    if not raw and off // 4 < 4096:
        body = np.array(hdr, "<u4").tobytes() + b"".join(lo) + b"".join(codes) + b"".join(escs)
        body += b"\0" * (_pad16(len(body)) - len(body))
        if len(body) < RAW:
            return body
    t = W[nb * TR:(nb + 1) * TR, kb * TC:(kb + 1) * TC]
    return np.array([1 << 8] + [0] * 7, "<u4").tobytes() + t.astype("<u2").tobytes()


def decode_tile(tile: np.ndarray) -> np.ndarray:
    hdr = tile[:32].view("<u4").astype(np.int64)
    if hdr[0] & (1 << 8):
        assert tile.size == RAW and not np.any(hdr[1:]) and hdr[0] == 1 << 8
        return tile[32:].view("<u2").reshape(TR, TC).astype(np.uint16)
    out = np.empty((TR, TC), np.uint16)
    off = ESC_OFF
    for s in range(8):
        E, n, eoff = int(hdr[s] & 0xFF), int((hdr[s] >> 9) & 0x7FF), int(hdr[s] >> 20) * 4
        assert eoff == off and not (hdr[s] >> 8) & 1 and E >= 7
        lo = tile[32 + s * SEG:32 + (s + 1) * SEG].astype(np.uint32)
        code = _codes(tile[CODE_OFF + 384 * s:CODE_OFF + 384 * (s + 1)].view("<u4"))
        e = (E - code) & 0xFF
        pos = tile[eoff:eoff + 2 * n].view("<u2").astype(np.int64)
        ex = tile[eoff + 2 * n:eoff + 3 * n]
        assert np.all(code[pos] == 7) and np.sum(code == 7) == n and np.all(np.diff(pos) > 0)
        e[pos] = ex
        used = (3 * n + 3) & ~3
        assert not np.any(tile[eoff + 3 * n:eoff + used])
        out[s * SR:(s + 1) * SR] = (((lo & 0x80) << 8) | (e.astype(np.uint32) << 7) | (lo & 0x7F)).reshape(SR, TC)
        off += used
    assert tile.size == _pad16(off) and not np.any(tile[off:])
    return out


def encode(mats) -> bytes:
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
    b = np.asarray(block, np.uint16)
    m = h * hi
    return encode([b[:m].reshape(hi, h), b[m:2 * m].reshape(hi, h), b[2 * m:3 * m].reshape(h, hi)])


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
