"""Test infrastructure: the K5 unary link format (paper_2508_21706_b200/csrc/
xfer.cu header) restated in numpy — encoder and decoder — so the byte layout
is pinned on the CPU tier and the GPU encoder is checked byte for byte.

Format, per block of n bf16 values (n % 1024 == 0, segments of 1024):
  table: (segs + 1) entries of 8 bytes (offset u32, base E u8, flags u8,
         words u16), entry [segs].offset = total bytes; zero-padded to 16 B.
  segment (16-B aligned): lo[1024] = sign << 7 | mantissa; `words` 32-bit
         code words, MSB-first: value i codes j = E - e ones then a zero
         (j = 15 escapes: e > E or e <= E - 15, literal exponent byte in the
         escape list); bits after the last code are ones; escape bytes in
         position order; zero padding.
  E = the segment maximum or up to 7 below it, the fewest bits wins (ties:
  the higher E)."""
import numpy as np

SEG, ESC = 1024, 15


def encode(x: np.ndarray) -> bytes:
    x = np.asarray(x, np.uint16)
    assert x.size % SEG == 0
    segs = x.size // SEG
    table = np.zeros((segs + 1, 2), np.uint32)
    tbytes = ((segs + 1) * 8 + 15) & ~15
    body = []
    off = tbytes
    for s in range(segs):
        v = x[s * SEG:(s + 1) * SEG].astype(np.int64)
        e = (v >> 7) & 0xFF
        emax = int(e.max())
        base, best = emax, None
        for c in range(8):
            b0 = emax - c
            if b0 < 0:
                break
            cost = int(np.sum(np.where(e <= b0, np.minimum(b0 - e, ESC) + 1, ESC + 1 + 8)))
            if best is None or cost < best:
                best, base = cost, b0
        j = np.where(e <= base, np.minimum(base - e, ESC), ESC)
        bits = np.ones(int(np.sum(j + 1)), np.uint8)
        ends = np.cumsum(j + 1) - 1
        bits[ends] = 0
        nw = (bits.size + 31) // 32
        bits = np.concatenate([bits, np.ones(nw * 32 - bits.size, np.uint8)])
        words = np.packbits(bits).view(">u4").astype("<u4")  # MSB-first within each word
        lo = (((v >> 8) & 0x80) | (v & 0x7F)).astype(np.uint8)
        esc = e[j == ESC].astype(np.uint8)
        seg = lo.tobytes() + words.tobytes() + esc.tobytes()
        seg += b"\0" * ((-len(seg)) % 16)
        table[s, 0] = off
        table[s, 1] = base | ((1 if esc.size else 0) << 8) | (nw << 16)
        body.append(seg)
        off += len(seg)
    table[segs, 0] = off
    head = table.astype("<u4").tobytes()
    head += b"\0" * (tbytes - len(head))
    return head + b"".join(body)


def decode(code: bytes, n: int) -> np.ndarray:
    c = np.frombuffer(code, np.uint8)
    segs = n // SEG
    out = np.empty(n, np.uint16)
    for s in range(segs):
        t = c[8 * s:8 * s + 8]
        off = int(t[:4].view("<u4")[0])
        base, flags, nw = int(t[4]), int(t[5]), int(t[6:8].view("<u2")[0])
        lo = c[off:off + SEG].astype(np.uint32)
        words = c[off + SEG:off + SEG + 4 * nw].view("<u4")
        bits = np.unpackbits(words.astype(">u4").view(np.uint8))
        zeros = np.flatnonzero(bits == 0)
        assert len(zeros) == SEG and np.all(bits[zeros[-1] + 1:] == 1)
        j = np.diff(np.concatenate([[-1], zeros])) - 1
        e = (base - j).astype(np.int64) & 0xFF
        at = np.flatnonzero(j >= ESC)
        assert flags == (1 if at.size else 0)
        e[at] = c[off + SEG + 4 * nw:off + SEG + 4 * nw + at.size]
        out[s * SEG:(s + 1) * SEG] = (((lo & 0x80) << 8) | (e.astype(np.uint32) << 7) | (lo & 0x7F)).astype(np.uint16)
    return out


def total_bytes(code: bytes, n: int) -> int:
    segs = n // SEG
    return int(np.frombuffer(code, np.uint8)[8 * segs:8 * segs + 4].view("<u4")[0])
