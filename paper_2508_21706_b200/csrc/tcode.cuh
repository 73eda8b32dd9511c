// tcode.cuh — K5 tile code "T2": the lossless expert-weight code the fused
// expert kernel (moe_tc.cu, moe_coded_kernel) decodes straight into its
// shared-memory weight tiles, so coded blocks never expand in HBM.
//
// Format (restated in numpy by tests/tcode_ref.py, which pins it):
//   block   the matrices of one expert ([W1 | W3 | W2]: (h_i, h), (h_i, h),
//           (h, h_i) row-major bf16) cut into tiles of 128 rows x 64
//           columns, in (matrix, row tile, column tile) order — one tile =
//           one k-block of the expert kernel's A operand. u32 toff[nt + 1]
//           (tile byte offsets from the block start; toff[nt] = total),
//           zero-padded to 16 B, then the tiles (16-B aligned).
//   tile    8 segments of 16 rows x 64 columns. u32 hdr[8] (E | flags << 8
//           | soff4 << 12; flags 1 raw tile, 2 some value leaves level 1,
//           4 nibble level reached, 8 literals; soff4 = the segment's stream
//           offset / 4), lo[8][1024] (sign << 7 | mantissa), L1[8][256]
//           (2-bit level-1 codes: "lane" L of a segment owns values 32 L ..
//           32 L + 31 = row L / 2, columns 32 (L % 2) ..; its word w at byte
//           8 L + 4 w holds value 16 w + 2 q at bits 2 q and value
//           16 w + 2 q + 1 at bits 16 + 2 q), then per segment a 4-B aligned
//           stream: L2 (2-bit fields, LSB first, for the values whose level-1
//           code is 3, value order), L3 (4-bit nibbles for the values whose
//           level-2 code is 3), literal exponent bytes (nibble 15), zero
//           padding to 4; the tile is padded to 16 B. A raw tile (hdr[0] =
//           1 << 8, other words 0) is the header + 128 x 64 bf16 row-major.
//   value   j = E - e: j <= 2 is its level-1 code; 3..5 codes 3, j - 3;
//           6..20 codes 3, 3, nibble j - 6; otherwise 3, 3, 15 + literal
//           (2, 4, 8, 16 bits). E (>= 6) = the segment maximum or up to 7
//           below it with the fewest code bits.
// Uniform-init weights: ~10.4 bits per weight (the unary code of xfer.cu:
// 10.25), gaussian-like: ~11.0 (unary: 11.45). What it buys is the decoder:
// level 1 is a fixed 2-bit field per value, so every value decodes with 5
// integer ops per pair and no serial dependence; the ~1/7 of values that
// leave level 1 are ranked with one ballot scan per level and rewritten
// from registers.
#pragma once

#include <stdint.h>

namespace smo {

namespace tcode {

constexpr int kTileRows = 128, kTileCols = 64, kSegRows = 16, kSegs = 8;
constexpr int kSeg = kSegRows * kTileCols;        // 1024 values
constexpr int kLoOff = 32;                        // lo[8][1024] after the header
constexpr int kL1Off = kLoOff + kSegs * kSeg;     // L1[8][256]
constexpr int kStreamOff = kL1Off + kSegs * 256;  // 10272: first segment stream
constexpr int kTileMax = 32 + 2 * kTileRows * kTileCols;  // 16416: a raw tile, the largest
// T3 (tests/tcode3_ref.py): hdr[8] = E | nesc << 9 | eoff4 << 20 (bit 8 of
// hdr[0]: raw tile), lo[8][1024], 3-bit codes C3[8][32 lanes][3 words], per
// segment an escape list (u16 positions, then u8 exponents, padded to 4 B)
constexpr int kC3Off = kLoOff + kSegs * kSeg;     // 8224
constexpr int kEsc3Off = kC3Off + kSegs * 384;    // 11296: first escape list

__device__ __forceinline__ int warp_excl_scan(int v, int lane, int* total) {
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  *total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

// Decode segment s of a tile whose code sits in shared memory at `tc` into
// the 128B-swizzled bf16 tile at `tile` (128 rows of 128 B, 1024-B aligned;
// 16-B chunk c of row r at (c ^ (r & 7)) — what TMA SWIZZLE_128B writes and
// the UMMA descriptors read). One warp; every lane writes its half-row with
// four 16-B stores, then rewrites the values that left level 1 (one warp scan
// per level ranks the lanes' fields; each lane walks its own from a register
// window).
__device__ __forceinline__ void decode_segment(const uint8_t* __restrict__ tc, uint8_t* tile, int s, int lane,
                                               uint32_t hw_mask = 0xffffffffu) {
  const int r = kSegRows * s + (lane >> 1);
  const int half = lane & 1;
  uint8_t* rowp = tile + r * 128;
  const int x = r & 7;
  const uint32_t* hdr = reinterpret_cast<const uint32_t*>(tc);
  if (hdr[0] & 0x100u) {  // raw tile: lane L's 64 bytes are its half-row
    const uint4* src = reinterpret_cast<const uint4*>(tc + 32 + 2 * kSeg * s) + 4 * lane;
#pragma unroll
    for (int k = 0; k < 4; ++k) *reinterpret_cast<uint4*>(rowp + (((4 * half + k) ^ x) << 4)) = src[k];
    return;
  }
  const uint32_t hw = hdr[s] & hw_mask;
  const uint32_t E = hw & 0xffu;
  const uint8_t* lob = tc + kLoOff + kSeg * s;
  const uint4 lo0 = reinterpret_cast<const uint4*>(lob)[2 * lane];
  const uint4 lo1 = reinterpret_cast<const uint4*>(lob)[2 * lane + 1];
  const uint2 cw = reinterpret_cast<const uint2*>(tc + kL1Off + 256 * s)[lane];
  const uint32_t lw[8] = {lo0.x, lo0.y, lo0.z, lo0.w, lo1.x, lo1.y, lo1.z, lo1.w};
  const uint32_t e2 = (E << 7) | (E << 23);
  const uint32_t* st = reinterpret_cast<const uint32_t*>(tc + 4 * (hw >> 12));
  // Level 2 first, into registers: the values whose level-1 code is 3 (bit i
  // = value i of the lane) take their 2-bit code c2 from the lane's run of
  // fields (consecutive from its rank; <= 16 sit in one register window) and
  // deposit it in d0 / d1, laid out like the level-1 words, so the pair
  // compose below subtracts both codes at once: e = E - c1 - c2 (E >= 6, so
  // E - 6 never borrows). Per escape this is ALU work only.
  uint32_t d0 = 0u, d1 = 0u, m3 = 0u;
  int tot2 = 0;
  if (hw & 0x200u) {  // warp-uniform
    const uint32_t m0 = cw.x & (cw.x >> 1), m1 = cw.y & (cw.y >> 1);
    const uint32_t m2 = ((m0 & 0x5555u) | ((m0 >> 15) & 0xAAAAu)) | (((m1 & 0x5555u) | ((m1 >> 15) & 0xAAAAu)) << 16);
    const int n2 = __popc(m2);
    const int r2 = warp_excl_scan(n2, lane, &tot2);
    auto dep = [&](int i, uint32_t c) {
      const uint32_t v = c << ((i & 14) | ((i & 1) << 4));
      if (i < 16) d0 |= v;
      else d1 |= v;
      m3 |= (c == 3u ? 1u : 0u) << i;
    };
    if (__all_sync(0xffffffffu, n2 <= 16)) {
      const int nw = (tot2 + 15) >> 4, wi = r2 >> 4;
      const uint32_t w0 = wi < nw ? st[wi] : 0u, w1 = wi + 1 < nw ? st[wi + 1] : 0u;
      uint32_t win = uint32_t(((uint64_t(w1) << 32) | w0) >> (2 * (r2 & 15)));
      for (uint32_t mm = m2; mm; mm &= mm - 1u) {
        dep(__ffs(mm) - 1, win & 3u);
        win >>= 2;
      }
    } else {  // > 16 in some lane (wide-range data): fields from shared memory
      int f = r2;
      for (uint32_t mm = m2; mm; mm &= mm - 1u, ++f) dep(__ffs(mm) - 1, (st[f >> 4] >> (2 * (f & 15))) & 3u);
    }
  }
  uint32_t out[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    // pair k = values 2k, 2k+1: codes at bits 2q and 16 + 2q of word k / 8,
    // moved to the exponent fields (bits 7-8 and 23-24) and subtracted from E
    const int q = k & 7;
    const uint32_t w = k < 8 ? cw.x : cw.y, dw = k < 8 ? d0 : d1;
    const uint32_t cc = (q <= 3 ? (w << (7 - 2 * q)) : (w >> (2 * q - 7))) & 0x01800180u;
    const uint32_t dd = (q <= 3 ? (dw << (7 - 2 * q)) : (dw >> (2 * q - 7))) & 0x01800180u;
    // two lo bytes -> 16-bit lanes with the sign replicated into the high byte
    const uint32_t t = __byte_perm(lw[k >> 1], 0u, (k & 1) ? 0xB3A2u : 0x9180u);
    out[k] = (t & 0x807F807Fu) | (e2 - cc - dd);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
    *reinterpret_cast<uint4*>(rowp + (((4 * half + k) ^ x) << 4)) =
        make_uint4(out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]);
  // value i of this lane rewritten whole with exponent e: its sign /
  // mantissa byte from lo, at 16-B chunk (4 half + i / 8) ^ x of the row,
  // i.e. byte ((hx << 3) ^ i) << 1 of the row with hx = 4 half ^ x
  const uint8_t* mylo = lob + 32 * lane;
  const int hx3 = ((4 * half) ^ x) << 3;
  auto put = [&](int i, uint32_t e) {
    const uint32_t lo = mylo[i];
    *reinterpret_cast<uint16_t*>(rowp + ((hx3 ^ i) << 1)) = uint16_t(((lo & 0x80u) << 8) | (e << 7) | (lo & 0x7fu));
  };
  if (!(hw & 0x400u)) return;  // no value reaches the nibble level
  // level 3: nibbles j - 6 of the values whose level-2 code is 3
  const uint32_t* st3 = st + ((tot2 + 15) >> 4);
  int tot3 = 0;
  const int n3 = __popc(m3);
  const int r3 = warp_excl_scan(n3, lane, &tot3);
  uint32_t ml = 0u;
  if (__all_sync(0xffffffffu, n3 <= 8)) {
    const int nw = (tot3 + 7) >> 3, wi = r3 >> 3;
    const uint32_t w0 = wi < nw ? st3[wi] : 0u, w1 = wi + 1 < nw ? st3[wi + 1] : 0u;
    uint32_t win = uint32_t(((uint64_t(w1) << 32) | w0) >> (4 * (r3 & 7)));
    for (uint32_t mm = m3; mm; mm &= mm - 1u) {
      const int i = __ffs(mm) - 1;
      const uint32_t c = win & 15u;
      win >>= 4;
      if (c == 15u) ml |= 1u << i;
      else put(i, E - 6u - c);
    }
  } else {
    int f = r3;
    for (uint32_t mm = m3; mm; mm &= mm - 1u, ++f) {
      const int i = __ffs(mm) - 1;
      const uint32_t c = (st3[f >> 3] >> (4 * (f & 7))) & 15u;
      if (c == 15u) ml |= 1u << i;
      else put(i, E - 6u - c);
    }
  }
  if (!(hw & 0x800u)) return;
  // literal exponent bytes, in value order
  const uint8_t* lit = reinterpret_cast<const uint8_t*>(st3 + ((tot3 + 7) >> 3));
  int totl = 0;
  int f = warp_excl_scan(__popc(ml), lane, &totl);
  for (uint32_t mm = ml; mm; mm &= mm - 1u) put(__ffs(mm) - 1, lit[f++]);
}

// T3: decode segment s into the swizzled tile (one warp). Every value is a
// fixed 3-bit code j = E - e (7: escape); pair k < 15 of lane L sits at bits
// 3 (k % 5) (even) and 16 + 3 (k % 5) (odd) of word k / 5, so one shift and
// mask place both codes under the bf16 pair's exponent fields (E >= 7: no
// borrow) — five integer ops per pair and no per-lane loop. The escapes
// (code 7) are rewritten afterwards from the segment's (position, exponent)
// list, the warp's lanes taking consecutive entries.
__device__ __forceinline__ void decode_segment3(const uint8_t* __restrict__ tc, uint8_t* tile, int s, int lane) {
  const int r = kSegRows * s + (lane >> 1);
  const int half = lane & 1;
  uint8_t* rowp = tile + r * 128;
  const int x = r & 7;
  const uint32_t* hdr = reinterpret_cast<const uint32_t*>(tc);
  if (hdr[0] & 0x100u) {  // raw tile: lane L's 64 bytes are its half-row
    const uint4* src = reinterpret_cast<const uint4*>(tc + 32 + 2 * kSeg * s) + 4 * lane;
#pragma unroll
    for (int k = 0; k < 4; ++k) *reinterpret_cast<uint4*>(rowp + (((4 * half + k) ^ x) << 4)) = src[k];
    return;
  }
  const uint32_t hw = hdr[s];
  const uint32_t E = hw & 0xffu;
  const uint8_t* lob = tc + kLoOff + kSeg * s;
  const uint4 lo0 = reinterpret_cast<const uint4*>(lob)[2 * lane];
  const uint4 lo1 = reinterpret_cast<const uint4*>(lob)[2 * lane + 1];
  const uint32_t* cw = reinterpret_cast<const uint32_t*>(tc + kC3Off + 384 * s) + 3 * lane;
  const uint32_t w0 = cw[0], w1 = cw[1], w2 = cw[2];
  const uint32_t lw[8] = {lo0.x, lo0.y, lo0.z, lo0.w, lo1.x, lo1.y, lo1.z, lo1.w};
  const uint32_t e2 = (E << 7) | (E << 23);
  uint32_t out[16];
#pragma unroll
  for (int k = 0; k < 15; ++k) {
    const int j = k % 5;
    const uint32_t w = k < 5 ? w0 : k < 10 ? w1 : w2;
    const uint32_t cc = (3 * j <= 7 ? (w << (7 - 3 * j)) : (w >> (3 * j - 7))) & 0x03800380u;
    const uint32_t t = __byte_perm(lw[k >> 1], 0u, (k & 1) ? 0xB3A2u : 0x9180u);
    out[k] = (t & 0x807F807Fu) | (e2 - cc);
  }
  {  // pair 15: code bit b of the even / odd value at bit 15 / 31 of word b
    const uint32_t ce = ((w0 >> 15) & 1u) | ((w1 >> 14) & 2u) | ((w2 >> 13) & 4u);
    const uint32_t co = (w0 >> 31) | ((w1 >> 30) & 2u) | ((w2 >> 29) & 4u);
    const uint32_t t = __byte_perm(lw[7], 0u, 0xB3A2u);
    out[15] = (t & 0x807F807Fu) | (e2 - ((ce << 7) | (co << 23)));
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
    *reinterpret_cast<uint4*>(rowp + (((4 * half + k) ^ x) << 4)) =
        make_uint4(out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]);
  const int nesc = int((hw >> 9) & 0x7ffu);
  if (nesc) {  // warp-uniform
    __syncwarp();  // the escape's row may belong to another lane's stores
    const uint8_t* el = tc + 4 * (hw >> 20);
    for (int q = lane; q < nesc; q += 32) {
      const int pos = reinterpret_cast<const uint16_t*>(el)[q];
      const uint32_t e = el[2 * nesc + q];
      const int r2 = kSegRows * s + (pos >> 6), c = pos & 63;
      const uint32_t lo = lob[pos];
      *reinterpret_cast<uint16_t*>(tile + r2 * 128 + ((((c >> 3) ^ (r2 & 7)) << 4) | ((c & 7) << 1))) =
          uint16_t(((lo & 0x80u) << 8) | (e << 7) | (lo & 0x7fu));
    }
  }
}

}  // namespace tcode

}  // namespace smo
