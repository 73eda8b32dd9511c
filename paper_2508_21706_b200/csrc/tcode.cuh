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
//   tile    u32 hdr[8] (E | flags << 8 | size16 << 16; flags bit 0 raw,
//           bit 1 some value escapes level 1; size16 = segment bytes / 16),
//           then 8 segments of 16 rows x 64 columns.
//   segment value order v = 64 r + c; "lane" L owns values 32 L .. 32 L + 31
//           (row L / 2, columns 32 (L % 2) ..). Raw: 1024 bf16. Coded:
//           lo[1024] (sign << 7 | mantissa), L1[256] (2-bit level-1 codes:
//           lane L's word w at byte 8 L + 4 w holds value 16 w + 2 q at bits
//           2 q and value 16 w + 2 q + 1 at bits 16 + 2 q), the level stream
//           (2-bit fields LSB first: level-2 codes of the values whose level-1
//           code is 3, in value order, then level 3, ... 5), literal exponent
//           bytes (values whose five codes are all 3), zero padding to 16 B.
//   value   j = E - e; 0 <= j <= 14: j // 3 + 1 levels (3 on all but the
//           last, j - 3 (levels - 1) on the last); otherwise five 3s and a
//           literal. E (>= 3) = the segment maximum or up to 7 below it with
//           the fewest code bits; >= 2048 coded bytes -> raw.
// Uniform-init weights: ~10.4 bits per weight (the unary code of xfer.cu:
// 10.25), gaussian-like: ~10.9 (unary: 11.45). What it buys is the decoder:
// level 1 is a fixed 2-bit field per value, so 30 of every 32 values decode
// with 5 integer ops per pair and no serial dependence; only the ~1/8 of
// values that escape level 1 take a short ranked walk.
#pragma once

#include <stdint.h>

namespace smo {

namespace tcode {

constexpr int kTileRows = 128, kTileCols = 64, kSegRows = 16, kSegs = 8;
constexpr int kSeg = kSegRows * kTileCols;         // 1024 values
constexpr int kRawBytes = 2 * kSeg;                // 2048
constexpr int kL1Off = kSeg;                       // L1 codes after lo
constexpr int kLvOff = kSeg + 256;                 // level stream
constexpr int kTileMax = 32 + kSegs * kRawBytes;   // 16416: the largest tile code

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

// Decode segment s of a tile (code in shared memory at `seg`, header word hw)
// into the 128B-swizzled bf16 tile at `tile` (128 rows of 128 B, 1024-B
// aligned; 16-B chunk c of row r at (c ^ (r & 7)) — what TMA SWIZZLE_128B
// writes and the UMMA descriptors read). One warp; every lane writes its
// half-row with four 16-B stores, escaped values are then patched in place.
__device__ __forceinline__ void decode_segment(const uint8_t* __restrict__ seg, uint32_t hw, uint8_t* tile, int s,
                                               int lane) {
  const int r = kSegRows * s + (lane >> 1);
  const int half = lane & 1;
  uint8_t* rowp = tile + r * 128;
  const int x = r & 7;
  if (hw & 0x100u) {  // raw segment: lane L's 64 bytes are its half-row
    const uint4* src = reinterpret_cast<const uint4*>(seg) + 4 * lane;
#pragma unroll
    for (int k = 0; k < 4; ++k) *reinterpret_cast<uint4*>(rowp + (((4 * half + k) ^ x) << 4)) = src[k];
    return;
  }
  const uint32_t E = hw & 0xffu;
  const uint4 lo0 = reinterpret_cast<const uint4*>(seg)[2 * lane];
  const uint4 lo1 = reinterpret_cast<const uint4*>(seg)[2 * lane + 1];
  const uint2 cw = reinterpret_cast<const uint2*>(seg + kL1Off)[lane];
  const uint32_t lw[8] = {lo0.x, lo0.y, lo0.z, lo0.w, lo1.x, lo1.y, lo1.z, lo1.w};
  const uint32_t e2 = (E << 7) | (E << 23);
  uint32_t out[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    // pair k = values 2k, 2k+1: codes at bits 2q and 16 + 2q of word k / 8,
    // moved to the exponent fields (bits 7-8 and 23-24) and subtracted from E
    const uint32_t w = k < 8 ? cw.x : cw.y;
    const int q = k & 7;
    const uint32_t cc = (q <= 3 ? (w << (7 - 2 * q)) : (w >> (2 * q - 7))) & 0x01800180u;
    // two lo bytes -> 16-bit lanes with the sign replicated into the high byte
    const uint32_t t = __byte_perm(lw[k >> 1], 0u, (k & 1) ? 0xB3A2u : 0x9180u);
    out[k] = (t & 0x807F807Fu) | (e2 - cc);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
    *reinterpret_cast<uint4*>(rowp + (((4 * half + k) ^ x) << 4)) =
        make_uint4(out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]);
  if (!(hw & 0x200u)) return;  // no value escapes level 1 (warp-uniform)
  // values whose level-1 code is 3, as a value-indexed mask (bit i = value i)
  const uint32_t m0 = cw.x & (cw.x >> 1), m1 = cw.y & (cw.y >> 1);
  uint32_t m = ((m0 & 0x5555u) | ((m0 >> 15) & 0xAAAAu)) | (((m1 & 0x5555u) | ((m1 >> 15) & 0xAAAAu)) << 16);
  const uint32_t* lv = reinterpret_cast<const uint32_t*>(seg + kLvOff);
  auto at = [&](int i) -> uint16_t* {
    return reinterpret_cast<uint16_t*>(rowp + (((4 * half + (i >> 3)) ^ x) << 4) + ((i & 7) << 1));
  };
  int base = 0;  // fields of the earlier levels
#pragma unroll 1
  for (int lev = 2; lev <= 5; ++lev) {
    int tot = 0;
    int f = base + warp_excl_scan(__popc(m), lane, &tot);
    if (tot == 0) break;
    uint32_t next = 0u;
    for (uint32_t mm = m; mm; mm &= mm - 1u) {
      const int i = __ffs(mm) - 1;
      const uint32_t c = (lv[f >> 4] >> (2 * (f & 15))) & 3u;
      ++f;
      // the value ends here: j = 3 (lev - 1) + c, stored as E - 3 so far
      // (e >= 0, so the subtraction never borrows into the sign)
      const uint32_t dj = 3u * uint32_t(lev - 2) + c;
      if (c != 3u && dj) {
        uint16_t* p = at(i);
        *p = uint16_t(*p - (dj << 7));
      }
      next |= (c == 3u ? 1u : 0u) << i;
    }
    base += tot;
    m = next;
  }
  // values whose five codes are all 3: literal exponent bytes, in value order
  int tot = 0;
  int f = warp_excl_scan(__popc(m), lane, &tot);
  if (tot) {
    const uint8_t* lit = reinterpret_cast<const uint8_t*>(lv + ((base + 15) >> 4));
    for (uint32_t mm = m; mm; mm &= mm - 1u) {
      uint16_t* p = at(__ffs(mm) - 1);
      *p = uint16_t((*p & 0x807Fu) | (uint32_t(lit[f++]) << 7));
    }
  }
}

}  // namespace tcode

}  // namespace smo
