// xfer.cu — K5 codec: lossless packing of expert weights for the host link.
//
// The verify step is bound by the PCIe link (55.6 GB/s on this box whatever
// the copy-stream count or pinned-memory flavour, profiles/r01_h2d_link.jsonl),
// so the bytes that cross it are the step time. bf16 weights carry an 8-bit
// exponent that takes few values inside a block; this format keeps sign and
// mantissa verbatim and codes the exponent in B bits (B = 3 or 4) relative to
// a per-segment base — bit-exact, 11.4 (B = 3) or 12.4 (B = 4) bits/weight.
//
// Segment = 1024 consecutive bf16 values, 16 + 1024 + 128 B + 32 bytes:
//   [0, 16)               header: byte 0 = base exponent, byte 1 = escapes
//   [16, 1040)            lo[i] = sign << 7 | mantissa (7 bits)
//   [1040, 1040 + 128 B)  B-bit exponent codes in value order: value i's
//                         code at bits [B i, B i + B), little-endian (code
//                         c < 2^B - 1: exponent = base + c; 2^B - 1: escape)
//   [.., + 32)            up to 32 escaped exponents, in position order
// base: of the W = 2^B - 1 windows ending at e_max, e_max - 1, ..., e_max - 6
// the one holding the most values (a few large outliers then escape instead
// of dragging the window up). A segment with more than 32 escapes cannot be
// coded: the encoder raises a flag; callers retry with B = 4, then keep the
// block raw (bf16) — lossless either way. Uniform-init weights code at B = 3
// (0.8 % escapes), gaussian-like trained weights need B = 4.
// One warp per segment in both directions; lane l owns the 8-value groups
// 32q + l, so every memory instruction is one contiguous run; escapes are
// ranked in position order with a warp exclusive scan per group column.
//
// Unary format (bits = 1, variable length, the engine's first choice):
// exponent e of a segment with base E codes as j = E - e ONES followed by
// a ZERO (bit stream MSB-first in 32-bit words: stream bit k = bit
// 31 - k % 32 of word k / 32, so a code's length is one count-leading-ones); j = 15 is an escape (15 ones + zero, the
// exponent byte in the escape list) for e > E or e <= E - 15. E is the
// segment maximum or up to 7 below it, whichever gives the fewest bits. For uniform-init weights j is geometric
// with p = 1/2 — unary is its optimal prefix code, 2 bits per exponent on
// average: ~10.2 bits/weight (1.57x) against 11.4 for the 3-bit window, and
// 3.3 instead of 4 bits for gaussian weights. Block layout:
//   table  USeg[segs + 1] (8 B each: byte offset of the segment in the block,
//          base E, 1 if the segment has escapes, stream words nw), entry [segs].off = total coded bytes;
//          padded to 16 B
//   per segment (16-B aligned): lo[1024] (sign << 7 | mantissa), nw 32-bit
//          code words (trailing bits of the last word are ones), escaped
//          exponent bytes in position order, zero padding.
// Decoding is parallel without per-value offsets: value i ends at the i-th
// zero of the stream, so where each lane's run of 32 values starts follows
// from a warp scan of zero counts per code word.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace smo {

namespace {

constexpr int kSeg = 1024;
constexpr int kLoOff = 16, kCodeOff = 1040, kMaxEsc = 32;
template <int B>
struct Fmt {
  static constexpr int kCodeBytes = 128 * B;       // 1024 codes of B bits
  static constexpr int kEscOff = kCodeOff + kCodeBytes;
  static constexpr int kSegBytes = kEscOff + kMaxEsc;  // 1456 (B=3), 1584 (B=4)
  static constexpr int kWin = (1 << B) - 1;         // exponents a code can name
  static constexpr uint32_t kEscape = (1u << B) - 1u;
  static constexpr uint32_t kLsbMask = B == 3 ? 0x00249249u : 0x11111111u;  // bit 0 of each of 8 fields
};

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

// Lane l of a segment's warp owns the four 8-value groups G = 32q + l
// (q = 0..3): every load and store instruction of the warp then touches one
// contiguous run (512 B of bf16, 256 B of lo bytes, 32·B bytes of codes).
template <int B>
__device__ __forceinline__ uint32_t load_group_codes(const uint8_t* codes, int G) {
  if constexpr (B == 4) return reinterpret_cast<const uint32_t*>(codes)[G];
  const uint8_t* c = codes + 3 * G;
  return uint32_t(c[0]) | (uint32_t(c[1]) << 8) | (uint32_t(c[2]) << 16);
}
template <int B>
__device__ __forceinline__ void store_group_codes(uint8_t* codes, int G, uint32_t w) {
  if constexpr (B == 4) {
    reinterpret_cast<uint32_t*>(codes)[G] = w;
  } else {
    uint8_t* c = codes + 3 * G;
    c[0] = uint8_t(w);
    c[1] = uint8_t(w >> 8);
    c[2] = uint8_t(w >> 16);
  }
}

template <int B>
__global__ void expert_encode_kernel(const uint16_t* __restrict__ src, size_t segs, uint8_t* __restrict__ dst,
                                     int* __restrict__ overflow) {
  using F = Fmt<B>;
  const size_t warp = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (warp >= segs) return;
  const uint16_t* s = src + warp * kSeg;
  uint8_t* d = dst + warp * F::kSegBytes;
  uint16_t v[32];  // v[8q + j] = value 8 (32q + lane) + j
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 u = reinterpret_cast<const uint4*>(s)[32 * q + lane];
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      v[q * 8 + 2 * t] = uint16_t(w[t] & 0xffffu);
      v[q * 8 + 2 * t + 1] = uint16_t(w[t] >> 16);
    }
  }
  int emax = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) emax = max(emax, int((v[j] >> 7) & 0xff));
#pragma unroll
  for (int o = 16; o; o >>= 1) emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  // the window [base, base + kWin) with the most values among the 7 ending
  // at e_max .. e_max - 6 (ties: the higher window)
  int base = max(emax - (F::kWin - 1), 0), best = -1;
#pragma unroll
  for (int sh = 0; sh < 7; ++sh) {
    const int b0 = emax - (F::kWin - 1) - sh;
    if (b0 < 0) break;
    int c = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int e = (v[j] >> 7) & 0xff;
      c += (e >= b0 && e < b0 + F::kWin) ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (c > best) {
      best = c;
      base = b0;
    }
  }
  // escapes in position order: group-major (q), then lane
  int at[4], total = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int e = (v[8 * q + j] >> 7) & 0xff;
      cnt += (e >= base && e < base + F::kWin) ? 0 : 1;
    }
    int tq = 0;
    at[q] = total + warp_excl_scan(cnt, lane, &tq);
    total += tq;
  }
  if (total > kMaxEsc) {
    if (lane == 0) atomicOr(overflow, 1);
    return;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int G = 32 * q + lane;
    uint32_t code = 0u, lo0 = 0u, lo1 = 0u;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t x = v[8 * q + j];
      const int e = int((x >> 7) & 0xffu);
      const bool in = e >= base && e < base + F::kWin;
      code |= (in ? uint32_t(e - base) : F::kEscape) << (B * j);
      if (!in) d[F::kEscOff + at[q]++] = uint8_t(e);
      const uint32_t lo = ((x >> 8) & 0x80u) | (x & 0x7fu);
      if (j < 4) lo0 |= lo << (8 * j);
      else lo1 |= lo << (8 * (j - 4));
    }
    reinterpret_cast<uint2*>(d + kLoOff)[G] = make_uint2(lo0, lo1);
    store_group_codes<B>(d + kCodeOff, G, code);
  }
  if (lane == 0) *reinterpret_cast<uint4*>(d) = make_uint4(uint32_t(base) | (uint32_t(total) << 8), 0u, 0u, 0u);
  if (lane < kMaxEsc - total) d[F::kEscOff + total + lane] = 0;  // deterministic padding
}

// Decode stages the warp's whole segment in shared memory with coalesced
// 16-byte loads first (3 per lane, all in flight together), then expands it
// from there — the byte-granular code / escape reads never wait on DRAM.
constexpr int kDecWarps = 8;
constexpr int kDecSegs = 1;  // segments per warp (2: 135 us vs 117 us per Mixtral block, profiles/r01_codec.md)
// Up to 64 equally sized blocks per launch (one layer's experts): blockIdx.y
// picks the block, so a layer's expansion is one launch with no tail per block.
struct DecodeJobs {
  const uint8_t* src[64];
  uint16_t* dst[64];
};

template <int B>
__global__ void __launch_bounds__(32 * kDecWarps) expert_decode_kernel(const __grid_constant__ DecodeJobs jobs,
                                                                       size_t segs) {
  using F = Fmt<B>;
  const uint8_t* __restrict__ src = jobs.src[blockIdx.y];
  uint16_t* __restrict__ dst = jobs.dst[blockIdx.y];
  constexpr int kVec = F::kSegBytes / 16;  // 91 (B = 3) or 99 (B = 4) uint4 per segment
  constexpr int kLd = (kDecSegs * kVec + 31) / 32;
  __shared__ uint4 stage[kDecWarps][kDecSegs * kVec];
  const int wib = threadIdx.x / 32, lane = threadIdx.x % 32;
  const size_t seg0 = (size_t(blockIdx.x) * kDecWarps + wib) * kDecSegs;
  if (seg0 >= segs) return;
  const int nseg = segs - seg0 < size_t(kDecSegs) ? int(segs - seg0) : kDecSegs;
  // all of the warp's segments in flight at once (contiguous in the code)
  const uint4* g = reinterpret_cast<const uint4*>(src + seg0 * F::kSegBytes);
  uint4 r[kLd];
#pragma unroll
  for (int i = 0; i < kLd; ++i)
    if (lane + 32 * i < nseg * kVec) r[i] = g[lane + 32 * i];
#pragma unroll
  for (int i = 0; i < kLd; ++i)
    if (lane + 32 * i < nseg * kVec) stage[wib][lane + 32 * i] = r[i];
  __syncwarp();
  for (int sg = 0; sg < nseg; ++sg) {
  const uint8_t* s = reinterpret_cast<const uint8_t*>(stage[wib] + sg * kVec);
  const int base = int(s[0]);
  uint4* d = reinterpret_cast<uint4*>(dst + (seg0 + sg) * kSeg);
  // escape counts of the lane's four groups packed in 8-bit fields (each
  // column sum <= 32 escapes per segment): one warp scan ranks them all
  uint2 lo[4];
  uint32_t code[4], em[4];
  uint32_t packed = 0u;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int G = 32 * q + lane;
    lo[q] = reinterpret_cast<const uint2*>(s + kLoOff)[G];
    code[q] = load_group_codes<B>(s + kCodeOff, G);
    // escape fields are all-ones: AND the field's bits down onto its LSB
    uint32_t m = code[q];
#pragma unroll
    for (int b = 1; b < B; ++b) m &= code[q] >> b;
    em[q] = m & F::kLsbMask;
    packed |= uint32_t(__popc(em[q])) << (8 * q);
  }
  int ptot = 0;
  const uint32_t pexcl = uint32_t(warp_excl_scan(int(packed), lane, &ptot));
  int col = 0;  // escapes in the columns q' < q (all lanes)
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int G = 32 * q + lane;
    int at = col + int((pexcl >> (8 * q)) & 0xffu);
    col += (ptot >> (8 * q)) & 0xff;
    // two values per 32-bit word: lo bytes spread to 16-bit lanes (PRMT),
    // exponents base + code added in both lanes at once; escaped values
    // (rare) are patched afterwards, so warps never split into two paths
    uint32_t out[4];
    const uint32_t base2 = uint32_t(base) * 0x10001u;
#pragma unroll
    for (int p2 = 0; p2 < 4; ++p2) {
      const uint32_t lw = p2 < 2 ? lo[q].x : lo[q].y;
      const uint32_t l16 = __byte_perm(lw, 0u, (p2 & 1) ? 0x4342u : 0x4140u);
      const uint32_t c2 =
          ((code[q] >> (2 * B * p2)) & F::kEscape) | (((code[q] >> (2 * B * p2 + B)) & F::kEscape) << 16);
      out[p2] = ((l16 & 0x00800080u) << 8) | (l16 & 0x007f007fu) | ((base2 + c2) << 7);
    }
    for (uint32_t m = em[q]; m; m &= m - 1u) {
      const int j = (__ffs(m) - 1) / B;  // escapes in position order
      const int sh = 7 + 16 * (j & 1);
      const uint32_t e = uint32_t(s[F::kEscOff + at++]);
      const uint32_t keep = ~(0xffu << sh);
#pragma unroll
      for (int p2 = 0; p2 < 4; ++p2)
        if (p2 == (j >> 1)) out[p2] = (out[p2] & keep) | (e << sh);
    }
    d[G] = make_uint4(out[0], out[1], out[2], out[3]);
  }
  }
}

// ---------------------------------------------------------------- unary
struct USeg {
  uint32_t off;   // segment byte offset in the block (entry [segs]: total bytes)
  uint8_t emax;   // largest exponent of the segment
  uint8_t flags;  // bit 0: the segment has escapes
  uint16_t nw;    // code stream words
};
static_assert(sizeof(USeg) == 8, "USeg is 8 bytes");
constexpr int kUEsc = 15;        // j >= 15 escapes
constexpr int kUMaxWords = 512;  // 1024 codes of <= 16 bits
constexpr int kUEncWarps = 8;
__host__ __device__ inline size_t u_table_bytes(size_t segs) { return ((segs + 1) * sizeof(USeg) + 15) & ~size_t(15); }

// Pass 1 (write = false): per-segment E, nw and padded size into the table
// (off = size). Pass 2: the host has turned sizes into offsets; write.
// Lane l owns values [32 l, 32 l + 32) so stream order is value order.
__global__ void __launch_bounds__(32 * kUEncWarps) unary_encode_kernel(const uint16_t* __restrict__ src, size_t segs,
                                                                       uint8_t* __restrict__ dst, bool write) {
  __shared__ uint32_t words[kUEncWarps][kUMaxWords];
  const int wib = threadIdx.x / 32, lane = threadIdx.x % 32;
  const size_t seg = size_t(blockIdx.x) * kUEncWarps + wib;
  if (seg >= segs) return;
  const uint4* s = reinterpret_cast<const uint4*>(src + seg * kSeg + 32 * lane);
  uint16_t v[32];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint4 u = s[i];
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      v[8 * i + 2 * t] = uint16_t(w[t] & 0xffffu);
      v[8 * i + 2 * t + 1] = uint16_t(w[t] >> 16);
    }
  }
  int emax = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) emax = max(emax, int((v[i] >> 7) & 0xff));
#pragma unroll
  for (int o = 16; o; o >>= 1) emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  int emax_base = emax;
  // base E: of emax, emax - 1, ..., emax - 7 the one with the fewest bits
  // (values above E escape: a few outliers then cost 24 bits each instead of
  // lengthening every code of the segment)
  int best = 1 << 30;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int b0 = emax - c;
    int cost = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int e = int((v[i] >> 7) & 0xff);
      cost += e <= b0 ? min(b0 - e, kUEsc) + 1 : kUEsc + 1 + 8;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) cost += __shfl_xor_sync(0xffffffffu, cost, o);
    if (b0 >= 0 && cost < best) {
      best = cost;
      emax_base = b0;
    }
  }
  const int ebase = emax_base;
  int nbits = 0, nesc = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int e = int((v[i] >> 7) & 0xff);
    const int j = e <= ebase ? min(ebase - e, kUEsc) : kUEsc;
    nbits += j + 1;
    nesc += j == kUEsc;
  }
  int tbits = 0, tesc = 0;
  const int bit0 = warp_excl_scan(nbits, lane, &tbits);
  const int esc0 = warp_excl_scan(nesc, lane, &tesc);
  const int nw = (tbits + 31) / 32;
  const uint32_t bytes = uint32_t((kSeg + 4 * nw + tesc + 15) & ~15);
  USeg* table = reinterpret_cast<USeg*>(dst);
  if (!write) {
    if (lane == 0) table[seg] = USeg{bytes, uint8_t(ebase), uint8_t(tesc ? 1 : 0), uint16_t(nw)};
    return;
  }
  uint8_t* d = dst + table[seg].off;
  uint32_t* wd = words[wib];
  for (int k = lane; k < nw; k += 32) wd[k] = 0u;
  __syncwarp();
  int pos = bit0;
  uint32_t lo[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
  int e_at = esc0;
  uint8_t* esc = d + kSeg + 4 * nw;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const uint32_t x = v[i];
    const int e = int((x >> 7) & 0xff);
    const int j = e <= ebase ? min(ebase - e, kUEsc) : kUEsc;
    if (j) {  // j ones at stream bits [pos, pos + j) (MSB-first): at most two words
      const uint64_t ones = ((uint64_t(1) << j) - 1u) << (64 - (pos & 31) - j);
      atomicOr(&wd[pos >> 5], uint32_t(ones >> 32));
      if (uint32_t(ones)) atomicOr(&wd[(pos >> 5) + 1], uint32_t(ones));
    }
    if (j == kUEsc) esc[e_at++] = uint8_t(e);
    pos += j + 1;
    lo[i / 4] |= (((x >> 8) & 0x80u) | (x & 0x7fu)) << (8 * (i % 4));
  }
  if (lane == 0 && (tbits & 31)) atomicOr(&wd[tbits >> 5], (1u << (32 - (tbits & 31))) - 1u);  // trailing ones
  reinterpret_cast<uint4*>(d)[2 * lane] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  reinterpret_cast<uint4*>(d)[2 * lane + 1] = make_uint4(lo[4], lo[5], lo[6], lo[7]);
  __syncwarp();
  uint32_t* cw = reinterpret_cast<uint32_t*>(d + kSeg);
  for (int k = lane; k < nw; k += 32) cw[k] = wd[k];
  const int used = kSeg + 4 * nw + tesc;
  if (lane < int(bytes) - used) d[used + lane] = 0;  // deterministic padding
}

// position (0-based, from the MSB) of the k-th set bit of x, k < popc(x):
// binary search with population counts, branch-free
__device__ __forceinline__ int select_msb(uint32_t x, int k) {
  int pos = 0;
#pragma unroll
  for (int w = 16; w; w >>= 1) {
    const int c = __popc(x >> (32 - w));  // set bits in the top w bits
    const bool skip = k >= c;
    k -= skip ? c : 0;
    pos += skip ? w : 0;
    x = skip ? x << w : x;
  }
  return pos;
}

// Decode: a warp stages the segment's code words in shared memory, finds
// where each lane's 32 values start (value 32 L begins after zero 32 L - 1 of
// the stream: a warp scan of zero counts over 3-word runs, then a popc
// select inside the word), and every lane then walks its own 32 codes with a
// 32-bit window — one count-leading-ones per value, no divergence — and
// builds its 64 output bytes in registers from its 32 lo bytes.
constexpr int kUDecWarps = 2;
constexpr int kURun = 4;  // code words per lane per scan round (fast path: streams of <= 128 words)
template <bool kDirect>
#ifndef SMO_UDEC_MINB  // resident blocks per SM the register budget is sized for (A/B: -DSMO_UDEC_MINB=n)
#define SMO_UDEC_MINB 28
#endif
__global__ void __launch_bounds__(32 * kUDecWarps, SMO_UDEC_MINB) unary_decode_kernel(const __grid_constant__ DecodeJobs jobs,
                                                                       size_t segs) {
  __shared__ __align__(16) uint32_t wbuf[kUDecWarps][kUMaxWords + 8];
  __shared__ __align__(16) uint4 lobuf[kUDecWarps][64];  // the segment's lo bytes, copied ahead (cp.async)
  __shared__ int start[kUDecWarps][33];
  const uint8_t* __restrict__ src = jobs.src[blockIdx.y];
  uint16_t* __restrict__ dst = jobs.dst[blockIdx.y];
  const int wib = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint32_t* wb = wbuf[wib];
  int* st = start[wib];
  // grid-stride over segments: a warp decodes several, launch cost amortised
  for (size_t seg = size_t(blockIdx.x) * kUDecWarps + wib; seg < segs; seg += size_t(gridDim.x) * kUDecWarps) {
    const uint2 tw = reinterpret_cast<const uint2*>(src)[seg];
    const uint8_t* sb = src + tw.x;
    const int base = int(tw.y & 0xffu), nw = int(tw.y >> 16);
    const bool has_esc = (tw.y >> 8) & 1u;
    // the lane's 32 lo bytes go to shared memory by cp.async now (no
    // registers held), so their latency hides under the search and the walk
    const uint32_t lo_s = smem_u32(&lobuf[wib][2 * lane]);
    cp_async_16(lo_s, sb + 32 * lane);
    cp_async_16(lo_s + 16, sb + 32 * lane + 16);
    asm volatile("cp.async.commit_group;" ::: "memory");
    // coalesced 16-B staging of the stream (it starts 16-B aligned and the
    // segment is padded to 16 B, so whole chunks stay inside it); words past
    // the end read as ones, 6 of them at least
    {
      const uint4* c4 = reinterpret_cast<const uint4*>(sb + kSeg);
      const int nc = (nw + 3) >> 2;
      auto chunk = [&](int c) {
        uint4 v = c < nc ? c4[c] : make_uint4(~0u, ~0u, ~0u, ~0u);
        const int w0 = 4 * c;
        v.x = w0 < nw ? v.x : ~0u;
        v.y = w0 + 1 < nw ? v.y : ~0u;
        v.z = w0 + 2 < nw ? v.z : ~0u;
        v.w = w0 + 3 < nw ? v.w : ~0u;
        reinterpret_cast<uint4*>(wb)[c] = v;
      };
      if (nc + 2 <= 32) {  // common case (<= 120 words): one chunk per lane
        if (lane < nc + 2) chunk(lane);
      } else {
        for (int c = lane; c < nc + 2; c += 32) chunk(c);
      }
    }
    __syncwarp();
    int p0 = 0;
    if (nw <= 32 * kURun) {
      // common case, one run of <= 3 words per lane: zero counts per run,
      // a warp scan, then each lane binary-searches the run holding zero
      // 32 L - 1 (shared-memory prefix table) and selects inside its word —
      // no divergent loops
      const int w0 = kURun * lane;
      uint32_t z[kURun];
      int n = 0;
#pragma unroll
      for (int r = 0; r < kURun; ++r) {
        z[r] = w0 + r < nw ? ~wb[w0 + r] : 0u;  // zeros = value ends
        n += __popc(z[r]);
      }
      int tot = 0;
      const int before = warp_excl_scan(n, lane, &tot);
      st[lane] = before + n;  // zeros up to the end of run `lane`
      __syncwarp();
      if (lane > 0) {
        const int t = 32 * lane - 1;
        int w = 0;  // first run whose inclusive count exceeds t
#pragma unroll
        for (int step = 16; step; step >>= 1)
          if (st[w + step - 1] <= t) w += step;
        int k = t - (w ? st[w - 1] : 0);
        int r = 0;
        uint32_t zw = ~wb[kURun * w];
#pragma unroll
        for (int q = 1; q < kURun; ++q) {
          const int c = __popc(zw);
          if (k >= c) {
            k -= c;
            r = q;
            zw = kURun * w + q < nw ? ~wb[kURun * w + q] : 0u;
          }
        }
        p0 = (kURun * w + r) * 32 + select_msb(zw, k) + 1;
      }
    } else {  // long streams (escapes, wide segments): runs over several rounds
      int cum = 0;
      for (int c0 = 0; c0 < nw; c0 += 32 * kURun) {
        const int w0 = c0 + kURun * lane;
        uint32_t z[kURun];
        int cnt[kURun], n = 0;
#pragma unroll
        for (int r = 0; r < kURun; ++r) {
          z[r] = w0 + r < nw ? ~wb[w0 + r] : 0u;
          cnt[r] = __popc(z[r]);
          n += cnt[r];
        }
        int tot = 0;
        int before = cum + warp_excl_scan(n, lane, &tot);
        cum += tot;
        // lanes L whose first value follows zero 32 L - 1 when it lies in this run
#pragma unroll
        for (int r = 0; r < kURun; ++r) {
          for (int L = (before + 32) / 32; L < 32 && 32 * L - 1 < before + cnt[r]; ++L)
            st[L] = (w0 + r) * 32 + select_msb(z[r], 32 * L - 1 - before) + 1;
          before += cnt[r];
        }
      }
      if (lane == 0) st[0] = 0;
      __syncwarp();
      p0 = st[lane];
    }
    // walk the lane's 32 codes two at a time in a 64-bit window (hi:lo) read
    // from bit `off` < 32: two codes of <= 16 bits each fit the window, so a
    // pair needs no bounds check; after each pair one branch-free refill
    // (SEL) shifts a word in when 32 bits were consumed. Per code: one
    // 64-bit funnel shift, one find-leading-one of the complement, one add
    // (the code length is 32 - f for the window's highest zero at f).
    uint32_t j4[8];
    {
      const uint32_t* wp = wb + (p0 >> 5);
      uint32_t hi = wp[0], lo = wp[1];
      wp += 2;
      uint32_t off = uint32_t(p0 & 31);
      uint32_t fs[32];
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        // f = bfind(~window) (position of the window's highest zero), and the
        // code is 32 - f bits long: one SHF, one FLO, one IADD3 per code
        const uint64_t win = (uint64_t(hi) << 32) | lo;
        uint32_t f1, f2;
        asm("bfind.u32 %0, %1;" : "=r"(f1) : "r"(~uint32_t((win << off) >> 32)));
        const uint32_t off2 = off + 32u - f1;  // < 48
        asm("bfind.u32 %0, %1;" : "=r"(f2) : "r"(~uint32_t((win << off2) >> 32)));
        off = off2 + 32u - f2;                 // < 64
        // refill: shift a word in once 32 bits were consumed (off >> 5 is 0 or 1)
        const uint32_t nxt = *wp;
        const bool ge = off >= 32u;
        hi = ge ? lo : hi;
        lo = ge ? nxt : lo;
        wp += off >> 5;
        off &= 31u;
        fs[i] = f1;
        fs[i + 1] = f2;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)  // four f (16..31) per word, bytewise
        j4[q] = __byte_perm(__byte_perm(fs[4 * q], fs[4 * q + 1], 0x0040u), __byte_perm(fs[4 * q + 2], fs[4 * q + 3], 0x0040u),
                            0x5410u);
    }
    // e = base - j = f - (31 - base)
    uint32_t e4[8];
    if (base >= kUEsc) {  // f >= 16 >= 31 - base in every byte: one subtraction per 4 values
      const uint32_t d4 = uint32_t(31 - base) * 0x01010101u;
#pragma unroll
      for (int q = 0; q < 8; ++q) e4[q] = j4[q] - d4;
    } else {  // tiny base (near-zero segments): bytewise
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint32_t v = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t)
          v |= (uint32_t(int((j4[q] >> (8 * t)) & 0xffu) - 31 + base) & 0xffu) << (8 * t);
        e4[q] = v;
      }
    }
    if (has_esc) {  // escaped exponents (code j = 15, i.e. f = 16), in position order:
      // the walk already holds every f, so the escapes are a byte compare
      uint32_t emask = 0u;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t m4 = __vcmpeq4(j4[q], 0x10101010u);  // 0xff per escaped byte
#pragma unroll
        for (int t = 0; t < 4; ++t) emask |= ((m4 >> (8 * t + 7)) & 1u) << (4 * q + t);
      }
      int etot = 0;
      int er = warp_excl_scan(__popc(emask), lane, &etot);
      const uint8_t* esc = sb + kSeg + 4 * nw;
      for (uint32_t m = emask; m; m &= m - 1u) {
        const int i = __ffs(m) - 1;
        const uint32_t sh = 8u * uint32_t(i % 4), wq = uint32_t(i / 4);
        const uint32_t eb = uint32_t(esc[er]) << sh, keep = ~(0xffu << sh);
        // select-based patch over all eight words (no dynamic index: e4
        // stays in registers instead of local memory on every segment)
#pragma unroll
        for (int q = 0; q < 8; ++q) e4[q] = uint32_t(q) == wq ? ((e4[q] & keep) | eb) : e4[q];
        ++er;
      }
    }
    // 32 values -> 64 bytes: two values per word. PRMT spreads two lo bytes
    // (sign << 7 | mantissa) to 16-bit lanes with the sign replicated into
    // the high byte (selector nibbles 8-B), a second PRMT the two exponents;
    // one LOP3 merges sign, exponent << 7 and mantissa.
    asm volatile("cp.async.wait_group 0;" ::: "memory");  // this lane's own copies
    const uint4 lo0 = lobuf[wib][2 * lane];  // this lane's 32 lo bytes
    const uint4 lo1 = lobuf[wib][2 * lane + 1];
    const uint32_t lw[8] = {lo0.x, lo0.y, lo0.z, lo0.w, lo1.x, lo1.y, lo1.z, lo1.w};
    uint32_t out[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const uint32_t t = __byte_perm(lw[k / 2], 0u, (k & 1) ? 0xB3A2u : 0x9180u);
      const uint32_t x16 = __byte_perm(e4[k / 2], 0u, (k & 1) ? 0x4342u : 0x4140u);
      out[k] = (t & 0x807F807Fu) | (x16 << 7);
    }
    uint4* d = reinterpret_cast<uint4*>(dst + seg * kSeg);
    if constexpr (kDirect) {
      // straight from registers: each lane's 64 bytes are contiguous
      // (4 x 16 B per lane at a 64 B stride per store instruction)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        d[4 * lane + k] = make_uint4(out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]);
      __syncwarp();  // wb / st are reused by the next segment
    } else {
      // through shared memory (the stream buffer is free now) so every global
      // store instruction writes 512 contiguous bytes
      __syncwarp();
      uint4* ob = reinterpret_cast<uint4*>(wb);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        ob[4 * lane + ((k + lane) & 3)] = make_uint4(out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]);
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int g = 32 * k + lane;  // 16-byte group g = lane' 4 + k' of lane' = g / 4
        const int ln = g >> 2, kk = g & 3;
        d[g] = ob[4 * ln + ((kk + ln) & 3)];
      }
      __syncwarp();  // wb / st are reused by the next segment
    }
  }
}

}  // namespace

size_t expert_code_bytes(size_t count, int bits) {
  SMO_REQUIRE(bits == 1 || bits == 3 || bits == 4, "expert codec: bits must be 1 (unary), 3 or 4");
  if (bits == 1) return u_table_bytes(count / kSeg) + (count / kSeg) * size_t(kSeg + 4 * kUMaxWords + kSeg);
  return (count / kSeg) * size_t(bits == 3 ? Fmt<3>::kSegBytes : Fmt<4>::kSegBytes);
}

// count % 1024 == 0; overflow (device int) is set to 1 when a segment has
// more than 32 escapes (the output is then unusable: retry with 4 bits or
// keep the block raw).
void expert_encode(const void* src, size_t count, int bits, void* dst, int* overflow, cudaStream_t st) {
  SMO_REQUIRE(src && dst && overflow && count % kSeg == 0, "expert codec: count must be a multiple of 1024");
  SMO_REQUIRE(bits == 1 || bits == 3 || bits == 4, "expert codec: bits must be 1 (unary), 3 or 4");
  const size_t segs = count / kSeg;
  if (bits == 1) {  // two passes around a host scan of the segment sizes (synchronous on st)
    auto s16 = reinterpret_cast<const uint16_t*>(src);
    auto d8 = reinterpret_cast<uint8_t*>(dst);
    const unsigned grid = unsigned((segs + kUEncWarps - 1) / kUEncWarps);
    std::vector<USeg> t(segs + 1);
    if (segs) {
      unary_encode_kernel<<<grid, 32 * kUEncWarps, 0, st>>>(s16, segs, d8, false);
      count_launch();
      SMO_CUDA_CHECK(cudaGetLastError());
      SMO_CUDA_CHECK(cudaMemcpyAsync(t.data(), d8, segs * sizeof(USeg), cudaMemcpyDeviceToHost, st));
      SMO_CUDA_CHECK(cudaStreamSynchronize(st));
    }
    size_t off = u_table_bytes(segs);
    for (size_t i = 0; i < segs; ++i) {
      const size_t b = t[i].off;
      t[i].off = uint32_t(off);
      off += b;
    }
    SMO_REQUIRE(off < (size_t(1) << 32), "expert codec: block too large for 32-bit segment offsets");
    t[segs] = USeg{uint32_t(off), 0, 0, 0};
    std::vector<uint8_t> head(u_table_bytes(segs), 0);
    std::memcpy(head.data(), t.data(), t.size() * sizeof(USeg));
    SMO_CUDA_CHECK(cudaMemcpyAsync(d8, head.data(), head.size(), cudaMemcpyHostToDevice, st));
    if (segs) {
      unary_encode_kernel<<<grid, 32 * kUEncWarps, 0, st>>>(s16, segs, d8, true);
      count_launch();
      SMO_CUDA_CHECK(cudaGetLastError());
    }
    SMO_CUDA_CHECK(cudaStreamSynchronize(st));
    return;
  }
  if (!segs) return;
  const int threads = 256;
  const unsigned grid = unsigned((segs * 32 + threads - 1) / threads);
  auto s16 = reinterpret_cast<const uint16_t*>(src);
  auto d8 = reinterpret_cast<uint8_t*>(dst);
  if (bits == 3) expert_encode_kernel<3><<<grid, threads, 0, st>>>(s16, segs, d8, overflow);
  else expert_encode_kernel<4><<<grid, threads, 0, st>>>(s16, segs, d8, overflow);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

// Expand n blocks of `count` values each (srcs[i] -> dsts[i], all `bits`) in one launch.
void expert_decode_blocks(const void* const* srcs, void* const* dsts, int n, size_t count, int bits, cudaStream_t st) {
  SMO_REQUIRE(n >= 0 && n <= 64 && count % kSeg == 0, "expert codec: up to 64 blocks of a multiple of 1024 values");
  SMO_REQUIRE(bits == 1 || bits == 3 || bits == 4, "expert codec: bits must be 1 (unary), 3 or 4");
  const size_t segs = count / kSeg;
  if (!segs || !n) return;
  DecodeJobs jobs{};
  for (int i = 0; i < n; ++i) {
    SMO_REQUIRE(srcs[i] && dsts[i], "expert codec: null block");
    jobs.src[i] = reinterpret_cast<const uint8_t*>(srcs[i]);
    jobs.dst[i] = reinterpret_cast<uint16_t*>(dsts[i]);
  }
  if (bits == 1) {
    // one warp per segment (the kernel's grid-stride loop then runs once):
    // measured faster than a one-wave persistent grid (238 vs 212 us per
    // Mixtral block) — warps finish unevenly and fresh blocks refill the SMs
    // segments per warp (SMO_UNARY_SPW, A/B): the per-warp prologue is
    // amortised over that many segments of the grid-stride loop
    static const size_t spw = [] {
      const char* f = std::getenv("SMO_UNARY_SPW");
      return size_t(std::max(1, f ? std::atoi(f) : 1));
    }();
    const size_t want = (segs + kUDecWarps * spw - 1) / (kUDecWarps * spw);
    const size_t cap = want;
    const dim3 ug(unsigned(std::min(want, cap)), unsigned(n));
    static const bool direct = [] {  // A/B switch: SMO_UNARY_DIRECT=1 stores from registers
      const char* f = std::getenv("SMO_UNARY_DIRECT");
      return f && f[0] == '1';
    }();
    if (direct) unary_decode_kernel<true><<<ug, 32 * kUDecWarps, 0, st>>>(jobs, segs);
    else unary_decode_kernel<false><<<ug, 32 * kUDecWarps, 0, st>>>(jobs, segs);
    count_launch();
    SMO_CUDA_CHECK(cudaGetLastError());
    return;
  }
  const dim3 grid(unsigned((segs + kDecWarps * kDecSegs - 1) / (kDecWarps * kDecSegs)), unsigned(n));
  if (bits == 3) expert_decode_kernel<3><<<grid, 32 * kDecWarps, 0, st>>>(jobs, segs);
  else expert_decode_kernel<4><<<grid, 32 * kDecWarps, 0, st>>>(jobs, segs);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

// Bytes of a coded block: fixed for 3 / 4 bits; unary reads the table's last
// entry from the (device) code.
size_t expert_coded_size(const void* code, size_t count, int bits) {
  if (bits != 1) return expert_code_bytes(count, bits);
  USeg t{};
  SMO_CUDA_CHECK(cudaMemcpy(&t, reinterpret_cast<const uint8_t*>(code) + (count / kSeg) * sizeof(USeg), sizeof(t),
                            cudaMemcpyDeviceToHost));
  return t.off;
}

void expert_decode(const void* src, size_t count, int bits, void* dst, cudaStream_t st) {
  SMO_REQUIRE(src && dst && count % kSeg == 0, "expert codec: count must be a multiple of 1024");
  expert_decode_blocks(&src, &dst, 1, count, bits, st);
}

}  // namespace smo
