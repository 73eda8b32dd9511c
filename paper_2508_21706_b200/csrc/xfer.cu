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

}  // namespace

size_t expert_code_bytes(size_t count, int bits) {
  SMO_REQUIRE(bits == 3 || bits == 4, "expert codec: bits must be 3 or 4");
  return (count / kSeg) * size_t(bits == 3 ? Fmt<3>::kSegBytes : Fmt<4>::kSegBytes);
}

// count % 1024 == 0; overflow (device int) is set to 1 when a segment has
// more than 32 escapes (the output is then unusable: retry with 4 bits or
// keep the block raw).
void expert_encode(const void* src, size_t count, int bits, void* dst, int* overflow, cudaStream_t st) {
  SMO_REQUIRE(src && dst && overflow && count % kSeg == 0, "expert codec: count must be a multiple of 1024");
  SMO_REQUIRE(bits == 3 || bits == 4, "expert codec: bits must be 3 or 4");
  const size_t segs = count / kSeg;
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
  SMO_REQUIRE(bits == 3 || bits == 4, "expert codec: bits must be 3 or 4");
  const size_t segs = count / kSeg;
  if (!segs || !n) return;
  DecodeJobs jobs{};
  for (int i = 0; i < n; ++i) {
    SMO_REQUIRE(srcs[i] && dsts[i], "expert codec: null block");
    jobs.src[i] = reinterpret_cast<const uint8_t*>(srcs[i]);
    jobs.dst[i] = reinterpret_cast<uint16_t*>(dsts[i]);
  }
  const dim3 grid(unsigned((segs + kDecWarps * kDecSegs - 1) / (kDecWarps * kDecSegs)), unsigned(n));
  if (bits == 3) expert_decode_kernel<3><<<grid, 32 * kDecWarps, 0, st>>>(jobs, segs);
  else expert_decode_kernel<4><<<grid, 32 * kDecWarps, 0, st>>>(jobs, segs);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void expert_decode(const void* src, size_t count, int bits, void* dst, cudaStream_t st) {
  SMO_REQUIRE(src && dst && count % kSeg == 0, "expert codec: count must be a multiple of 1024");
  expert_decode_blocks(&src, &dst, 1, count, bits, st);
}

}  // namespace smo
