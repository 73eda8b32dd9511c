// tcode.cu — K5 tile code "T2" (format: tcode.cuh): the GPU encoder of an
// expert block and a standalone decoder to bf16 (tests, bf16 expansions).
// The production decoder is tcode::decode_segment inside the fused expert
// kernel (moe_tc.cu), which never writes the bf16 weights to HBM.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "tcode.cuh"

namespace smo {

namespace {

using namespace tcode;

// the matrices of one expert block, tiles numbered matrix-major
struct TMats {
  const uint16_t* src[3];
  int R[3], C[3];
  int t0[4];  // first tile of each matrix; t0[3] = tiles
};

TMats expert_mats(const void* src, int h, int hi) {
  TMats m{};
  const size_t n = size_t(h) * hi;
  for (int i = 0; i < 3; ++i) {
    m.src[i] = src ? reinterpret_cast<const uint16_t*>(src) + i * n : nullptr;
    m.R[i] = i < 2 ? hi : h;
    m.C[i] = i < 2 ? h : hi;
  }
  const int per = int(n / (kTileRows * kTileCols));
  for (int i = 0; i <= 3; ++i) m.t0[i] = i * per;
  return m;
}

struct TileAt {
  int m, nb, kb;
};
__device__ __forceinline__ TileAt tile_at(const TMats& M, int t) {
  const int m = t >= M.t0[2] ? 2 : t >= M.t0[1] ? 1 : 0;
  const int tl = t - M.t0[m];
  const int kbs = M.C[m] / kTileCols;
  return TileAt{m, tl / kbs, tl % kbs};
}

// code class of an exponent offset j: 0 level 1 (j <= 2), 1 level 2
// (3..5), 2 nibble (6..20), 3 literal; bits 2, 4, 8, 16
__device__ __forceinline__ int class_of(int j) {
  return (j >= 0 && j <= 2) ? 0 : (j >= 3 && j <= 5) ? 1 : (j >= 6 && j <= 20) ? 2 : 3;
}

constexpr int kEncWarps = 8;

// Pass 1 (write = false): per segment E | flags << 8 | (stream bytes / 4)
// << 12 into meta[]. The host then turns stream sizes into offsets (and
// marks incompressible tiles raw) and rewrites meta[] with the final header
// words. Pass 2 writes the tiles. One warp per segment, lane L owns values
// 32 L .. 32 L + 31 (row L / 2 of the segment, half L % 2).
__global__ void __launch_bounds__(32 * kEncWarps) tcode_encode_kernel(const __grid_constant__ TMats M, int segs,
                                                                      uint32_t* __restrict__ meta,
                                                                      uint8_t* __restrict__ dst, bool write) {
  __shared__ uint32_t fw[kEncWarps][64 + 128];  // L2 (<= 1024 x 2 bits) and L3 (<= 1024 x 4 bits) words
  const int wib = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int g = blockIdx.x * kEncWarps + wib;
  if (g >= segs) return;
  const int t = g / kSegs, s = g % kSegs;
  const TileAt ta = tile_at(M, t);
  const int C = M.C[ta.m];
  const int row = ta.nb * kTileRows + s * kSegRows + (lane >> 1);
  const int col = ta.kb * kTileCols + 32 * (lane & 1);
  const uint4* sp = reinterpret_cast<const uint4*>(M.src[ta.m] + size_t(row) * C + col);
  uint32_t v2[16];  // two values per word, value 2k in the low half
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint4 u = sp[i];
    v2[4 * i] = u.x;
    v2[4 * i + 1] = u.y;
    v2[4 * i + 2] = u.z;
    v2[4 * i + 3] = u.w;
  }
  auto val = [&](int i) -> uint32_t { return (v2[i >> 1] >> (16 * (i & 1))) & 0xffffu; };
  auto expo = [&](int i) -> int { return int((val(i) >> 7) & 0xffu); };
  if (!write) {
    int emax = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) emax = max(emax, expo(i));
#pragma unroll
    for (int o = 16; o; o >>= 1) emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    int E = max(emax, 6), best = -1;
    for (int c = 0; c < 8; ++c) {
      const int b0 = emax - c;
      if (b0 < 6) break;  // warp-uniform (E >= 6: no borrow in the decoder's E - c1 - c2)
      int cost = 0;
#pragma unroll
      for (int i = 0; i < 32; ++i) cost += 2 << class_of(b0 - expo(i));
#pragma unroll
      for (int o = 16; o; o >>= 1) cost += __shfl_xor_sync(0xffffffffu, cost, o);
      if (best < 0 || cost < best) {
        best = cost;
        E = b0;
      }
    }
    int n2 = 0, n3 = 0, nl = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int k = class_of(E - expo(i));
      n2 += k >= 1;
      n3 += k >= 2;
      nl += k == 3;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      n2 += __shfl_xor_sync(0xffffffffu, n2, o);
      n3 += __shfl_xor_sync(0xffffffffu, n3, o);
      nl += __shfl_xor_sync(0xffffffffu, nl, o);
    }
    const uint32_t words = uint32_t((n2 + 15) / 16 + (n3 + 7) / 8 + (nl + 3) / 4);
    const uint32_t flags = (n2 ? 2u : 0u) | (n3 ? 4u : 0u) | (nl ? 8u : 0u);
    if (lane == 0) meta[g] = uint32_t(E) | (flags << 8) | (words << 12);
    return;
  }
  const uint32_t hw = meta[g];
  uint8_t* tb = dst + reinterpret_cast<const uint32_t*>(dst)[t];
  if (hw & 0x100u) {  // raw tile: the header, then the segment's 16 rows verbatim
    uint4* d = reinterpret_cast<uint4*>(tb + 32 + 2 * kSeg * s) + 4 * lane;
#pragma unroll
    for (int i = 0; i < 4; ++i) d[i] = make_uint4(v2[4 * i], v2[4 * i + 1], v2[4 * i + 2], v2[4 * i + 3]);
    if (lane == 0) reinterpret_cast<uint32_t*>(tb)[s] = s == 0 ? 0x100u : 0u;
    return;
  }
  if (lane == 0) reinterpret_cast<uint32_t*>(tb)[s] = hw;
  const int E = int(hw & 0xffu);
  uint32_t lo[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u}, l1[2] = {0u, 0u};
  int n2 = 0, n3 = 0, nl = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const uint32_t x = val(i);
    lo[i >> 2] |= (((x >> 8) & 0x80u) | (x & 0x7fu)) << (8 * (i & 3));
    const int j = E - expo(i);
    const int k = class_of(j);
    const uint32_t c1 = k ? 3u : uint32_t(j);
    const int ii = i & 15;
    l1[i >> 4] |= c1 << (2 * (ii >> 1) + 16 * (ii & 1));
    n2 += k >= 1;
    n3 += k >= 2;
    nl += k == 3;
  }
  reinterpret_cast<uint4*>(tb + kLoOff + kSeg * s)[2 * lane] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  reinterpret_cast<uint4*>(tb + kLoOff + kSeg * s)[2 * lane + 1] = make_uint4(lo[4], lo[5], lo[6], lo[7]);
  reinterpret_cast<uint2*>(tb + kL1Off + 256 * s)[lane] = make_uint2(l1[0], l1[1]);
  uint32_t* w2 = fw[wib];
  uint32_t* w3 = fw[wib] + 64;
  for (int k = lane; k < 64 + 128; k += 32) fw[wib][k] = 0u;
  __syncwarp();
  int t2 = 0, t3 = 0, tl = 0;
  int f2 = warp_excl_scan(n2, lane, &t2), f3 = warp_excl_scan(n3, lane, &t3), fl = warp_excl_scan(nl, lane, &tl);
  uint8_t* stp = tb + 4 * (hw >> 12);
  const int nw2 = (t2 + 15) / 16, nw3 = (t3 + 7) / 8;
  uint8_t* lit = stp + 4 * (nw2 + nw3);
  for (int i = 0; i < 32; ++i) {
    const int e = expo(i);
    const int j = E - e;
    const int k = class_of(j);
    if (k >= 1) {
      atomicOr(&w2[f2 >> 4], (k == 1 ? uint32_t(j - 3) : 3u) << (2 * (f2 & 15)));
      ++f2;
    }
    if (k >= 2) {
      atomicOr(&w3[f3 >> 3], (k == 2 ? uint32_t(j - 6) : 15u) << (4 * (f3 & 7)));
      ++f3;
    }
    if (k == 3) lit[fl++] = uint8_t(e);
  }
  __syncwarp();
  uint32_t* sw = reinterpret_cast<uint32_t*>(stp);
  for (int k = lane; k < nw2; k += 32) sw[k] = w2[k];
  for (int k = lane; k < nw3; k += 32) sw[nw2 + k] = w3[k];
  const int lpad = ((tl + 3) & ~3) - tl;
  if (lane < lpad) lit[tl + lane] = 0;
  if (s == kSegs - 1) {  // tile padding to 16 bytes
    const uint8_t* end = lit + tl + lpad;
    const uint8_t* tend = dst + reinterpret_cast<const uint32_t*>(dst)[t + 1];
    if (lane < int(tend - end)) const_cast<uint8_t*>(end)[lane] = 0;
  }
}

// T3 encoder (format: tcode.cuh / tests/tcode3_ref.py), the same two passes:
// pass 1 writes E | nesc << 9 per segment (0xffffffff: the segment forces a
// raw tile — its maximum exponent is below 7 or it has > 1023 escapes), the
// host lays out the escape lists and raw tiles, pass 2 writes the tiles.
__global__ void __launch_bounds__(32 * kEncWarps) tcode3_encode_kernel(const __grid_constant__ TMats M, int segs,
                                                                       uint32_t* __restrict__ meta,
                                                                       uint8_t* __restrict__ dst, bool write) {
  const int wib = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int g = blockIdx.x * kEncWarps + wib;
  if (g >= segs) return;
  const int t = g / kSegs, s = g % kSegs;
  const TileAt ta = tile_at(M, t);
  const int C = M.C[ta.m];
  const int row = ta.nb * kTileRows + s * kSegRows + (lane >> 1);
  const int col = ta.kb * kTileCols + 32 * (lane & 1);
  const uint4* sp = reinterpret_cast<const uint4*>(M.src[ta.m] + size_t(row) * C + col);
  uint32_t v2[16];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint4 u = sp[i];
    v2[4 * i] = u.x;
    v2[4 * i + 1] = u.y;
    v2[4 * i + 2] = u.z;
    v2[4 * i + 3] = u.w;
  }
  auto val = [&](int i) -> uint32_t { return (v2[i >> 1] >> (16 * (i & 1))) & 0xffffu; };
  auto expo = [&](int i) -> int { return int((val(i) >> 7) & 0xffu); };
  if (!write) {
    int emax = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) emax = max(emax, expo(i));
#pragma unroll
    for (int o = 16; o; o >>= 1) emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    int E = -1, best = -1;
    for (int c = 0; c < 8; ++c) {
      const int b0 = emax - c;
      if (b0 < 7) break;  // warp-uniform
      int n = 0;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int j = b0 - expo(i);
        n += (j < 0 || j > 6) ? 1 : 0;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
      if (best < 0 || n < best) {
        best = n;
        E = b0;
      }
    }
    if (lane == 0) meta[g] = (E < 0 || best > 1023) ? 0xffffffffu : (uint32_t(E) | (uint32_t(best) << 9));
    return;
  }
  const uint32_t hw = meta[g];
  uint8_t* tb = dst + reinterpret_cast<const uint32_t*>(dst)[t];
  if (hw & 0x100u) {  // raw tile
    uint4* d = reinterpret_cast<uint4*>(tb + 32 + 2 * kSeg * s) + 4 * lane;
#pragma unroll
    for (int i = 0; i < 4; ++i) d[i] = make_uint4(v2[4 * i], v2[4 * i + 1], v2[4 * i + 2], v2[4 * i + 3]);
    if (lane == 0) reinterpret_cast<uint32_t*>(tb)[s] = s == 0 ? 0x100u : 0u;
    return;
  }
  if (lane == 0) reinterpret_cast<uint32_t*>(tb)[s] = hw;
  const int E = int(hw & 0xffu), nesc = int((hw >> 9) & 0x7ffu);
  uint32_t lo[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u}, w[3] = {0u, 0u, 0u};
  int ne = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const uint32_t x = val(i);
    lo[i >> 2] |= (((x >> 8) & 0x80u) | (x & 0x7fu)) << (8 * (i & 3));
    const int j = E - expo(i);
    const bool esc = j < 0 || j > 6;
    const uint32_t c = esc ? 7u : uint32_t(j);
    ne += esc ? 1 : 0;
    const int k = i >> 1, odd = i & 1;
    if (k < 15) {
      w[k / 5] |= c << (3 * (k % 5) + 16 * odd);
    } else {
#pragma unroll
      for (int b = 0; b < 3; ++b) w[b] |= ((c >> b) & 1u) << (15 + 16 * odd);
    }
  }
  reinterpret_cast<uint4*>(tb + kLoOff + kSeg * s)[2 * lane] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  reinterpret_cast<uint4*>(tb + kLoOff + kSeg * s)[2 * lane + 1] = make_uint4(lo[4], lo[5], lo[6], lo[7]);
  uint32_t* cwp = reinterpret_cast<uint32_t*>(tb + kC3Off + 384 * s) + 3 * lane;
  cwp[0] = w[0];
  cwp[1] = w[1];
  cwp[2] = w[2];
  // escape list: this lane's escapes at its rank, in value order
  int tot = 0;
  int f = warp_excl_scan(ne, lane, &tot);
  uint8_t* el = tb + 4 * (hw >> 20);
  for (int i = 0; i < 32; ++i) {
    const int j = E - expo(i);
    if (j < 0 || j > 6) {
      reinterpret_cast<uint16_t*>(el)[f] = uint16_t(32 * lane + i);
      el[2 * nesc + f] = uint8_t(expo(i));
      ++f;
    }
  }
  const int used = 3 * nesc, pad = ((used + 3) & ~3) - used;
  if (lane < pad) el[used + lane] = 0;
  if (s == kSegs - 1) {  // tile padding to 16 bytes
    const uint8_t* end = el + used + pad;
    const uint8_t* tend = dst + reinterpret_cast<const uint32_t*>(dst)[t + 1];
    if (lane < int(tend - end)) const_cast<uint8_t*>(end)[lane] = 0;
  }
}

// One CTA per tile: stage the tile code in shared memory, eight warps decode
// one segment each into a swizzled tile (the expert kernel's decoder), then
// the tile is written back row-major.
template <int kFmt>
__global__ void __launch_bounds__(256) tcode_decode_kernel(const __grid_constant__ TMats M,
                                                           const uint8_t* const* __restrict__ srcs,
                                                           uint16_t* const* __restrict__ dsts) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* tile = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* code = tile + kTileRows * 128;
  const uint8_t* src = srcs[blockIdx.y];
  const int t = blockIdx.x;
  const uint32_t* toff = reinterpret_cast<const uint32_t*>(src);
  const uint32_t o0 = toff[t], o1 = toff[t + 1];
  const uint4* g = reinterpret_cast<const uint4*>(src + o0);
  for (uint32_t i = threadIdx.x; i < (o1 - o0) / 16; i += blockDim.x) reinterpret_cast<uint4*>(code)[i] = g[i];
  __syncthreads();
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  if constexpr (kFmt == 3) decode_segment3(code, tile, w, lane);
  else decode_segment(code, tile, w, lane);
  __syncthreads();
  const TileAt ta = tile_at(M, t);
  const int C = M.C[ta.m];
  uint16_t* dst = dsts[blockIdx.y] + size_t(ta.m) * M.R[0] * M.C[0];
  for (int i = threadIdx.x; i < kTileRows * 8; i += blockDim.x) {
    const int r = i >> 3, c = i & 7;
    const uint4 v = *reinterpret_cast<const uint4*>(tile + r * 128 + ((c ^ (r & 7)) << 4));
    *reinterpret_cast<uint4*>(dst + size_t(ta.nb * kTileRows + r) * C + ta.kb * kTileCols + 8 * c) = v;
  }
}

}  // namespace

size_t tcode_max_bytes(int h, int hi) {
  const size_t nt = size_t(3) * h * hi / (kTileRows * kTileCols);
  return ((4 * (nt + 1) + 15) & ~size_t(15)) + nt * size_t(kTileMax);
}

// [W1 | W3 | W2] (bf16, device) -> T2 (fmt 2) or T3 (fmt 3) code at dst
// (device, >= tcode_max_bytes). Synchronous on st (host scan of the tile
// sizes between the passes); returns the code bytes.
size_t tcode_encode(const void* src, int h, int hi, void* dst, cudaStream_t st, int fmt) {
  SMO_REQUIRE(fmt == 2 || fmt == 3, "tcode: format must be 2 (T2) or 3 (T3)");
  SMO_REQUIRE(src && dst, "tcode: null pointer");
  SMO_REQUIRE(h % kTileRows == 0 && hi % kTileRows == 0 && h > 0 && hi > 0, "tcode: h and h_i must be multiples of 128");
  const TMats M = expert_mats(src, h, hi);
  const int nt = M.t0[3], segs = nt * kSegs;
  uint32_t* meta = nullptr;
  SMO_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&meta), size_t(segs) * 4, st));
  auto d8 = reinterpret_cast<uint8_t*>(dst);
  const unsigned grid = unsigned((segs + kEncWarps - 1) / kEncWarps);
  auto pass = [&](bool write) {
    if (fmt == 3) tcode3_encode_kernel<<<grid, 32 * kEncWarps, 0, st>>>(M, segs, meta, d8, write);
    else tcode_encode_kernel<<<grid, 32 * kEncWarps, 0, st>>>(M, segs, meta, d8, write);
    count_launch();
    SMO_CUDA_CHECK(cudaGetLastError());
  };
  pass(false);
  std::vector<uint32_t> hm(static_cast<size_t>(segs));
  SMO_CUDA_CHECK(cudaMemcpyAsync(hm.data(), meta, hm.size() * 4, cudaMemcpyDeviceToHost, st));
  SMO_CUDA_CHECK(cudaStreamSynchronize(st));
  const size_t tb = (4 * (size_t(nt) + 1) + 15) & ~size_t(15);
  std::vector<uint32_t> head(tb / 4, 0u);
  size_t off = tb;
  for (int t = 0; t < nt; ++t) {
    head[size_t(t)] = uint32_t(off);
    uint32_t* mt = hm.data() + size_t(t) * kSegs;
    if (fmt == 3) {  // escape lists after the codes; raw if a segment asks or nothing is saved
      bool raw = false;
      size_t sz = kEsc3Off;
      for (int s = 0; s < kSegs; ++s) {
        if (mt[s] == 0xffffffffu) raw = true;
        else sz += (3 * size_t((mt[s] >> 9) & 0x7ffu) + 3) & ~size_t(3);
      }
      const size_t end = sz;
      sz = (sz + 15) & ~size_t(15);
      if (raw || sz >= size_t(kTileMax) || end / 4 >= 4096) {
        for (int s = 0; s < kSegs; ++s) mt[s] = 0x100u;
        sz = kTileMax;
      } else {
        uint32_t eo = kEsc3Off;
        for (int s = 0; s < kSegs; ++s) {
          const uint32_t n = (mt[s] >> 9) & 0x7ffu;
          mt[s] = (mt[s] & 0xfffffu) | ((eo / 4) << 20);
          eo += (3 * n + 3) & ~3u;
        }
      }
      off += sz;
      continue;
    }
    size_t sz = kStreamOff;
    for (int s = 0; s < kSegs; ++s) sz += 4 * size_t(mt[s] >> 12);
    sz = (sz + 15) & ~size_t(15);
    if (sz >= size_t(kTileMax)) {  // incompressible: the whole tile raw
      for (int s = 0; s < kSegs; ++s) mt[s] = 0x100u;
      sz = kTileMax;
    } else {
      uint32_t so = kStreamOff / 4;
      for (int s = 0; s < kSegs; ++s) {
        const uint32_t words = mt[s] >> 12;
        mt[s] = (mt[s] & 0xfffu) | (so << 12);
        so += words;
      }
    }
    off += sz;
  }
  SMO_REQUIRE(off < (size_t(1) << 32), "tcode: block too large for 32-bit tile offsets");
  head[size_t(nt)] = uint32_t(off);
  SMO_CUDA_CHECK(cudaMemcpyAsync(d8, head.data(), tb, cudaMemcpyHostToDevice, st));
  SMO_CUDA_CHECK(cudaMemcpyAsync(meta, hm.data(), hm.size() * 4, cudaMemcpyHostToDevice, st));
  pass(true);
  SMO_CUDA_CHECK(cudaFreeAsync(meta, st));
  SMO_CUDA_CHECK(cudaStreamSynchronize(st));
  return off;
}

// Code bytes of a T2 block (reads toff[nt] from the device code).
size_t tcode_size(const void* code, int h, int hi) {
  const size_t nt = size_t(3) * h * hi / (kTileRows * kTileCols);
  uint32_t v = 0;
  SMO_CUDA_CHECK(cudaMemcpy(&v, reinterpret_cast<const uint8_t*>(code) + 4 * nt, 4, cudaMemcpyDeviceToHost));
  return v;
}

// n T2 / T3 blocks -> bf16 [W1 | W3 | W2] blocks, one launch.
void tcode_decode(const void* const* srcs, void* const* dsts, int n, int h, int hi, cudaStream_t st, int fmt) {
  SMO_REQUIRE(fmt == 2 || fmt == 3, "tcode: format must be 2 (T2) or 3 (T3)");
  SMO_REQUIRE(n >= 0 && n <= 64, "tcode: up to 64 blocks per launch");
  SMO_REQUIRE(h % kTileRows == 0 && hi % kTileRows == 0 && h > 0 && hi > 0, "tcode: h and h_i must be multiples of 128");
  if (!n) return;
  const TMats M = expert_mats(nullptr, h, hi);
  // pointer tables in device memory (stream-ordered scratch)
  void** tab = nullptr;
  SMO_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&tab), size_t(2 * n) * sizeof(void*), st));
  std::vector<const void*> ht(size_t(2 * n));
  for (int i = 0; i < n; ++i) {
    SMO_REQUIRE(srcs[i] && dsts[i], "tcode: null block");
    ht[size_t(i)] = srcs[i];
    ht[size_t(n + i)] = dsts[i];
  }
  SMO_CUDA_CHECK(cudaMemcpyAsync(tab, ht.data(), ht.size() * sizeof(void*), cudaMemcpyHostToDevice, st));
  const size_t smem = 1024 + kTileRows * 128 + kTileMax;
  static bool attr = false;
  if (!attr) {
    SMO_CUDA_CHECK(cudaFuncSetAttribute(tcode_decode_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    SMO_CUDA_CHECK(cudaFuncSetAttribute(tcode_decode_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
  }
  const dim3 grid(unsigned(M.t0[3]), unsigned(n));
  if (fmt == 3)
    tcode_decode_kernel<3><<<grid, 256, smem, st>>>(M, reinterpret_cast<const uint8_t* const*>(tab),
                                                     reinterpret_cast<uint16_t* const*>(tab + n));
  else
    tcode_decode_kernel<2><<<grid, 256, smem, st>>>(M, reinterpret_cast<const uint8_t* const*>(tab),
                                                     reinterpret_cast<uint16_t* const*>(tab + n));
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
  // the host vector must outlive the async copy
  SMO_CUDA_CHECK(cudaStreamSynchronize(st));
  SMO_CUDA_CHECK(cudaFreeAsync(tab, st));
}

}  // namespace smo
