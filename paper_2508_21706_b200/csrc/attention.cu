// attention.cu — K1: chunked verification attention on tcgen05.
//
// Semantics: moeplan::chunked_attention (attention.hpp:117-156) batched over
// requests and GQA heads: for draft query i of request r, the s_r prefix keys
// are implicitly visible and draft key j is visible iff bit j of mask[r,i]
// (the compact n x n mask, attention.hpp:41-58; never expanded). Softmax is
// stabilised by the running row maximum (online across 128-key chunks).
//
// Layout / mapping:
//  * work item = (request r, KV head h, KV split); persistent CTAs stride over
//    items. The g*n query rows sharing KV head h (row = i*g + hh) form the
//    M=128 A tile (Q, K-major, TMA 3D box {64, g, n}); a 128-key chunk of K is
//    the B operand of S = Q K^T (N=128); P (bf16, written by the softmax warps
//    into a swizzled K-major smem tile) times V (MN-major B, N=d) gives the
//    chunk's O contribution in TMEM, folded into fp32 registers with the
//    online-softmax rescale.
//  * warps: w0 TMA producer, w1 TMEM alloc + MMA issuer, w2..w5 softmax
//    (thread = query row = TMEM lane).
//  * TMEM: S double buffer cols [0,256), O-chunk double buffer cols [256,512).
//  * HBM-bound: algorithmic bytes = 2*b*(s+n)*n_kv*d*2 (roofline.hpp:88) +
//    Q/O; FLOPs = 4*n*(s+n)*n_q*d per request.
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace smo {

namespace {

constexpr int kThreads = 192;
constexpr int kChunk = 128;
constexpr int kKvStages = 2;

struct AttnParams {
  const uint64_t* mask;
  const int32_t* prefix;
  uint16_t* out;
  float* ws_o;
  float2* ws_ml;
  int b, n, n_q, n_kv, g, rows, s_max;
  int splits, split_chunks, items;
  float scale_log2;
};

template <int D>
struct AttnSmem {
  static constexpr int kKBlocks = D / 64;
  static constexpr int kQBytes = kKBlocks * 16384;      // 128 rows x D
  static constexpr int kKvBytes = kKBlocks * 16384;     // 128 keys x D (K or V)
  static constexpr int kPBytes = 2 * 16384;             // 128 rows x 128 keys (bf16)
  // d=128 keeps one Q buffer so that P can be held as hi+lo bf16 planes
  static constexpr int kQBufs = D == 128 ? 1 : 2;
  static constexpr int kQOff = 0;
  static constexpr int kKvOff = kQBufs * kQBytes;
  static constexpr int kPOff = kKvOff + kKvStages * 2 * kKvBytes;
  static constexpr int kPLoOff = kPOff + kPBytes;
  static constexpr int kTotal = kPLoOff + kPBytes;
};

#ifdef SMO_ATTN_TRACE
// Debug timeline of CTA 0 (globaltimer ns << 8 | event code) per role.
__device__ unsigned long long g_trace[3][4096];
__device__ int g_trace_n[3];
__device__ __forceinline__ void trace_ev(int role, int code) {
  if (blockIdx.x != 0) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  const int i = g_trace_n[role]++;
  if (i < 4096) g_trace[role][i] = (t << 8) | unsigned(code);
}
#define TR(role, code) trace_ev(role, code)
#else
#define TR(role, code)
#endif

struct ItemInfo {
  int r, h, c_begin, c_end, keys;
};

__device__ __forceinline__ ItemInfo item_info(const AttnParams& p, int item) {
  ItemInfo it;
  const int pair = item / p.splits, split = item % p.splits;
  it.r = pair / p.n_kv;
  it.h = pair % p.n_kv;
  it.keys = p.prefix[it.r] + p.n;
  const int chunks = (it.keys + kChunk - 1) / kChunk;
  it.c_begin = min(split * p.split_chunks, chunks);
  it.c_end = min(it.c_begin + p.split_chunks, chunks);
  return it;
}

// Visibility of the 32 keys [p0, p0+32) for one query row: prefix keys are
// implicitly visible, draft key d = key - prefix follows bit d of the row's
// compact mask (bits >= n are clear). One 32-bit word per piece replaces
// per-element 64-bit shifts.
__device__ __forceinline__ uint32_t visible_bits(int p0, int prefix, uint64_t mbits) {
  const int pre = prefix - p0;
  const uint32_t pm = pre <= 0 ? 0u : (pre >= 32 ? 0xffffffffu : ((1u << pre) - 1u));
  const int sh = p0 - prefix;
  uint32_t dm = 0;
  if (sh >= 0 && sh < 64) dm = uint32_t(mbits >> sh);
  else if (sh < 0 && sh > -32) dm = uint32_t(mbits << (-sh));
  return pm | dm;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    verify_attention_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kv_k,
                            const __grid_constant__ CUtensorMap tm_kv_v, AttnParams p) {
  using L = AttnSmem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t q_full[2], q_empty[2];
  __shared__ __align__(8) uint64_t kv_full[kKvStages], kv_empty[kKvStages];
  __shared__ __align__(8) uint64_t s_full[2], s_empty[2], o_full, p_full;
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4);
    }
    for (int i = 0; i < kKvStages; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(&o_full, 1);
    mbar_init(&p_full, 4);
    fence_barrier_init();
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_kv_k);
    tma_prefetch_desc(&tm_kv_v);
  }
  if (warp == 1) tmem_alloc<512>(&tmem_base_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  constexpr uint32_t kOAcc = 256;  // O accumulator columns [256, 256+D)

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (elect_one()) {
      int used = 0, gc = 0;
      for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
        const ItemInfo it = item_info(p, item);
        if (it.c_end <= it.c_begin) continue;
        const int qb = used % L::kQBufs;
        mbar_wait(&q_empty[qb], ((used / L::kQBufs) & 1) ^ 1);
        ++used;
        mbar_arrive_expect_tx(&q_full[qb], uint32_t(L::kKBlocks * 64 * p.g * p.n * 2));
        for (int kb = 0; kb < L::kKBlocks; ++kb)
          tma_load_3d(smem + L::kQOff + qb * L::kQBytes + kb * 16384, &tm_q, &q_full[qb], kb * 64, it.h * p.g,
                      it.r * p.n);
        const int row_base = (it.r * p.n_kv + it.h) * p.s_max;
        for (int c = it.c_begin; c < it.c_end; ++c, ++gc) {
          const int s = gc % kKvStages;
          TR(0, 1);
          mbar_wait(&kv_empty[s], ((gc / kKvStages) & 1) ^ 1);
          TR(0, 2);
          mbar_arrive_expect_tx(&kv_full[s], uint32_t(2 * L::kKvBytes));
          uint8_t* kdst = smem + L::kKvOff + s * 2 * L::kKvBytes;
          uint8_t* vdst = kdst + L::kKvBytes;
          for (int kb = 0; kb < L::kKBlocks; ++kb) {
            tma_load_2d(kdst + kb * 16384, &tm_kv_k, &kv_full[s], kb * 64, row_base + c * kChunk);
            tma_load_2d(vdst + kb * 16384, &tm_kv_v, &kv_full[s], kb * 64, row_base + c * kChunk);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      const uint32_t id_s = make_idesc_bf16(128, kChunk);
      const uint32_t id_o = make_idesc_bf16(128, D, /*b_mn_major=*/1);
      int used = 0, gc = 0;
      uint32_t p_phase = 0;
      for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
        const ItemInfo it = item_info(p, item);
        if (it.c_end <= it.c_begin) continue;
        const int qb = used % L::kQBufs;
        mbar_wait(&q_full[qb], (used / L::kQBufs) & 1);
        ++used;
        const uint32_t q_addr = smem_u32(smem + L::kQOff + qb * L::kQBytes);
        const int nch = it.c_end - it.c_begin;
        auto issue_s = [&](int ci) {
          const int g2 = gc + ci;
          const int s = g2 % kKvStages, sb = g2 & 1;
          TR(1, 1);
          mbar_wait(&kv_full[s], (g2 / kKvStages) & 1);
          mbar_wait(&s_empty[sb], ((g2 >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t k_addr = smem_u32(smem + L::kKvOff + s * 2 * L::kKvBytes);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
            umma_bf16(tmem + sb * 128, make_sdesc_sw128(q_addr + off, 16, 1024),
                      make_sdesc_sw128(k_addr + off, 16, 1024), id_s, kk > 0 ? 1u : 0u);
          }
          umma_commit(&s_full[sb]);
          if (ci == nch - 1) umma_commit(&q_empty[qb]);
          TR(1, 2);
        };
        issue_s(0);
        for (int ci = 0; ci < nch; ++ci) {
          if (ci + 1 < nch) issue_s(ci + 1);
          const int g2 = gc + ci;
          const int s = g2 % kKvStages;
          TR(1, 4);
          mbar_wait(&p_full, p_phase);
          TR(1, 5);
          p_phase ^= 1;
          tc_fence_after();
          const uint32_t p_addr = smem_u32(smem + L::kPOff);
          const uint32_t plo_addr = smem_u32(smem + L::kPLoOff);
          const uint32_t v_addr = smem_u32(smem + L::kKvOff + s * 2 * L::kKvBytes + L::kKvBytes);
          // O += P_hi V + P_lo V: P carried to ~16 mantissa bits
#pragma unroll
          for (int kk = 0; kk < kChunk / 16; ++kk) {
            const uint32_t aoff = (kk / 4) * 16384 + (kk % 4) * 32;
            const uint64_t vd = make_sdesc_sw128(v_addr + kk * 2048, 16384, 1024);
            umma_bf16(tmem + kOAcc, make_sdesc_sw128(p_addr + aoff, 16, 1024), vd, id_o,
                      (ci > 0 || kk > 0) ? 1u : 0u);
            umma_bf16(tmem + kOAcc, make_sdesc_sw128(plo_addr + aoff, 16, 1024), vd, id_o, 1u);
          }
          umma_commit(&o_full);
          umma_commit(&kv_empty[s]);
          TR(1, 6);
        }
        gc += nch;
      }
    }
  } else {
    // ------------------------------------------------------------ softmax
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const uint32_t tlane = uint32_t(q4 * 32) << 16;
    const bool warp_live = q4 * 32 < p.rows;  // warp-uniform
    uint8_t* pbuf = smem + L::kPOff;
    int gc = 0;
    for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
      const ItemInfo it = item_info(p, item);
      const int nch = it.c_end - it.c_begin;
      const bool live = row < p.rows;
      const int qi = live ? row / p.g : 0;
      const int hh = live ? row % p.g : 0;
      uint64_t mbits = live ? p.mask[it.r * p.n + qi] : 0ull;
      if (p.n < 64) mbits &= (1ull << p.n) - 1ull;
      const int prefix = live ? it.keys - p.n : 0;
      float m_run = -INFINITY, l_run = 0.f;
      for (int ci = 0; ci < nch; ++ci) {
        const int g2 = gc + ci;
        const int sb = g2 & 1;
        const int key0 = (it.c_begin + ci) * kChunk;
        if (warp == 4 && lane == 0) TR(2, 1);
        mbar_wait(&s_full[sb], (g2 >> 1) & 1);
        if (warp == 4 && lane == 0) TR(2, 2);
        tc_fence_after();
        float m_new = m_run, alpha = 1.f;
        if (warp_live) {
          // pass 1: masked row max of this chunk (log2 domain)
          float cmax = -INFINITY;
#pragma unroll 1
          for (int c0 = 0; c0 < kChunk; c0 += 32) {
            uint32_t r[32];
            tmem_ld32(tmem + tlane + sb * 128 + c0, r);
            const uint32_t vb = visible_bits(key0 + c0, prefix, mbits);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if ((vb >> j) & 1u) cmax = fmaxf(cmax, __uint_as_float(r[j]));
          }
          m_new = fmaxf(m_run, cmax * p.scale_log2);
          alpha = (m_run == -INFINITY) ? 0.f : ex2_approx(m_run - m_new);
        }
        if (warp == 4 && lane == 0) TR(2, 3);
        // the previous chunk's PV must be done before P is overwritten and
        // before O is rescaled in TMEM (FA4-style correction, skipped when no
        // row of this warp moved its maximum)
        if (ci > 0) {
          mbar_wait(&o_full, (g2 - 1) & 1);
          tc_fence_after();
          if (warp_live && __any_sync(0xffffffffu, live && alpha != 1.f)) {
#pragma unroll 1
            for (int c0 = 0; c0 < D; c0 += 32) {
              uint32_t r[32];
              tmem_ld32(tmem + tlane + kOAcc + c0, r);
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * alpha);
              tmem_st32(tmem + tlane + kOAcc + c0, r);
            }
            tmem_st_wait();
          }
        }
        if (warp == 4 && lane == 0) TR(2, 4);
        // pass 2: p = 2^(s*scale - m), row sum, P = hi + lo bf16 planes
        const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
        float psum = 0.f;
        if (warp_live) {
#pragma unroll 1
          for (int c0 = 0; c0 < kChunk; c0 += 32) {
            uint32_t r[32];
            tmem_ld32(tmem + tlane + sb * 128 + c0, r);
            const uint32_t vb = live ? visible_bits(key0 + c0, prefix, mbits) : 0u;
            tmem_ld_wait();
            uint32_t pk[16], pl[16];
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const float a = ((vb >> j) & 1u) ? ex2_approx(__uint_as_float(r[j]) * p.scale_log2 - m_use) : 0.f;
              const float b =
                  ((vb >> (j + 1)) & 1u) ? ex2_approx(__uint_as_float(r[j + 1]) * p.scale_log2 - m_use) : 0.f;
              psum += a + b;
              const uint32_t hi = pack_bf16x2(a, b);
              pk[j / 2] = hi;
              pl[j / 2] = pack_bf16x2(a - __uint_as_float(hi << 16), b - __uint_as_float(hi & 0xffff0000u));
            }
            const int kb = c0 / 64;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int lc = ((c0 % 64) / 8) + t;
              const int off = kb * 16384 + row * 128 + ((lc ^ (row & 7)) * 16);
              *reinterpret_cast<uint4*>(pbuf + off) = make_uint4(pk[4 * t], pk[4 * t + 1], pk[4 * t + 2], pk[4 * t + 3]);
              *reinterpret_cast<uint4*>(pbuf + (L::kPLoOff - L::kPOff) + off) =
                  make_uint4(pl[4 * t], pl[4 * t + 1], pl[4 * t + 2], pl[4 * t + 3]);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[sb]);
        l_run = l_run * alpha + psum;
        m_run = m_new;
        // keys past the request's end in the last chunk: zero their V rows so
        // stale (possibly non-finite) cache contents cannot reach the MMA
        if (key0 + kChunk > it.keys && key0 + row >= it.keys) {
          uint8_t* vbuf = smem + L::kKvOff + (g2 % kKvStages) * 2 * L::kKvBytes + L::kKvBytes;
#pragma unroll
          for (int kb = 0; kb < L::kKBlocks; ++kb)
#pragma unroll
            for (int t = 0; t < 8; ++t)
              *reinterpret_cast<uint4*>(vbuf + kb * 16384 + row * 128 + t * 16) = make_uint4(0, 0, 0, 0);
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full);
        if (warp == 4 && lane == 0) TR(2, 5);
      }
      if (nch > 0) {
        mbar_wait(&o_full, (gc + nch - 1) & 1);
        tc_fence_after();
      }
      gc += nch;
      if (!warp_live) continue;
      const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t r[32];
        if (nch > 0) {
          tmem_ld32(tmem + tlane + kOAcc + c0, r);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = 0u;
        }
        if (!live) continue;
        if (p.splits == 1) {
          uint16_t* dst = p.out + ((size_t(it.r) * p.n + qi) * p.n_q + size_t(it.h) * p.g + hh) * D + c0;
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            uint4 v;
            v.x = pack_bf16x2(__uint_as_float(r[j]) * inv, __uint_as_float(r[j + 1]) * inv);
            v.y = pack_bf16x2(__uint_as_float(r[j + 2]) * inv, __uint_as_float(r[j + 3]) * inv);
            v.z = pack_bf16x2(__uint_as_float(r[j + 4]) * inv, __uint_as_float(r[j + 5]) * inv);
            v.w = pack_bf16x2(__uint_as_float(r[j + 6]) * inv, __uint_as_float(r[j + 7]) * inv);
            *reinterpret_cast<uint4*>(dst + j) = v;
          }
        } else {
          float* dst = p.ws_o + (size_t(item) * p.rows + row) * D + c0;
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(dst + j) =
                make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                            __uint_as_float(r[j + 3]));
        }
      }
      if (live && p.splits > 1)
        p.ws_ml[size_t(item) * p.rows + row] = make_float2(nch > 0 ? m_run : -INFINITY, l_run);
      tc_fence_before();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------------------
// K1 v3 ("swap-AB"), used when the g*n query rows of a KV head fit in 64:
// S^T = K Q^T puts the 128 keys of a chunk on the TMEM lanes and the query
// rows on the columns, so each of the 128 softmax threads owns ONE key and
// does NP=64 exps per chunk (v2: one row, 128 exps, mostly one busy warp).
//   * P^T [keys][rows] is written by its key-thread as one 128-byte swizzled
//     row (MN-major B operand); O^T [d][rows] = V^T P^T with V^T the MN-major
//     A operand (V's natural layout); l[rows] = ones . P^T on the tensor core
//     (a 256-byte all-ones A tile, SBO = 0) so no cross-thread row sums.
//   * row maxima are kept per row and only refreshed (cross-thread reduce +
//     O/l rescale in TMEM) when some score exceeds max + 8 in log2 units —
//     always at an item's first chunk, rarely afterwards; p stays <= 2^8.
namespace v3 {
constexpr int kNP = 64;  // query rows per item (padded)

template <int D>
struct Smem {
  static constexpr int kKBlocks = D / 64;
  static constexpr int kQBytes = kKBlocks * 16384;
  static constexpr int kKvBytes = kKBlocks * 16384;
  static constexpr int kQOff = 0;
  static constexpr int kKvOff = kQBytes;
  static constexpr int kPOff = kKvOff + kKvStages * 2 * kKvBytes;  // P^T hi, then lo: [128 keys][64 rows]
  static constexpr int kPPlane = 16384;
  static constexpr int kOnesOff = kPOff + 2 * kPPlane;
  static constexpr int kTotal = kOnesOff + 1024;
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kv_k,
           const __grid_constant__ CUtensorMap tm_kv_v, AttnParams p) {
  using L = Smem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t q_full, q_empty;
  __shared__ __align__(8) uint64_t kv_full[kKvStages], kv_empty[kKvStages];
  __shared__ __align__(8) uint64_t s_full[2], s_empty[2], o_full, p_full;
  __shared__ uint32_t tmem_base_sh;
  __shared__ float red_sh[4][kNP];
  __shared__ float alpha_sh[kNP];
  __shared__ float m_sh[kNP];  // per-row running max (log2 units)
  __shared__ uint64_t vis_sh[64];  // draft key j -> rows that see it
  __shared__ uint64_t mrow_sh[64]; // compact mask word of draft query i
  __shared__ int flag_sh[4];

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    mbar_init(&q_full, 1);
    mbar_init(&q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4);
    }
    for (int i = 0; i < kKvStages; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(&o_full, 1);
    mbar_init(&p_full, 4);
    fence_barrier_init();
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_kv_k);
    tma_prefetch_desc(&tm_kv_v);
  }
  if (warp == 1) tmem_alloc<256>(&tmem_base_sh);
  if (warp >= 2) {  // all-ones A tile for the row-sum MMA (bf16 1.0)
    for (int i = threadIdx.x - 64; i < 64; i += 128) reinterpret_cast<uint32_t*>(smem + L::kOnesOff)[i] = 0x3F803F80u;
    fence_proxy_async();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  constexpr uint32_t kS = 0, kO = 2 * kNP, kL = 3 * kNP;  // TMEM columns

  if (warp == 0) {
    if (elect_one()) {
      int used = 0, gc = 0;
      for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
        const ItemInfo it = item_info(p, item);
        if (it.c_end <= it.c_begin) continue;
        mbar_wait(&q_empty, (used & 1) ^ 1);
        ++used;
        mbar_arrive_expect_tx(&q_full, uint32_t(L::kKBlocks * 64 * p.g * p.n * 2));
        for (int kb = 0; kb < L::kKBlocks; ++kb)
          tma_load_3d(smem + L::kQOff + kb * 16384, &tm_q, &q_full, kb * 64, it.h * p.g, it.r * p.n);
        const int row_base = (it.r * p.n_kv + it.h) * p.s_max;
        for (int c = it.c_begin; c < it.c_end; ++c, ++gc) {
          const int s = gc % kKvStages;
          TR(0, 1);
          mbar_wait(&kv_empty[s], ((gc / kKvStages) & 1) ^ 1);
          TR(0, 2);
          mbar_arrive_expect_tx(&kv_full[s], uint32_t(2 * L::kKvBytes));
          uint8_t* kdst = smem + L::kKvOff + s * 2 * L::kKvBytes;
          uint8_t* vdst = kdst + L::kKvBytes;
          for (int kb = 0; kb < L::kKBlocks; ++kb) {
            tma_load_2d(kdst + kb * 16384, &tm_kv_k, &kv_full[s], kb * 64, row_base + c * kChunk);
            tma_load_2d(vdst + kb * 16384, &tm_kv_v, &kv_full[s], kb * 64, row_base + c * kChunk);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      const uint32_t id_s = make_idesc_bf16(128, kNP);                      // K (keys) x Q^T
      const uint32_t id_o = make_idesc_bf16(128, kNP, /*b_mn=*/1, /*a_mn=*/1);  // V^T x P^T
      const uint32_t id_l = make_idesc_bf16(128, kNP, /*b_mn=*/1, /*a_mn=*/0);  // ones x P^T
      const uint32_t q_addr = smem_u32(smem + L::kQOff);
      const uint32_t p_addr = smem_u32(smem + L::kPOff);
      // all-ones A: no swizzle, K core matrices 128 B apart, every 8-row group
      // aliases the same 256 bytes (SBO = 0)
      uint64_t ones_d = uint64_t((smem_u32(smem + L::kOnesOff) >> 4) & 0x3FFFu) | (uint64_t(128 >> 4) << 16) |
                        (uint64_t(1) << 46);
      int used = 0, gc = 0;
      uint32_t p_phase = 0;
      for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
        const ItemInfo it = item_info(p, item);
        if (it.c_end <= it.c_begin) continue;
        mbar_wait(&q_full, used & 1);
        ++used;
        const int nch = it.c_end - it.c_begin;
        auto issue_s = [&](int ci) {
          const int g2 = gc + ci;
          const int s = g2 % kKvStages, sb = g2 & 1;
          TR(1, 1);
          mbar_wait(&kv_full[s], (g2 / kKvStages) & 1);
          mbar_wait(&s_empty[sb], ((g2 >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t k_addr = smem_u32(smem + L::kKvOff + s * 2 * L::kKvBytes);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
            umma_bf16(tmem + kS + sb * kNP, make_sdesc_sw128(k_addr + off, 16, 1024),
                      make_sdesc_sw128(q_addr + off, 16, 1024), id_s, kk > 0 ? 1u : 0u);
          }
          umma_commit(&s_full[sb]);
          if (ci == nch - 1) umma_commit(&q_empty);
          TR(1, 2);
        };
        issue_s(0);
        for (int ci = 0; ci < nch; ++ci) {
          if (ci + 1 < nch) issue_s(ci + 1);
          const int g2 = gc + ci;
          const int s = g2 % kKvStages;
          TR(1, 4);
          mbar_wait(&p_full, p_phase);
          TR(1, 5);
          p_phase ^= 1;
          tc_fence_after();
          const uint32_t v_addr = smem_u32(smem + L::kKvOff + s * 2 * L::kKvBytes + L::kKvBytes);
#pragma unroll
          for (int kk = 0; kk < kChunk / 16; ++kk) {
            const uint64_t vd = make_sdesc_sw128(v_addr + kk * 2048, 16384, 1024);
            const uint64_t ph = make_sdesc_sw128(p_addr + kk * 2048, 16384, 1024);
            const uint64_t pl = make_sdesc_sw128(p_addr + L::kPPlane + kk * 2048, 16384, 1024);
            const uint32_t acc = (ci > 0 || kk > 0) ? 1u : 0u;
            umma_bf16(tmem + kO, vd, ph, id_o, acc);
            umma_bf16(tmem + kO, vd, pl, id_o, 1u);
            umma_bf16(tmem + kL, ones_d, ph, id_l, acc);
            umma_bf16(tmem + kL, ones_d, pl, id_l, 1u);
          }
          umma_commit(&o_full);
          umma_commit(&kv_empty[s]);
          TR(1, 6);
        }
        gc += nch;
      }
    }
  } else {
    // ---------------------------------------------- softmax: thread = key lane
    const int q4 = warp & 3;
    const int kt = q4 * 32 + lane;                 // key within the chunk (TMEM lane)
    const uint32_t tl = uint32_t(q4 * 32) << 16;
    const int st = threadIdx.x - 64;               // 0..127
    uint8_t* pbuf = smem + L::kPOff;
    int gc = 0;
    for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
      const ItemInfo it = item_info(p, item);
      const int nch = it.c_end - it.c_begin;
      const int prefix = it.keys - p.n;
      // draft visibility per draft key j: rows (i*g+hh) whose query i sees j
      if (st < p.n) mrow_sh[st] = p.mask[it.r * p.n + st];
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (st < 64) {
        uint64_t rows = 0;
        if (st < p.n)
          for (int r = 0; r < p.rows; ++r)
            if ((mrow_sh[r / p.g] >> st) & 1ull) rows |= 1ull << r;
        vis_sh[st] = rows;
      }
      const uint64_t live_rows = p.rows >= 64 ? ~0ull : ((1ull << p.rows) - 1ull);
      if (st < kNP) m_sh[st] = -INFINITY;
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (st == 0) TR(2, 8);
      for (int ci = 0; ci < nch; ++ci) {
        const int g2 = gc + ci;
        const int sb = g2 & 1;
        const int key = (it.c_begin + ci) * kChunk + kt;
        const uint64_t vis = key < prefix ? live_rows : (key < it.keys ? vis_sh[key - prefix] & live_rows : 0ull);
        if (st == 0) TR(2, 1);
        mbar_wait(&s_full[sb], (g2 >> 1) & 1);
        if (st == 0) TR(2, 2);
        tc_fence_after();
        uint32_t sr[kNP];
        {
          uint32_t a[32], b[32];
          tmem_ld32(tmem + tl + kS + sb * kNP, a);
          tmem_ld32(tmem + tl + kS + sb * kNP + 32, b);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            sr[j] = __float_as_uint(__uint_as_float(a[j]) * p.scale_log2);
            sr[j + 32] = __float_as_uint(__uint_as_float(b[j]) * p.scale_log2);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[sb]);
        // does any visible score exceed its row max by more than 2^8?
        bool grow = false;
#pragma unroll
        for (int j = 0; j < kNP; ++j) grow |= ((vis >> j) & 1ull) && (__uint_as_float(sr[j]) > m_sh[j] + 8.f);
        grow = __any_sync(0xffffffffu, grow);
        if (lane == 0) flag_sh[q4] = grow ? 1 : 0;
        asm volatile("bar.sync 2, 128;" ::: "memory");
        const bool any_grow = (flag_sh[0] | flag_sh[1] | flag_sh[2] | flag_sh[3]) != 0;
        if (st == 0) TR(2, any_grow ? 9 : 3);
        if (any_grow) {
          // exact per-row max of this chunk over the 128 keys: warp max, then 4 warps
#pragma unroll
          for (int j = 0; j < kNP; ++j) {
            const float v = warp_max(((vis >> j) & 1ull) ? __uint_as_float(sr[j]) : -INFINITY);
            if (lane == 0) red_sh[q4][j] = v;
          }
          asm volatile("bar.sync 2, 128;" ::: "memory");
          if (st < kNP) {
            // per-row decision (a row's reference max depends only on its own
            // scores, which keeps causality bit-exact): refresh only rows that
            // are unset or grew past max + 8
            const int j = st;
            const float cm = fmaxf(fmaxf(red_sh[0][j], red_sh[1][j]), fmaxf(red_sh[2][j], red_sh[3][j]));
            const float mo = m_sh[j];
            const bool refresh = cm != -INFINITY && (mo == -INFINITY || cm > mo + 8.f);
            const float mn = refresh ? cm : mo;
            alpha_sh[j] = refresh ? (mo == -INFINITY ? 0.f : ex2_approx(mo - mn)) : 1.f;
            m_sh[j] = mn;
          }
          asm volatile("bar.sync 2, 128;" ::: "memory");  // m_sh/alpha_sh visible, red_sh reusable
        }
        // previous PV must be done before P is overwritten / O rescaled
        if (ci > 0) {
          mbar_wait(&o_full, (g2 - 1) & 1);
          tc_fence_after();
          if (any_grow) {  // O^T[d][row] and l[row] *= alpha[row]
#pragma unroll 1
            for (int part = 0; part < 2; ++part) {
              const uint32_t col = part == 0 ? kO : kL;
#pragma unroll
              for (int h2 = 0; h2 < 2; ++h2) {
                uint32_t r[32];
                tmem_ld32(tmem + tl + col + h2 * 32, r);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * alpha_sh[h2 * 32 + j]);
                tmem_st32(tmem + tl + col + h2 * 32, r);
              }
            }
            tmem_st_wait();
          }
        }
        if (st == 0) TR(2, 4);
        // p = 2^(s - m) for visible (key,row) pairs; P^T row `kt` as hi + lo bf16
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint32_t hi4[4], lo4[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int j = c * 8 + t * 2;
            const float a = ((vis >> j) & 1ull) ? ex2_approx(__uint_as_float(sr[j]) - m_sh[j]) : 0.f;
            const float b = ((vis >> (j + 1)) & 1ull) ? ex2_approx(__uint_as_float(sr[j + 1]) - m_sh[j + 1]) : 0.f;
            const uint32_t hh = pack_bf16x2(a, b);
            hi4[t] = hh;
            lo4[t] = pack_bf16x2(a - __uint_as_float(hh << 16), b - __uint_as_float(hh & 0xffff0000u));
          }
          const int off = kt * 128 + ((c ^ (kt & 7)) * 16);
          *reinterpret_cast<uint4*>(pbuf + off) = make_uint4(hi4[0], hi4[1], hi4[2], hi4[3]);
          *reinterpret_cast<uint4*>(pbuf + L::kPPlane + off) = make_uint4(lo4[0], lo4[1], lo4[2], lo4[3]);
        }
        // keys past the request's end: zero their V rows (stale cache contents)
        if (key >= it.keys) {
          uint8_t* vbuf = smem + L::kKvOff + (g2 % kKvStages) * 2 * L::kKvBytes + L::kKvBytes;
#pragma unroll
          for (int kb = 0; kb < L::kKBlocks; ++kb)
#pragma unroll
            for (int t = 0; t < 8; ++t)
              *reinterpret_cast<uint4*>(vbuf + kb * 16384 + kt * 128 + t * 16) = make_uint4(0, 0, 0, 0);
        }
        fence_proxy_async();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full);
        if (st == 0) TR(2, 5);
      }
      if (nch > 0) {
        mbar_wait(&o_full, (gc + nch - 1) & 1);
        tc_fence_after();
      }
      if (st == 0) TR(2, 6);
      gc += nch;
      // epilogue: thread = d lane; l from the ones-MMA (identical on every lane)
      if (kt < D) {
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          uint32_t lr[32], o[32];
          if (nch > 0) {
            tmem_ld32(tmem + tl + kL + h2 * 32, lr);
            tmem_ld32(tmem + tl + kO + h2 * 32, o);
            tmem_ld_wait();
            if (st == 0) TR(2, 10 + h2);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) lr[j] = o[j] = 0u;
          }
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const int j = h2 * 32 + jj;
            if (j >= p.rows) continue;
            const float l = __uint_as_float(lr[jj]);
            const int qi = j / p.g, hh = j % p.g;
            if (p.splits == 1) {
              p.out[((size_t(it.r) * p.n + qi) * p.n_q + size_t(it.h) * p.g + hh) * D + kt] =
                  f2bf(l > 0.f ? __uint_as_float(o[jj]) / l : 0.f);
            } else {
              p.ws_o[(size_t(item) * p.rows + j) * D + kt] = __uint_as_float(o[jj]);
              if (kt == 0) p.ws_ml[size_t(item) * p.rows + j] = make_float2(nch > 0 ? m_sh[j] : -INFINITY, l);
            }
          }
        }
      }
      if (st == 0) TR(2, 7);
      tc_fence_before();
      asm volatile("bar.sync 2, 128;" ::: "memory");  // TMEM O/l read before the next item's PV(0)
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<256>(tmem);
}
}  // namespace v3

// Merge the split-KV partials: O = sum_s O_s 2^(m_s - M) / sum_s l_s 2^(m_s - M).
template <int D>
__global__ void attn_combine_kernel(AttnParams p) {
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  const int pairs = p.b * p.n_kv;
  if (warp_global >= pairs * p.rows) return;
  const int pair = warp_global / p.rows, row = warp_global % p.rows;
  const int r = pair / p.n_kv, h = pair % p.n_kv;
  float M = -INFINITY;
  for (int s = 0; s < p.splits; ++s) M = fmaxf(M, p.ws_ml[size_t(pair * p.splits + s) * p.rows + row].x);
  constexpr int V = D / 32;
  float acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = 0.f;
  float L = 0.f;
  for (int s = 0; s < p.splits; ++s) {
    const size_t item = size_t(pair) * p.splits + s;
    const float2 ml = p.ws_ml[item * p.rows + row];
    if (ml.x == -INFINITY) continue;
    const float w = exp2f(ml.x - M);
    L += ml.y * w;
    const float* src = p.ws_o + (item * p.rows + row) * D;
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] += src[lane + 32 * v] * w;
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  const int qi = row / p.g, hh = row % p.g;
  uint16_t* dst = p.out + ((size_t(r) * p.n + qi) * p.n_q + size_t(h) * p.g + hh) * D;
#pragma unroll
  for (int v = 0; v < V; ++v) dst[lane + 32 * v] = f2bf(acc[v] * inv);
}

struct AttnPlan {
  int splits, split_chunks, items, grid;
  size_t ws_bytes;
};

AttnPlan plan_attention(const smo_attn_args& a, int sms) {
  AttnPlan pl{};
  const int g = a.n_q / a.n_kv;
  const int rows = g * a.n;
  const int max_keys = std::max(1, a.max_prefix + a.n);
  const int chunks = (max_keys + kChunk - 1) / kChunk;
  const int pairs = a.b * a.n_kv;
  // enough items for ~2 rounds of the persistent grid, at least 2 chunks each
  int splits = std::max(1, std::min(chunks, (2 * sms + pairs - 1) / pairs));
  if (splits > 1) splits = std::min(splits, std::max(1, chunks / 2));
  pl.split_chunks = (chunks + splits - 1) / splits;
  pl.splits = (chunks + pl.split_chunks - 1) / pl.split_chunks;
  pl.items = pairs * pl.splits;
  pl.grid = std::min(pl.items, sms);
  pl.ws_bytes = pl.splits > 1 ? size_t(pl.items) * rows * (a.d * sizeof(float) + sizeof(float2)) : 0;
  return pl;
}

int device_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// K1 variant for rows <= 64: 2 = row-per-thread (default), 3 = swap-AB
// key-per-thread; SMO_ATTN_VARIANT overrides (read once)
int attn_variant() {
  static int v = [] {
    const char* e = std::getenv("SMO_ATTN_VARIANT");
    return e && std::atoi(e) == 3 ? 3 : 2;
  }();
  return v;
}

void check_attn_args(const smo_attn_args& a) {
  SMO_REQUIRE(a.q && a.k_cache && a.v_cache && a.mask && a.prefix_len && a.out, "attention: null pointer");
  SMO_REQUIRE(a.b > 0 && a.n > 0 && a.n_q > 0 && a.n_kv > 0, "attention: shape mismatch");
  SMO_REQUIRE(a.n_q % a.n_kv == 0, "attention: shape mismatch");
  SMO_REQUIRE(a.d == 64 || a.d == 128, "attention: head_dim must be 64 or 128");
  SMO_REQUIRE(a.n <= 64, "attention: mask size mismatch");
  SMO_REQUIRE((a.n_q / a.n_kv) * a.n <= 128, "attention: n * (n_q/n_kv) must be <= 128");
  SMO_REQUIRE(a.max_prefix >= 0 && a.max_prefix + a.n <= a.s_max, "attention: shape mismatch");
}

}  // namespace

size_t attention_workspace(const smo_attn_args& a) {
  check_attn_args(a);
  return plan_attention(a, device_sms()).ws_bytes;
}

void attention_launch(const smo_attn_args& a, cudaStream_t stream) {
  check_attn_args(a);
  const AttnPlan pl = plan_attention(a, device_sms());
  SMO_REQUIRE(pl.ws_bytes == 0 || (a.workspace && a.workspace_bytes >= pl.ws_bytes),
              "attention: workspace too small");
  const int g = a.n_q / a.n_kv;
  AttnParams p{};
  p.mask = a.mask;
  p.prefix = a.prefix_len;
  p.out = reinterpret_cast<uint16_t*>(a.out);
  p.ws_o = reinterpret_cast<float*>(a.workspace);
  p.ws_ml = reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(a.workspace) +
                                      (pl.ws_bytes ? size_t(pl.items) * g * a.n * a.d * sizeof(float) : 0));
  p.b = a.b;
  p.n = a.n;
  p.n_q = a.n_q;
  p.n_kv = a.n_kv;
  p.g = g;
  p.rows = g * a.n;
  p.s_max = a.s_max;
  p.splits = pl.splits;
  p.split_chunks = pl.split_chunks;
  p.items = pl.items;
  p.scale_log2 = float(1.4426950408889634 / std::sqrt(double(a.d)));

  CUtensorMap tq, tk, tv;
  {
    uint64_t dims[3] = {uint64_t(a.d), uint64_t(a.n_q), uint64_t(a.b) * a.n};
    uint64_t strides[2] = {uint64_t(a.d) * 2, uint64_t(a.n_q) * a.d * 2};
    uint32_t box[3] = {64, uint32_t(g), uint32_t(a.n)};
    make_tmap_bf16(&tq, a.q, 3, dims, strides, box, true);
  }
  {
    uint64_t dims[2] = {uint64_t(a.d), uint64_t(a.b) * a.n_kv * a.s_max};
    uint64_t strides[1] = {uint64_t(a.d) * 2};
    uint32_t box[2] = {64, uint32_t(kChunk)};
    make_tmap_bf16(&tk, a.k_cache, 2, dims, strides, box, true);
    make_tmap_bf16(&tv, a.v_cache, 2, dims, strides, box, true);
  }
  if (p.rows <= v3::kNP && attn_variant() == 3) {
    if (a.d == 128) {
      constexpr size_t smem = v3::Smem<128>::kTotal + 1024;
      static bool set = false;
      if (!set) {
        SMO_CUDA_CHECK(cudaFuncSetAttribute(v3::kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        set = true;
      }
      v3::kernel<128><<<pl.grid, kThreads, smem, stream>>>(tq, tk, tv, p);
    } else {
      constexpr size_t smem = v3::Smem<64>::kTotal + 1024;
      static bool set = false;
      if (!set) {
        SMO_CUDA_CHECK(cudaFuncSetAttribute(v3::kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        set = true;
      }
      v3::kernel<64><<<pl.grid, kThreads, smem, stream>>>(tq, tk, tv, p);
    }
  } else if (a.d == 128) {
    constexpr size_t smem = AttnSmem<128>::kTotal + 1024;
    static bool set = false;
    if (!set) {
      SMO_CUDA_CHECK(cudaFuncSetAttribute(verify_attention_kernel<128>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      set = true;
    }
    verify_attention_kernel<128><<<pl.grid, kThreads, smem, stream>>>(tq, tk, tv, p);
  } else {
    constexpr size_t smem = AttnSmem<64>::kTotal + 1024;
    static bool set = false;
    if (!set) {
      SMO_CUDA_CHECK(cudaFuncSetAttribute(verify_attention_kernel<64>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      set = true;
    }
    verify_attention_kernel<64><<<pl.grid, kThreads, smem, stream>>>(tq, tk, tv, p);
  }
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
  if (pl.splits > 1) {
    const int warps = a.b * a.n_kv * p.rows;
    const int blocks = (warps * 32 + 255) / 256;
    if (a.d == 128)
      attn_combine_kernel<128><<<blocks, 256, 0, stream>>>(p);
    else
      attn_combine_kernel<64><<<blocks, 256, 0, stream>>>(p);
    count_launch();
    SMO_CUDA_CHECK(cudaGetLastError());
  }
}

// ---------------------------------------------------------------------------
// fp64 desk-scale operator (the reference API, attention.hpp:117-156), one
// block per query row; columns visited prefix-first then masked drafts, the
// same order as the reference so results agree to fp64 rounding.
__global__ void chunked_attention_f64_kernel(int n, int p, int d, const double* Q, const double* K,
                                             const double* V, const uint8_t* mask, double* scores,
                                             double* out, int* blocked) {
  const int i = blockIdx.x;
  const int total = p + n;
  const double scale = 1.0 / sqrt(double(d));
  double* sc = scores + size_t(i) * total;
  __shared__ double red[256];
  double mx = -INFINITY;
  for (int j = threadIdx.x; j < total; j += blockDim.x) {
    const bool vis = j < p || mask[size_t(i) * n + (j - p)];
    double s = -INFINITY;
    if (vis) {
      double acc = 0.0;
      for (int c = 0; c < d; ++c) acc += Q[size_t(i) * d + c] * K[size_t(j) * d + c];
      s = acc * scale;
    }
    sc[j] = s;
    mx = fmax(mx, s);
  }
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int o = blockDim.x / 2; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  mx = red[0];
  __syncthreads();
  if (mx == -INFINITY) {
    if (threadIdx.x == 0) *blocked = 1;
    return;
  }
  // serial denominator in column order (matches the reference's summation)
  if (threadIdx.x == 0) {
    double den = 0.0;
    for (int j = 0; j < total; ++j)
      if (sc[j] != -INFINITY) {
        sc[j] = exp(sc[j] - mx);
        den += sc[j];
      } else {
        sc[j] = 0.0;
      }
    red[0] = den;
  }
  __syncthreads();
  const double den = red[0];
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < total; ++j)
      if (j < p || mask[size_t(i) * n + (j - p)]) acc += (sc[j] / den) * V[size_t(j) * d + c];
    out[size_t(i) * d + c] = acc;
  }
}

#ifdef SMO_ATTN_TRACE
extern "C" int smo_debug_attn_trace(unsigned long long* out, int* counts) {
  cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace));
  cudaMemcpyFromSymbol(counts, g_trace_n, sizeof(g_trace_n));
  int z[3] = {0, 0, 0};
  cudaMemcpyToSymbol(g_trace_n, z, sizeof(z));
  return 0;
}
#endif

void chunked_attention_f64(size_t n, size_t p, size_t d, const double* Q, const double* K, const double* V,
                           size_t mask_n, const uint8_t* mask, double* out) {
  const size_t total = p + n;
  for (size_t i = 0; i < n * d; ++i)
    if (!std::isfinite(Q[i])) throw Error(SMO_INVALID_ARG, "attention: non-finite Q");
  for (size_t i = 0; i < total * d; ++i)
    if (!std::isfinite(K[i])) throw Error(SMO_INVALID_ARG, "attention: non-finite K");
  for (size_t i = 0; i < total * d; ++i)
    if (!std::isfinite(V[i])) throw Error(SMO_INVALID_ARG, "attention: non-finite V");
  if (mask_n != n) throw Error(SMO_INVALID_ARG, "attention: mask size mismatch");
  if (n == 0) return;
  double *dQ, *dK, *dV, *dS, *dO;
  uint8_t* dM;
  int* dB;
  SMO_CUDA_CHECK(cudaMalloc(&dQ, sizeof(double) * n * d + 16));
  SMO_CUDA_CHECK(cudaMalloc(&dK, sizeof(double) * total * d + 16));
  SMO_CUDA_CHECK(cudaMalloc(&dV, sizeof(double) * total * d + 16));
  SMO_CUDA_CHECK(cudaMalloc(&dS, sizeof(double) * n * total + 16));
  SMO_CUDA_CHECK(cudaMalloc(&dO, sizeof(double) * n * d + 16));
  SMO_CUDA_CHECK(cudaMalloc(&dM, n * n + 16));
  SMO_CUDA_CHECK(cudaMalloc(&dB, sizeof(int)));
  SMO_CUDA_CHECK(cudaMemcpy(dQ, Q, sizeof(double) * n * d, cudaMemcpyHostToDevice));
  SMO_CUDA_CHECK(cudaMemcpy(dK, K, sizeof(double) * total * d, cudaMemcpyHostToDevice));
  SMO_CUDA_CHECK(cudaMemcpy(dV, V, sizeof(double) * total * d, cudaMemcpyHostToDevice));
  SMO_CUDA_CHECK(cudaMemcpy(dM, mask, n * n, cudaMemcpyHostToDevice));
  SMO_CUDA_CHECK(cudaMemset(dB, 0, sizeof(int)));
  chunked_attention_f64_kernel<<<int(n), 256>>>(int(n), int(p), int(d), dQ, dK, dV, dM, dS, dO, dB);
  count_launch();
  int blocked = 0;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(&blocked, dB, sizeof(int), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(out, dO, sizeof(double) * n * d, cudaMemcpyDeviceToHost);
  cudaFree(dQ); cudaFree(dK); cudaFree(dV); cudaFree(dS); cudaFree(dO); cudaFree(dM); cudaFree(dB);
  cuda_check(e, "chunked_attention_f64");
  if (blocked) throw Error(SMO_INVALID_ARG, "attention: fully blocked query row");
}

}  // namespace smo
