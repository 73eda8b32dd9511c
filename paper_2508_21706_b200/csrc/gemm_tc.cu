// gemm_tc.cu — K4: tcgen05/TMEM GEMM fed by TMA, used for the grouped SwiGLU
// experts and (one group) for the dense QKV / O / LM-head projections.
//
// Swap-AB: the weight matrix W [N, K] (nn.Linear layout, K contiguous) is the
// 128-row A operand; the small token batch X [rows, K] is the B operand
// (MMA N = tokens, up to 256 per instruction, two instructions for up to 512).
// One CTA = one 128-row weight tile x one token tile of one group (expert).
// Warp roles: w0 TMA producer, w1 TMEM allocator + single-thread MMA issuer,
// w2..w5 epilogue (TMEM -> registers -> global). The smem ring is a
// full/empty mbarrier pipeline; tcgen05.commit releases stages.
//
// Algorithmic cost (roofline.hpp:56-64, moe_cost_large_batch):
//   FLOPs = 2 * rows * N * K (x2 for SwiGLU), HBM bytes ~= weight bytes
//   (N*K*2 per group, x2 for SwiGLU) + activations.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace smo {

namespace {

constexpr int kThreads = 192;
constexpr int kBK = 64;           // K elements per stage (one 128 B swizzle atom)
constexpr int kTileBytesA = 128 * kBK * 2;
constexpr int kMaxStages = 8;
constexpr int kSmemBudget = 220 * 1024;

struct GemmParams {
  int K, N, rows;
  const int32_t* row_offsets;
  const int32_t* w_index;
  int tile_tokens;
  int stages;
  int epilogue;
  void* out;
  int64_t ldo;
  float* amax_val;
  int32_t* amax_idx;
  int n_tiles;
  int split_k;       // K split across blockIdx.z (deterministic partials + reduce)
  int kb_per_split;
  int token_tiles;
  float* partial;    // [split_k][rows][N] fp32 when split_k > 1
  int cluster;       // CTAs along the weight tiles sharing each token-row box by TMA multicast (1: none)
  int csplit;        // split-K reduced inside a (1, 1, split_k) cluster through DSMEM (no partials in HBM)
};

__device__ __forceinline__ void tmem_alloc_dyn(uint32_t cols, uint32_t* dst) {
  switch (cols) {
    case 32: tmem_alloc<32>(dst); break;
    case 64: tmem_alloc<64>(dst); break;
    case 128: tmem_alloc<128>(dst); break;
    case 256: tmem_alloc<256>(dst); break;
    default: tmem_alloc<512>(dst); break;
  }
}
__device__ __forceinline__ void tmem_dealloc_dyn(uint32_t cols, uint32_t taddr) {
  switch (cols) {
    case 32: tmem_dealloc<32>(taddr); break;
    case 64: tmem_dealloc<64>(taddr); break;
    case 128: tmem_dealloc<128>(taddr); break;
    case 256: tmem_dealloc<256>(taddr); break;
    default: tmem_dealloc<512>(taddr); break;
  }
}

__device__ __forceinline__ void tmem_alloc_pair_dyn(uint32_t cols, uint32_t* dst) {
  switch (cols) {
    case 32: tmem_alloc_pair<32>(dst); break;
    case 64: tmem_alloc_pair<64>(dst); break;
    case 128: tmem_alloc_pair<128>(dst); break;
    case 256: tmem_alloc_pair<256>(dst); break;
    default: tmem_alloc_pair<512>(dst); break;
  }
}
__device__ __forceinline__ void tmem_dealloc_pair_dyn(uint32_t cols, uint32_t taddr) {
  switch (cols) {
    case 32: tmem_dealloc_pair<32>(taddr); break;
    case 64: tmem_dealloc_pair<64>(taddr); break;
    case 128: tmem_dealloc_pair<128>(taddr); break;
    case 256: tmem_dealloc_pair<256>(taddr); break;
    default: tmem_dealloc_pair<512>(taddr); break;
  }
}

// kPair: CTA pairs (tcgen05 cta_group::2, cluster x = 2): the pair's two
// 128-row weight tiles form one M = 256 MMA issued by the even CTA; each CTA
// loads its own weight rows and HALF of the token rows (N split across the
// pair), so every token row crosses into shared memory once per 256 weight
// rows instead of once per 128 — the token operand is 2.25x the weight bytes
// per stage at 288 tokens. Each CTA's TMEM holds its 128 rows x all tokens,
// so the epilogues are the single-CTA ones.
template <bool kPair>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_u,
                   const __grid_constant__ CUtensorMap tm_x, GemmParams p, uint32_t tmem_cols) {
  // z = token tile * split_k + K slice: the K slices of one output tile are
  // consecutive, i.e. one (1, 1, split_k) cluster in the DSMEM-reduce mode
  const int nb = blockIdx.x, g = blockIdx.y, tt = blockIdx.z / p.split_k, ks = blockIdx.z % p.split_k;
  const int g_begin = p.row_offsets ? p.row_offsets[g] : 0;
  const int g_end = p.row_offsets ? p.row_offsets[g + 1] : p.rows;
  const int row0 = g_begin + tt * p.tile_tokens;
  const int cnt = min(p.tile_tokens, g_end - row0);
  if (cnt <= 0) return;  // uniform across the CTA

  const bool swiglu = p.epilogue == SMO_EPI_SWIGLU;
  const int wblk = p.w_index ? p.w_index[g] : g;
  // pair: tokens padded to 64 so each instruction's N (n1 <= 256, n2) splits
  // into two halves of whole 32-row boxes; CTA r loads rows [r n1/2, ..) and
  // [n1 + r n2/2, ..) of the tile (rows past the batch load as zeros)
  const int n_pad = kPair ? (cnt + 63) & ~63 : (cnt + 15) & ~15;
  const int n_load = kPair ? n_pad / 2 : (cnt + 31) & ~31;  // token rows this CTA loads per stage
  const int a_bytes = kTileBytesA * (swiglu ? 2 : 1);
  const int stage_bytes = a_bytes + (kPair ? p.tile_tokens / 2 : p.tile_tokens) * 128;
  const uint32_t tx_bytes = uint32_t(a_bytes + (n_load / 32) * 4096);
  const int kb0 = ks * p.kb_per_split;
  const int KB = min(p.K / kBK - kb0, p.kb_per_split);  // k-blocks of this CTA's K slice

  extern __shared__ uint8_t smem_raw[];
  // align within the shared array (keeps the shared address space visible to
  // the compiler: LDS/STS instead of generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full_bar[kMaxStages];
  __shared__ __align__(8) uint64_t empty_bar[kMaxStages];
  __shared__ __align__(8) uint64_t tmem_full_bar;
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // cluster of p.cluster CTAs over consecutive weight tiles (same group, token
  // tile and K slice): each loads 1/cluster of the token-row boxes of a stage
  // and multicasts them to all, and a stage is reused only once every CTA's
  // MMA released it (the commit arrives on every CTA's empty barrier)
  const int cs = p.cluster;
  const uint32_t crank = (cs > 1 || kPair || p.csplit) ? cluster_ctarank() : 0u;
  const uint16_t cmask = uint16_t((1u << cs) - 1u);
  const uint32_t pr = kPair ? (crank & 1u) : 0u;          // rank within the CTA pair
  const uint32_t lead = crank & ~1u;                       // the pair's even (MMA-issuing) CTA
  const uint16_t pmask = uint16_t(3u << lead);             // both CTAs of the pair
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], uint32_t(cs));
    }
    mbar_init(&tmem_full_bar, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tm_w);
    tma_prefetch_desc(&tm_x);
    if (swiglu) tma_prefetch_desc(&tm_u);
  }
  if (warp == 1) {
    if constexpr (kPair) tmem_alloc_pair_dyn(tmem_cols, &tmem_base_sh);
    else tmem_alloc_dyn(tmem_cols, &tmem_base_sh);
  }
  tc_fence_before();
  __syncthreads();
  if (cs > 1 || kPair) cluster_sync_all();  // every CTA's barriers are initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0) {
    if (elect_one()) {
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % p.stages;
        const uint32_t ph = (kb / p.stages) & 1;
        mbar_wait(&empty_bar[s], ph ^ 1);
        uint8_t* sa = smem + s * stage_bytes;
        const int kc = (kb0 + kb) * kBK;
        uint8_t* sb = sa + a_bytes;
        if constexpr (kPair) {
          // own weight rows + own half of the token rows, completing on the
          // leader's full barrier; the leader alone arrives, expecting both
          // CTAs' bytes (the tx count may run ahead of the expectation: the
          // peer refills stage s only after the leader's commit released it)
          const uint32_t fb = mapa_u32(smem_u32(&full_bar[s]), lead);
          if (pr == 0) mbar_arrive_expect_tx(&full_bar[s], 2 * tx_bytes);
          tma_load_3d_pair(sa, &tm_w, fb, kc, nb * 128, wblk);
          const int n1 = min(n_pad, 256), n2 = n_pad - n1;
          for (int i = 0; i < n1 / 64; ++i)
            tma_load_2d_pair(sb + i * 4096, &tm_x, fb, kc, row0 + int(pr) * (n1 / 2) + i * 32);
          for (int i = 0; i < n2 / 64; ++i)
            tma_load_2d_pair(sb + (n1 / 64 + i) * 4096, &tm_x, fb, kc, row0 + n1 + int(pr) * (n2 / 2) + i * 32);
          continue;
        }
        mbar_arrive_expect_tx(&full_bar[s], tx_bytes);
        tma_load_3d(sa, &tm_w, &full_bar[s], kc, nb * 128, wblk);
        if (swiglu) tma_load_3d(sa + kTileBytesA, &tm_u, &full_bar[s], kc, nb * 128, wblk);
        if (cs > 1) {
          for (int i = int(crank); i < n_load / 32; i += cs)
            tma_load_2d_mc(sb + i * 4096, &tm_x, &full_bar[s], kc, row0 + i * 32, cmask);
        } else {
          for (int i = 0; i < n_load / 32; ++i) tma_load_2d(sb + i * 4096, &tm_x, &full_bar[s], kc, row0 + i * 32);
        }
      }
    }
  } else if (warp == 1) {
    if (kPair && pr != 0) {
      // the pair's MMAs are issued by the even CTA
    } else if (kPair) {
      if (elect_one()) {
        const int n1 = min(n_pad, 256), n2 = n_pad - n1;
        const uint32_t id0 = make_idesc_bf16(256, n1);
        const uint32_t id1 = n2 > 0 ? make_idesc_bf16(256, n2) : 0u;
        for (int kb = 0; kb < KB; ++kb) {
          const int s = kb % p.stages;
          const uint32_t ph = (kb / p.stages) & 1;
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + s * stage_bytes);
          const uint64_t ad = make_sdesc_sw128(a_addr, 16, 1024);
          const uint64_t bd0 = make_sdesc_sw128(a_addr + a_bytes, 16, 1024);
          const uint64_t bd1 = bd0 + uint64_t(((n1 / 2) * 128) >> 4);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
            const uint64_t ko = uint64_t((k * 32) >> 4);
            umma_bf16_pair(tmem, ad + ko, bd0 + ko, id0, acc);
            if (n2 > 0) umma_bf16_pair(tmem + uint32_t(n1), ad + ko, bd1 + ko, id1, acc);
          }
          umma_commit_pair_mc(&empty_bar[s], pmask);
        }
        umma_commit_pair_mc(&tmem_full_bar, pmask);
      }
    } else if (elect_one()) {
      const int nc0 = min(n_pad, 256);
      const int nc1 = n_pad - nc0;
      const uint32_t id0 = make_idesc_bf16(128, nc0);
      const uint32_t id1 = nc1 > 0 ? make_idesc_bf16(128, nc1) : 0u;
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % p.stages;
        const uint32_t ph = (kb / p.stages) & 1;
        mbar_wait(&full_bar[s], ph);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(smem + s * stage_bytes);
        const uint32_t b_addr = a_addr + a_bytes;
        // descriptors built once per stage and advanced by constants (keeps
        // the single issuing thread ahead of the tensor pipe)
        const uint64_t ad = make_sdesc_sw128(a_addr, 16, 1024);
        const uint64_t bd0 = make_sdesc_sw128(b_addr, 16, 1024);
        const uint64_t bd1 = bd0 + uint64_t((256 * 128) >> 4);
        const uint64_t au = ad + uint64_t(kTileBytesA >> 4);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
          const uint64_t ko = uint64_t((k * 32) >> 4);
          umma_bf16(tmem, ad + ko, bd0 + ko, id0, acc);
          if (nc1 > 0) umma_bf16(tmem + 256, ad + ko, bd1 + ko, id1, acc);
          if (swiglu) umma_bf16(tmem + 256, au + ko, bd0 + ko, id0, acc);
        }
        if (cs > 1) umma_commit_mc(&empty_bar[s], cmask);
        else umma_commit(&empty_bar[s]);
      }
      umma_commit(&tmem_full_bar);
    }
  } else {
    // ---- epilogue: warps 2..5 own TMEM lane quarters (warp % 4) ----
    const int q = warp & 3;
    const int row = q * 32 + lane;  // weight row within the tile
    const int n = nb * 128 + row;   // output feature
    mbar_wait(&tmem_full_bar, 0);
    tc_fence_after();
    const uint32_t trow = tmem + (uint32_t(q * 32) << 16);
    if (p.epilogue == SMO_EPI_ARGMAX) {
      // All MMAs are done: the stage ring is free scratch, [32 tokens][129] f32
      // (padded so both the column writes and the row scans are conflict-free).
      float* scratch = reinterpret_cast<float*>(smem);
      for (int c0 = 0; c0 < n_pad; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(trow + c0, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) scratch[j * 129 + row] = __uint_as_float(r[j]);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp == 2 && c0 + lane < cnt) {
          // ties resolve to the lowest vocabulary index (strict >)
          float best = scratch[lane * 129];
          int bi = 0;
          for (int i = 1; i < 128; ++i) {
            const float v = scratch[lane * 129 + i];
            if (v > best) { best = v; bi = i; }
          }
          const size_t at = size_t(row0 + c0 + lane) * p.n_tiles + nb;
          p.amax_val[at] = best;
          p.amax_idx[at] = nb * 128 + bi;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    } else {
      for (int c0 = 0; c0 < n_pad; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(trow + c0, r);
        if (swiglu) {
          uint32_t u[32];
          tmem_ld32(trow + 256 + c0, u);
          tmem_ld_wait();
          uint16_t* out = reinterpret_cast<uint16_t*>(p.out);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (c0 + j < cnt) {
              const float gv = __uint_as_float(r[j]);
              const float hv = gv / (1.0f + __expf(-gv)) * __uint_as_float(u[j]);
              out[size_t(row0 + c0 + j) * p.ldo + n] = f2bf(hv);
            }
          }
        } else {
          tmem_ld_wait();
          if (p.csplit) {  // fp32 partial of this K slice into this CTA's smem, token-major [cnt][128]
            float* P = reinterpret_cast<float*>(smem);
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (c0 + j < cnt) P[(c0 + j) * 128 + row] = __uint_as_float(r[j]);
          } else if (p.split_k > 1) {  // fp32 partial of this K slice; reduced in fixed order later
            float* part = p.partial + size_t(ks) * p.rows * p.N;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (c0 + j < cnt) part[size_t(row0 + c0 + j) * p.N + n] = __uint_as_float(r[j]);
          } else if (p.epilogue == SMO_EPI_BF16) {
            uint16_t* out = reinterpret_cast<uint16_t*>(p.out);
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (c0 + j < cnt) out[size_t(row0 + c0 + j) * p.ldo + n] = f2bf(__uint_as_float(r[j]));
          } else if (p.epilogue == SMO_EPI_F32) {
            float* out = reinterpret_cast<float*>(p.out);
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (c0 + j < cnt) out[size_t(row0 + c0 + j) * p.ldo + n] = __uint_as_float(r[j]);
          } else {  // SMO_EPI_F32_ADD: all loads first, then the stores (no
                    // load-after-store serialisation through possible aliasing)
            float* out = reinterpret_cast<float*>(p.out);
            float cur[32];
#pragma unroll
            for (int j = 0; j < 32; ++j)
              cur[j] = (c0 + j < cnt) ? __ldcg(out + size_t(row0 + c0 + j) * p.ldo + n) : 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (c0 + j < cnt) out[size_t(row0 + c0 + j) * p.ldo + n] = cur[j] + __uint_as_float(r[j]);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kPair) cluster_sync_all();  // both CTAs done with the pair's TMEM
  if (warp == 1) {
    if constexpr (kPair) tmem_dealloc_pair_dyn(tmem_cols, tmem);
    else tmem_dealloc_dyn(tmem_cols, tmem);
  }
  if (cs > 1) cluster_sync_all();  // peers' last commits may still arrive on our barriers
  if (p.csplit) {
    // Split-K reduce through distributed shared memory: every CTA of the
    // cluster holds its K slice's fp32 tile [cnt][128] in its (now idle)
    // smem ring; after one cluster barrier CTA ks reduces tokens
    // [ks cnt / S, (ks + 1) cnt / S) over the S slices in slice order
    // (deterministic, = the partial-buffer path's sum) and applies the
    // epilogue; a second barrier keeps every slice alive until read.
    const int S = p.split_k;
    cluster_sync_all();
    const int t0 = ks * cnt / S, t1 = (ks + 1) * cnt / S;
    const uint32_t pbase = smem_u32(smem);
    const bool vec = (reinterpret_cast<uintptr_t>(p.out) & 15) == 0 && (p.ldo & 3) == 0;  // 16-B rows of 4
    for (int idx = threadIdx.x; idx < (t1 - t0) * 32; idx += kThreads) {
      const int t = t0 + idx / 32, c4 = idx % 32;
      const uint32_t off = uint32_t((t * 128 + 4 * c4) * 4);
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int j = 0; j < S; ++j) {
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(pbase + off), "r"(kPair ? int(pr) + 2 * j : j));
        float4 v;
        asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(ra) : "memory");
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
      const size_t o = size_t(row0 + t) * p.ldo + size_t(nb) * 128 + 4 * c4;
      if (p.epilogue == SMO_EPI_BF16) {
        uint16_t* dst = reinterpret_cast<uint16_t*>(p.out) + o;
        if (vec) {
          *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16x2(acc.x, acc.y), pack_bf16x2(acc.z, acc.w));
        } else {
          dst[0] = f2bf(acc.x);
          dst[1] = f2bf(acc.y);
          dst[2] = f2bf(acc.z);
          dst[3] = f2bf(acc.w);
        }
      } else {
        float* dst = reinterpret_cast<float*>(p.out) + o;
        if (p.epilogue == SMO_EPI_F32_ADD) {
          acc.x += dst[0];
          acc.y += dst[1];
          acc.z += dst[2];
          acc.w += dst[3];
        }
        if (vec) {
          *reinterpret_cast<float4*>(dst) = acc;
        } else {
          dst[0] = acc.x;
          dst[1] = acc.y;
          dst[2] = acc.z;
          dst[3] = acc.w;
        }
      }
    }
    cluster_sync_all();
  }
}

// Fixed-order split-K reduction fused with the epilogue: out = epi(sum_s P_s).
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int splits, int rows, int N, int epilogue,
                                     void* out, int64_t ldo) {
  const size_t total4 = size_t(rows) * N / 4;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total4; i += size_t(gridDim.x) * blockDim.x) {
    const size_t e = i * 4;
    const int r = int(e / N), c = int(e % N);
    float4 acc = reinterpret_cast<const float4*>(part)[i];
    for (int s = 1; s < splits; ++s) {
      const float4 v = reinterpret_cast<const float4*>(part + size_t(s) * rows * N)[i];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    if (epilogue == SMO_EPI_BF16) {
      uint16_t* o = reinterpret_cast<uint16_t*>(out) + size_t(r) * ldo + c;
      *reinterpret_cast<uint2*>(o) = make_uint2(pack_bf16x2(acc.x, acc.y), pack_bf16x2(acc.z, acc.w));
    } else {
      float* o = reinterpret_cast<float*>(out) + size_t(r) * ldo + c;
      if (epilogue == SMO_EPI_F32_ADD) {
        const float4 cur = *reinterpret_cast<float4*>(o);
        acc.x += cur.x;
        acc.y += cur.y;
        acc.z += cur.z;
        acc.w += cur.w;
      }
      *reinterpret_cast<float4*>(o) = acc;
    }
  }
}

void set_gemm_smem_attr() {
  static bool attr_set = false;
  if (!attr_set) {
    SMO_CUDA_CHECK(cudaFuncSetAttribute(gemm_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        kSmemBudget + 4096));
    SMO_CUDA_CHECK(cudaFuncSetAttribute(gemm_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        kSmemBudget + 4096));
    attr_set = true;
  }
}

// clusters of (cx, 1, cz) CTAs of gemm_tc_kernel<kPair> resident at once (-1: none / error)
template <bool kPair>
int gemm_cluster_fit(int cx, int cz, int smem_bytes) {
  set_gemm_smem_attr();
  cudaLaunchConfig_t q{};
  q.gridDim = dim3(unsigned(cx), 1, unsigned(cz));
  q.blockDim = dim3(kThreads);
  q.dynamicSmemBytes = size_t(smem_bytes);
  cudaLaunchAttribute qa[1];
  qa[0].id = cudaLaunchAttributeClusterDimension;
  qa[0].val.clusterDim.x = unsigned(cx);
  qa[0].val.clusterDim.y = 1;
  qa[0].val.clusterDim.z = unsigned(cz);
  q.attrs = qa;
  q.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, gemm_tc_kernel<kPair>, &q) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    return -1;
  }
  return n;
}

int device_sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

struct GemmPlan {
  int tile, token_tiles, stages, split, cluster;
  bool csplit;  // split-K reduced through DSMEM inside a (pair ? 2 : 1, 1, split) cluster
  bool pair;    // CTA pairs (cta_group::2, M = 256)
  uint32_t cols;
};

// Dense projections as CTA pairs (see the kernel): tokens in tiles of up to
// 512 rounded to 64, each CTA stages half of them; K split over clusters of
// (2, 1, split) reduced through DSMEM when the clusters fit one wave.
bool plan_pair(const smo_gemm_args& a, GemmPlan& pl) {
  const bool swiglu = a.epilogue == SMO_EPI_SWIGLU;
  const int per_group = a.max_rows_per_group > 0 ? std::min(a.max_rows_per_group, a.rows) : a.rows;
  pl = GemmPlan{};
  if (a.groups == 1 && !a.row_offsets && !a.w_index && !swiglu && a.N % 256 == 0 &&
      !std::getenv("SMO_GEMM_CLUSTER")) {
    pl.pair = true;
    pl.cluster = 1;
    pl.tile = std::min(512, (per_group + 63) & ~63);
    pl.token_tiles = (per_group + pl.tile - 1) / pl.tile;
    const int sb = kTileBytesA + (pl.tile / 2) * 128;
    pl.stages = std::min(kMaxStages, kSmemBudget / sb);
    pl.cols = 32;
    while (int(pl.cols) < pl.tile) pl.cols <<= 1;
    const int pairs = (a.N / 256) * pl.token_tiles;
    pl.split = 1;
    pl.csplit = false;
    const bool splittable = a.epilogue == SMO_EPI_BF16 || a.epilogue == SMO_EPI_F32 || a.epilogue == SMO_EPI_F32_ADD;
    if (splittable && a.split_k != 1 && pl.tile * 128 * 4 <= pl.stages * sb) {
      const int want = a.split_k > 1 ? a.split_k : device_sm_count() / std::max(1, 2 * pairs);
      const int top = std::max(1, std::min({want, a.K / kBK / 8, 4}));
      for (int sp = top; sp >= (a.split_k > 1 ? top : 2); --sp) {
        const int n = gemm_cluster_fit<true>(2, sp, pl.stages * sb + 1024);
        if (n > 0 && pairs <= n) {
          pl.split = sp;
          pl.csplit = true;
          break;
        }
      }
    }
    // an explicit split the pair clusters cannot hold: the single-CTA plan
    if (a.split_k > 1 && pl.split != a.split_k) return false;
    return true;
  }
  return false;
}

GemmPlan plan_single(const smo_gemm_args& a);

// The pair plan where it launches at least as many CTAs as the single-CTA
// plan (same-box A/B, tools/gemm_ab.py: QKV 38.4 -> 35.8 us, LM head + argmax
// 117 -> 103 us; O-proj and the K = 14336 projection keep the single-CTA
// plan, whose split 4 fills more SMs than the pair's clusters of 6 or 8 can).
// SMO_GEMM_PAIR=0: never, =2: always when eligible.
GemmPlan plan_gemm(const smo_gemm_args& a) {
  static const int env_pair = [] {
    const char* f = std::getenv("SMO_GEMM_PAIR");
    return f ? std::atoi(f) : 1;
  }();
  const GemmPlan single = plan_single(a);
  GemmPlan pair;
  if (env_pair && plan_pair(a, pair)) {
    const long ps = 2L * (a.N / 256) * pair.token_tiles * pair.split;
    const long ss = long(a.N / 128) * a.groups * single.token_tiles * single.split;
    if (env_pair == 2 || ps >= ss) return pair;
  }
  return single;
}

GemmPlan plan_single(const smo_gemm_args& a) {
  const bool swiglu = a.epilogue == SMO_EPI_SWIGLU;
  const int per_group = a.max_rows_per_group > 0 ? std::min(a.max_rows_per_group, a.rows) : a.rows;
  GemmPlan pl{};
  const int cap = swiglu ? 256 : 512;
  pl.tile = std::min(cap, (per_group + 31) & ~31);
  pl.token_tiles = (per_group + pl.tile - 1) / pl.tile;
  const int stage_bytes = kTileBytesA * (swiglu ? 2 : 1) + pl.tile * 128;
  pl.stages = std::min(kMaxStages, kSmemBudget / stage_bytes);
  pl.cols = 32;
  const int need = swiglu ? 512 : pl.tile;
  while (int(pl.cols) < need) pl.cols <<= 1;
  // split K so that a dense GEMM with few weight tiles still covers the SMs;
  // only for plain fp32/bf16/residual epilogues (argmax/SwiGLU need full sums)
  pl.cluster = 1;
  pl.split = 1;
  const bool splittable = a.epilogue == SMO_EPI_BF16 || a.epilogue == SMO_EPI_F32 || a.epilogue == SMO_EPI_F32_ADD;
  const int tiles = (a.N / 128) * a.groups * pl.token_tiles;
  if (splittable && a.groups == 1 && a.split_k != 1 && (a.N % 512) == 0) {
    const int want = a.split_k > 1 ? a.split_k : device_sm_count() / std::max(1, tiles);
    pl.split = std::max(1, std::min({want, a.K / kBK / 8, 8}));
  }
  // Dense GEMMs can run as clusters of 2 or 4 weight tiles that share the
  // token rows by TMA multicast (SMO_GEMM_CLUSTER=2|4; the rows are otherwise
  // re-read from L2 by every weight tile: 2.25x the weight bytes per stage at
  // 288 tokens). Measured and left off: QKV 42 -> 65 us, O-proj 38 -> 40 us,
  // LM head unchanged (tools/kbench.py gemm) — the lockstep of the cluster's
  // stage release costs more than the L2 reads it saves.
  static const int env_cluster = [] {
    const char* f = std::getenv("SMO_GEMM_CLUSTER");
    return f ? std::atoi(f) : 1;
  }();
  static const int env_csplit = [] {
    const char* f = std::getenv("SMO_GEMM_CSPLIT");
    return f ? std::atoi(f) : 1;
  }();
  // the split-K partials reduce through DSMEM (SMO_GEMM_CSPLIT=0: fp32
  // partials in a workspace + a reduce launch) when a cluster of `split`
  // CTAs is portable, the [tile][128] fp32 slice fits the smem ring, and
  // every cluster is resident in one wave (a GPC holds a whole number of
  // clusters: 148 SMs do not take 48 clusters of 3). The automatic split
  // steps down until the clusters fit (QKV at 288 tokens: split 2 in
  // clusters, 38.9 us, beats split 3 with partials, 42.0 us).
  pl.csplit = false;
  const bool cs_ok = env_csplit && env_cluster <= 1 && pl.tile * 128 * 4 <= pl.stages * stage_bytes;
  auto fits = [&](int sp) {
    static int fit[9][kMaxStages + 1] = {};
    int& nfit = fit[sp][pl.stages];
    if (nfit == 0) nfit = gemm_cluster_fit<false>(1, sp, pl.stages * stage_bytes + 1024);
    return nfit > 0 && long(a.N / 128) * a.groups * pl.token_tiles <= nfit;
  };
  if (cs_ok && pl.split > 1 && pl.split <= 8) {
    for (int sp = pl.split; sp >= (a.split_k > 1 ? pl.split : 2); --sp)
      if (fits(sp)) {
        pl.split = sp;
        pl.csplit = true;
        break;
      }
  }
  if (a.groups == 1 && !a.row_offsets && env_cluster > 1) {
    const int nt = a.N / 128;
    for (int c : {4, 2})
      if (env_cluster == c && nt % c == 0 && (pl.tile / 32) >= c) {
        pl.cluster = c;
        break;
      }
  }
  return pl;
}

}  // namespace

size_t gemm_workspace(const smo_gemm_args& a) {
  const GemmPlan pl = plan_gemm(a);
  return pl.split > 1 && !pl.csplit ? size_t(pl.split) * a.rows * a.N * sizeof(float) : 0;
}

void gemm_launch(const smo_gemm_args& a, cudaStream_t stream) {
  SMO_REQUIRE(a.x && a.w, "gemm: null operand");
  SMO_REQUIRE(a.K > 0 && a.K % kBK == 0, "gemm: K must be a positive multiple of 64");
  SMO_REQUIRE(a.N > 0 && a.N % 128 == 0, "gemm: N must be a positive multiple of 128");
  SMO_REQUIRE(a.rows > 0 && a.groups > 0, "gemm: rows/groups must be positive");
  SMO_REQUIRE(a.groups == 1 || a.row_offsets, "gemm: grouped GEMM needs row_offsets");
  const bool swiglu = a.epilogue == SMO_EPI_SWIGLU;
  SMO_REQUIRE(!swiglu || a.w_up, "gemm: SWIGLU needs w_up");
  SMO_REQUIRE(a.epilogue != SMO_EPI_ARGMAX || (a.argmax_val && a.argmax_idx), "gemm: ARGMAX needs partial buffers");
  SMO_REQUIRE(a.epilogue == SMO_EPI_ARGMAX || a.out, "gemm: null output");
  const GemmPlan pl = plan_gemm(a);
  if (std::getenv("SMO_GEMM_DEBUG"))
    std::fprintf(stderr, "gemm rows=%d K=%d N=%d: pair=%d tile=%d tt=%d stages=%d split=%d csplit=%d\n", a.rows, a.K,
                 a.N, int(pl.pair), pl.tile, pl.token_tiles, pl.stages, pl.split, int(pl.csplit));
  const int tile = pl.tile, token_tiles = pl.token_tiles, stages = pl.stages;
  const uint32_t cols = pl.cols;
  SMO_REQUIRE(stages >= 2, "gemm: token tile too large for the smem ring");
  const size_t ws_need = pl.split > 1 && !pl.csplit ? size_t(pl.split) * a.rows * a.N * sizeof(float) : 0;
  SMO_REQUIRE(ws_need == 0 || (a.workspace && a.workspace_bytes >= ws_need),
              "gemm: split-K workspace too small (smo_gemm_workspace)");

  CUtensorMap tw, tu, tx;
  const int pool = std::max(1, a.w_pool_blocks);
  const uint64_t stride_blk = a.w_block_stride ? a.w_block_stride : uint64_t(a.N) * a.K * 2;
  {
    uint64_t dims[3] = {uint64_t(a.K), uint64_t(a.N), uint64_t(pool)};
    uint64_t strides[2] = {uint64_t(a.K) * 2, stride_blk};
    uint32_t box[3] = {uint32_t(kBK), 128, 1};
    make_tmap_bf16(&tw, a.w, 3, dims, strides, box, true);
    make_tmap_bf16(&tu, swiglu ? a.w_up : a.w, 3, dims, strides, box, true);
  }
  {
    uint64_t dims[2] = {uint64_t(a.K), uint64_t(a.rows)};
    uint64_t strides[1] = {uint64_t(a.K) * 2};
    uint32_t box[2] = {uint32_t(kBK), 32};
    make_tmap_bf16(&tx, a.x, 2, dims, strides, box, true);
  }
  GemmParams p{};
  p.K = a.K;
  p.N = a.N;
  p.rows = a.rows;
  p.row_offsets = a.row_offsets;
  p.w_index = a.w_index;
  p.tile_tokens = tile;
  p.stages = stages;
  p.epilogue = a.epilogue;
  p.out = a.out;
  p.ldo = a.ldo > 0 ? a.ldo : a.N;
  p.amax_val = a.argmax_val;
  p.amax_idx = a.argmax_idx;
  p.n_tiles = a.N / 128;
  p.split_k = pl.split;
  p.kb_per_split = (a.K / kBK + pl.split - 1) / pl.split;
  p.token_tiles = token_tiles;
  p.partial = reinterpret_cast<float*>(a.workspace);
  const int stage_bytes = kTileBytesA * (swiglu ? 2 : 1) + (pl.pair ? tile / 2 : tile) * 128;
  const size_t smem = size_t(stages) * stage_bytes + 1024;
  set_gemm_smem_attr();
  p.cluster = pl.cluster;
  p.csplit = pl.csplit ? 1 : 0;
  dim3 grid(a.N / 128, a.groups, token_tiles * pl.split);
  if (pl.pair) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = pl.csplit ? unsigned(pl.split) : 1u;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SMO_CUDA_CHECK(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<true>, tw, tu, tx, p, cols));
  } else if (pl.csplit) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = unsigned(pl.split);
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SMO_CUDA_CHECK(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<false>, tw, tu, tx, p, cols));
  } else if (pl.cluster > 1) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(pl.cluster);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SMO_CUDA_CHECK(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<false>, tw, tu, tx, p, cols));
  } else {
    gemm_tc_kernel<false><<<grid, kThreads, smem, stream>>>(tw, tu, tx, p, cols);
  }
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
  if (pl.split > 1 && !pl.csplit) {
    const size_t total4 = size_t(a.rows) * a.N / 4;
    const int blocks = int(std::min<size_t>((total4 + 255) / 256, size_t(device_sm_count()) * 8));
    splitk_reduce_kernel<<<blocks, 256, 0, stream>>>(p.partial, pl.split, a.rows, a.N, a.epilogue, a.out, p.ldo);
    count_launch();
    SMO_CUDA_CHECK(cudaGetLastError());
  }
}

}  // namespace smo
