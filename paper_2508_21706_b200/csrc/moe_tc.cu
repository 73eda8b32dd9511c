// moe_tc.cu — K4-MoE: the whole expert block of one layer (grouped SwiGLU
// gate/up, then the down projection) as ONE persistent tcgen05 kernel.
//
// Why: as two grouped GEMMs each CTA streams one 128-row weight tile of one
// expert (2 MB gate/up, 3.7 MB down for Mixtral); 896 gate/up tiles are 6.05
// waves of 148 SMs and 256 down tiles 1.7 waves, so the last wave of each
// kernel runs on a few SMs (ncu: SMs active 85 % of the gate/up kernel, 0.76
// of HBM). Here one cooperative grid of one CTA per SM walks a single unit
// list — every gate/up tile (expert-major), then every down tile split into
// S K slices (S = 1, 2 or 4 by a waves model) — round robin, so the down
// units of early experts fill the gate/up tail and the grid drains on
// small units.
//
// Dependencies: a down unit of expert e reads rows of H written by the
// SwiGLU epilogues of e's gate/up units (other CTAs). Each gate/up epilogue
// publishes with a release fence + atomicAdd on done[e]; the down unit's TMA
// producer spins on done[e] (acquire), then orders the async-proxy reads
// after it (fence.proxy.async). Gate/up units precede down units in every
// CTA's sequence, so the waits always resolve (co-residency: cooperative
// launch, one CTA per SM).
//
// The down K slices land in y[0..S) (fp32); the combine (K3) adds them in
// slice order — deterministic, and expert parallelism packs the same sum, so
// EP stays bit-identical to one GPU (S depends only on the shapes).
//
// Per unit the warp roles are those of gemm_tc.cu (swap-AB: weight tile =
// 128-row A operand, tokens = MMA N <= 256): w0 TMA producer, w1 MMA issuer,
// w2..w5 epilogue (TMEM -> registers -> global). The smem ring runs
// continuously across units, so the producer prefetches the next unit's
// k-blocks while the epilogue drains the previous one (tmem_empty barrier).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "tcode.cuh"

namespace smo {

namespace {

constexpr int kThreads = 192;
constexpr int kBK = 64;
constexpr int kTileA = 128 * kBK * 2;                  // weight tile per k-block (16 KB)
constexpr int kTok = 256;                              // largest token tile (gate + up = 512 TMEM columns)
constexpr int kMaxE = 64;

struct MoeParams {
  int h, hi, E;
  const int32_t* offsets;  // [E+1] row offsets of the permuted (token, slot) pairs
  const int32_t* w_index;  // [E] pool block of each expert's [W1 | W3 | W2]
  uint16_t* hbuf;          // [rows, hi] bf16 SwiGLU activations
  float* y;                // [splits][rows, h] fp32 down partials, slice s over K in [s, s+1) * hi/splits
  size_t y_stride;         // rows * h
  int splits;
  int* done;               // [E] finished gate/up units (zero at launch)
  int dbg;                 // coded kernel A/B: 1 no decode, 2 no token loads, 4 no code loads
};

struct Unit {
  int down, e, row0, cnt, nb, ks;
};

struct Schedule {
  int nA, nB;           // units per token tile: hi/128 gate/up, splits*h/128 down
  int totalA, total;
  int splits, tok;      // down K slices, token tile of this variant
  int a_base[kMaxE + 1], b_base[kMaxE + 1];
  int off[kMaxE + 1];
};

__device__ __forceinline__ Unit unit_at(const Schedule& S, int u) {
  Unit x{};
  if (u < S.totalA) {
    int e = 0;
    while (S.a_base[e + 1] <= u) ++e;
    const int v = u - S.a_base[e];
    x.down = 0;
    x.e = e;
    x.row0 = S.off[e] + (v / S.nA) * S.tok;
    x.nb = v % S.nA;
    x.ks = 0;
  } else {
    const int w = u - S.totalA;
    int e = 0;
    while (S.b_base[e + 1] <= w) ++e;
    const int v = w - S.b_base[e];
    x.down = 1;
    x.e = e;
    x.row0 = S.off[e] + (v / S.nB) * S.tok;
    const int r = v % S.nB;
    x.nb = r / S.splits;
    x.ks = r % S.splits;
  }
  x.cnt = min(S.tok, S.off[x.e + 1] - x.row0);
  return x;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Warps 2..5 of both expert kernels: per unit, wait for the accumulators,
// then SwiGLU -> H (gate/up units; publish with a release + done[e]) or the
// fp32 down partial -> y[ks]; hand TMEM back to the MMA warp.
template <int kCols>  // TMEM columns per load (16 under register pressure)
__device__ __forceinline__ void epilogue_loop(const Schedule& S, const MoeParams& p, uint32_t tmem, int warp, int lane,
                                              uint64_t& tmem_full, uint64_t& tmem_empty) {
  const int q = warp & 3;
  const int row = q * 32 + lane;  // weight row within the 128-row tile
  const uint32_t trow = tmem + (uint32_t(q * 32) << 16);
  int it = 0;
  for (int u = blockIdx.x; u < S.total; u += gridDim.x, ++it) {
    const Unit x = unit_at(S, u);
    const int n_pad = (x.cnt + 15) & ~15;
    if (kCols == 16) mbar_wait_backoff(&tmem_full, it & 1, 256);  // coded kernel: leave the issue slots to the decoders
    else mbar_wait(&tmem_full, it & 1);
    tc_fence_after();
    if (!x.down) {
      const int n = x.nb * 128 + row;  // intermediate feature
      for (int c0 = 0; c0 < n_pad; c0 += kCols) {
        uint32_t g[kCols], v[kCols];
        if constexpr (kCols == 32) {
          tmem_ld32(trow + c0, g);
          tmem_ld32(trow + 256 + c0, v);
        } else {
          tmem_ld16(trow + c0, g);
          tmem_ld16(trow + 256 + c0, v);
        }
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < kCols; ++j)
          if (c0 + j < x.cnt) {
            const float gv = __uint_as_float(g[j]);
            p.hbuf[size_t(x.row0 + c0 + j) * p.hi + n] = f2bf(gv / (1.0f + __expf(-gv)) * __uint_as_float(v[j]));
          }
      }
      __threadfence();  // release this unit's H rows before the count
    } else {
      const int n = x.nb * 128 + row;  // output feature
      float* y = p.y + size_t(x.ks) * p.y_stride;
      for (int c0 = 0; c0 < n_pad; c0 += kCols) {
        uint32_t r[kCols];
        if constexpr (kCols == 32) tmem_ld32(trow + c0, r);
        else tmem_ld16(trow + c0, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < kCols; ++j)
          if (c0 + j < x.cnt) y[size_t(x.row0 + c0 + j) * p.h + n] = __uint_as_float(r[j]);
      }
    }
    tc_fence_before();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (warp == 2 && lane == 0) {
      if (!x.down) {
        __threadfence();
        atomicAdd(p.done + x.e, 1);
      }
      mbar_arrive(&tmem_empty);
    }
  }
}

// The last CTA to finish zeroes the counters for the next launch (every
// wait on them is over: all other CTAs have exited their unit loops).
__device__ __forceinline__ void reset_done(const MoeParams& p) {
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(p.done + kMaxE, 1) == int(gridDim.x) - 1) {
      for (int e = 0; e < p.E; ++e) atomicExch(p.done + e, 0);
      atomicExch(p.done + kMaxE, 0);
    }
  }
}

__device__ __forceinline__ void init_schedule(Schedule& S, const MoeParams& p, int tok) {
  S.nA = p.hi / 128;
  S.splits = p.splits;
  S.tok = tok;
  S.nB = p.splits * (p.h / 128);
  S.a_base[0] = S.b_base[0] = 0;
  for (int e = 0; e < p.E; ++e) {
    S.off[e] = p.offsets[e];
    const int cnt = p.offsets[e + 1] - p.offsets[e];
    const int tt = (cnt + tok - 1) / tok;
    S.a_base[e + 1] = S.a_base[e] + tt * S.nA;
    S.b_base[e + 1] = S.b_base[e] + tt * S.nB;
  }
  S.off[p.E] = p.offsets[p.E];
  S.totalA = S.a_base[p.E];
  S.total = S.totalA + S.b_base[p.E];
}

// kSub k-blocks of 64 per pipeline stage (kSub = 2: each weight row is read
// 256 contiguous bytes at a time), kTokT-row token tiles, kStagesT stages.
template <int kSub, int kTokT, int kStagesT>
__global__ void __launch_bounds__(kThreads, 1)
    moe_fused_kernel(const __grid_constant__ CUtensorMap tm_w1, const __grid_constant__ CUtensorMap tm_w3,
                     const __grid_constant__ CUtensorMap tm_w2, const __grid_constant__ CUtensorMap tm_x,
                     const __grid_constant__ CUtensorMap tm_h, MoeParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int kStages = kStagesT;
  constexpr int kXBytes = kTokT * 128;                              // one k-block of token rows
  constexpr int kStageBytes = kSub * (2 * kTileA + kXBytes);
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ __align__(8) uint64_t tmem_full, tmem_empty;
  __shared__ uint32_t tmem_base_sh;
  __shared__ Schedule S;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    init_schedule(S, p, kTokT);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&tmem_full, 1);
    mbar_init(&tmem_empty, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tm_w1);
    tma_prefetch_desc(&tm_w3);
    tma_prefetch_desc(&tm_w2);
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_h);
  }
  if (warp == 1) tmem_alloc<512>(&tmem_base_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const int KBa = p.h / (kBK * kSub);                 // gate/up stages per unit
  const int KBd = (p.hi / (kBK * kSub)) / p.splits;   // stages per down slice

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      int kbg = 0;
      for (int u = blockIdx.x; u < S.total; u += gridDim.x) {
        const Unit x = unit_at(S, u);
        const int wblk = p.w_index[x.e];
        const int n_load = (x.cnt + 31) & ~31;
        if (x.down) {
          // every gate/up unit of expert e has published its H rows
          const int need = ((S.off[x.e + 1] - S.off[x.e] + kTokT - 1) / kTokT) * S.nA;
          while (ld_acquire(p.done + x.e) < need) {
          }
          fence_proxy_async_global();
        }
        const int KB = x.down ? KBd : KBa;
        const int kb0 = x.down ? x.ks * KBd : 0;
        const uint32_t tx = uint32_t(kSub * ((x.down ? kTileA : 2 * kTileA) + (n_load / 32) * 4096));
        for (int kb = 0; kb < KB; ++kb, ++kbg) {
          const int s = kbg % kStages;
          mbar_wait(&empty_bar[s], ((kbg / kStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&full_bar[s], tx);
          uint8_t* sa = smem + s * kStageBytes;
          // stage layout: W1 (or W2) sub-tiles, W3 sub-tiles, token sub-tiles
#pragma unroll
          for (int j = 0; j < kSub; ++j) {
            const int kc = ((kb0 + kb) * kSub + j) * kBK;
            uint8_t* sb = sa + 2 * kSub * kTileA + j * kXBytes;
            if (x.down) {
              tma_load_3d(sa + j * kTileA, &tm_w2, &full_bar[s], kc, x.nb * 128, wblk);
              for (int i = 0; i < n_load / 32; ++i) tma_load_2d(sb + i * 4096, &tm_h, &full_bar[s], kc, x.row0 + i * 32);
            } else {
              tma_load_3d(sa + j * kTileA, &tm_w1, &full_bar[s], kc, x.nb * 128, wblk);
              tma_load_3d(sa + (kSub + j) * kTileA, &tm_w3, &full_bar[s], kc, x.nb * 128, wblk);
              for (int i = 0; i < n_load / 32; ++i) tma_load_2d(sb + i * 4096, &tm_x, &full_bar[s], kc, x.row0 + i * 32);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      int kbg = 0, it = 0;
      for (int u = blockIdx.x; u < S.total; u += gridDim.x, ++it) {
        const Unit x = unit_at(S, u);
        const int n_pad = (x.cnt + 15) & ~15;
        const uint32_t idesc = make_idesc_bf16(128, n_pad);
        const int KB = x.down ? KBd : KBa;
        // the epilogue has drained the accumulators of the previous unit
        mbar_wait(&tmem_empty, (it & 1) ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < KB; ++kb, ++kbg) {
          const int s = kbg % kStages;
          mbar_wait(&full_bar[s], (kbg / kStages) & 1);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + s * kStageBytes);
#pragma unroll
          for (int j = 0; j < kSub; ++j) {
            const uint64_t ad = make_sdesc_sw128(a_addr + j * kTileA, 16, 1024);
            const uint64_t au = make_sdesc_sw128(a_addr + (kSub + j) * kTileA, 16, 1024);
            const uint64_t bd = make_sdesc_sw128(a_addr + 2 * kSub * kTileA + j * kXBytes, 16, 1024);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint32_t acc = (kb > 0 || j > 0 || k > 0) ? 1u : 0u;
              const uint64_t ko = uint64_t((k * 32) >> 4);
              umma_bf16(tmem, ad + ko, bd + ko, idesc, acc);
              if (!x.down) umma_bf16(tmem + 256, au + ko, bd + ko, idesc, acc);
            }
          }
          umma_commit(&empty_bar[s]);
        }
        umma_commit(&tmem_full);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    epilogue_loop<32>(S, p, tmem, warp, lane, tmem_full, tmem_empty);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
  reset_done(p);
}

// ---------------------------------------------------------------------------
// K4-MoE on T2-coded experts (tcode.cuh): the same unit schedule, MMA and
// epilogue, but the weight tiles arrive in their link code and are expanded
// inside the kernel — no bf16 copy of the expert ever reaches HBM.
//   w0      code producer: bulk copies (cp.async.bulk) of the k-block's coded
//           tiles (W1 + W3, or W2) into a code ring of kCS stages
//   w1      MMA issuer (as above)
//   w2..w5  epilogue (as above)
//   w6..    kND decoder warps: warp d decodes segment d (16 rows) of each
//           coded tile of the stage into the 128B-swizzled A tile, orders its
//           shared-memory stores for the tensor core (fence.proxy.async) and
//           arrives on a_full; decoder 0 also issues the stage's token-row
//           TMA loads (and, for down units, first acquires done[e])
// The A ring (kAS stages of W1 | W3 | token rows) is released by the MMA
// commit, the code ring by the kND decoder arrivals.
constexpr int kCodeSlot = tcode::kTileMax;  // 16416 B: the largest tile code

// Down units with <= 128 token rows take two W2 k-blocks per stage (both code
// slots and both halves of the token region are free), so all decoder warps
// have a segment in every stage.
__device__ __forceinline__ bool down_pair(const Unit& x, int KBd) {
  return x.down && x.cnt <= 128 && (KBd % 2) == 0;
}

// kTS: stages of the token-row ring, fed by its own TMA warp (w6) so the
// token loads run kTS stages ahead of the MMA instead of waiting for the
// decoded weight stage to be released (decoder warps are w7..).
template <int kND, int kAS, int kCS, int kFmt = 2, int kTS = 2>  // kFmt: the tile code, T2 or T3 (tcode.cuh)
__global__ void __launch_bounds__(kThreads + 32 + 32 * kND, 1)
    moe_coded_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_h, MoeParams p,
                     const uint8_t* const* __restrict__ w_code) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int kXBytes = kTok * 128;
  constexpr int kAStage = 2 * kTileA;            // W1 (or W2) | W3, decoded
  uint8_t* tring = smem + kAS * kAStage;         // kTS x token rows
  uint8_t* cring = tring + kTS * kXBytes;        // kCS x (2 tile codes)
  __shared__ __align__(8) uint64_t a_full[kAS], a_empty[kAS], c_full[kCS], c_empty[kCS], t_full[kTS], t_empty[kTS];
  __shared__ __align__(8) uint64_t tmem_full, tmem_empty;
  __shared__ uint32_t tmem_base_sh;
  __shared__ Schedule S;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    init_schedule(S, p, kTok);
    for (int s = 0; s < kAS; ++s) {
      mbar_init(&a_full[s], kND);  // the kND decoder warps
      mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < kTS; ++s) {
      mbar_init(&t_full[s], 1);  // the token warp's expect_tx
      mbar_init(&t_empty[s], 1);
    }
    for (int s = 0; s < kCS; ++s) {
      mbar_init(&c_full[s], 1);
      mbar_init(&c_empty[s], kND);
    }
    mbar_init(&tmem_full, 1);
    mbar_init(&tmem_empty, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_h);
  }
  if (warp == 1) tmem_alloc<512>(&tmem_base_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  const int KBa = p.h / kBK;                     // gate/up k-blocks per unit
  const int KBd = (p.hi / kBK) / p.splits;       // k-blocks per down slice
  const int tiles = (p.h / 128) * (p.hi / kBK);  // tiles per matrix

  if (warp == 0) {
    // ------------------------------------------------------------ code producer
    // The whole warp reads the unit's tile offsets 32 tiles at a time
    // (coalesced; consecutive tiles of a unit are contiguous in the code, so
    // tile i ends where i + 1 starts) and lane 0 issues the bulk copies: a
    // stage holds W1 + W3 tile kb (gate/up), W2 tiles kb, kb + 1 (paired down
    // units) or W2 tile kb.
    int g = 0;
    for (int u = blockIdx.x; u < S.total; u += gridDim.x) {
      const Unit x = unit_at(S, u);
      const uint8_t* blk = w_code[x.e];
      const uint32_t* toff = reinterpret_cast<const uint32_t*>(blk);
      const int KB = x.down ? KBd : KBa;
      const int kb0 = x.down ? x.ks * KBd : 0;
      const bool pair = down_pair(x, KBd);
      // tile (matrix, row tile, k-block): W1 / W3 rows of h_i (h / 64 k-blocks), W2 rows of h (h_i / 64)
      const int t0 = x.down ? 2 * tiles + x.nb * (p.hi / kBK) + kb0 : x.nb * (p.h / kBK);
      for (int c0 = 0; c0 < KB; c0 += 32) {
        const int nc = min(32, KB - c0);
        const uint32_t a = lane < nc ? toff[t0 + c0 + lane] : 0u, a_end = toff[t0 + c0 + nc];
        const uint32_t b = (!x.down && lane < nc) ? toff[tiles + t0 + c0 + lane] : 0u;
        const uint32_t b_end = x.down ? 0u : toff[tiles + t0 + c0 + nc];
        for (int k = 0; k < nc; k += pair ? 2 : 1, ++g) {
          auto at = [&](uint32_t v, uint32_t end, int i) {
            const uint32_t r = __shfl_sync(0xffffffffu, v, i & 31);
            return i < nc ? r : end;
          };
          const uint32_t a0 = at(a, a_end, k), a1 = at(a, a_end, k + 1), a2 = at(a, a_end, k + 2);
          const uint32_t b0 = at(b, b_end, k), b1 = at(b, b_end, k + 1);
          if (lane == 0) {
            const int s = g % kCS;
            mbar_wait(&c_empty[s], ((g / kCS) & 1) ^ 1);
            uint8_t* dst = cring + size_t(s) * 2 * kCodeSlot;
            if (p.dbg & 4) {
              mbar_arrive(&c_full[s]);
            } else if (pair) {
              mbar_arrive_expect_tx(&c_full[s], a2 - a0);
              bulk_load(dst, blk + a0, a1 - a0, &c_full[s]);
              bulk_load(dst + kCodeSlot, blk + a1, a2 - a1, &c_full[s]);
            } else {
              mbar_arrive_expect_tx(&c_full[s], (a1 - a0) + (x.down ? 0u : b1 - b0));
              bulk_load(dst, blk + a0, a1 - a0, &c_full[s]);
              if (!x.down) bulk_load(dst + kCodeSlot, blk + b0, b1 - b0, &c_full[s]);
            }
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      int g = 0, it = 0;
      for (int u = blockIdx.x; u < S.total; u += gridDim.x, ++it) {
        const Unit x = unit_at(S, u);
        const int n_pad = (x.cnt + 15) & ~15;
        const uint32_t xb = uint32_t(((x.cnt + 31) & ~31) * 128);  // token rows of one k-block
        const uint32_t idesc = make_idesc_bf16(128, n_pad);
        const bool pair = down_pair(x, KBd);
        const int KS = x.down ? (pair ? KBd / 2 : KBd) : KBa;
        mbar_wait(&tmem_empty, (it & 1) ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < KS; ++kb, ++g) {
          const int s = g % kAS, ts = g % kTS;
          mbar_wait(&t_full[ts], (g / kTS) & 1);
          mbar_wait(&a_full[s], (g / kAS) & 1);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + s * kAStage);
          const uint32_t t_addr = smem_u32(tring + ts * kXBytes);
          const uint64_t ad = make_sdesc_sw128(a_addr, 16, 1024);
          const uint64_t au = make_sdesc_sw128(a_addr + kTileA, 16, 1024);
          const uint64_t bd = make_sdesc_sw128(t_addr, 16, 1024);
          const uint64_t bd2 = make_sdesc_sw128(t_addr + xb, 16, 1024);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
            const uint64_t ko = uint64_t((k * 32) >> 4);
            umma_bf16(tmem, ad + ko, bd + ko, idesc, acc);
            if (!x.down) umma_bf16(tmem + 256, au + ko, bd + ko, idesc, acc);
          }
          if (pair) {  // second k-block of the stage: W2 tile kb + 1 with its token rows
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint64_t ko = uint64_t((k * 32) >> 4);
              umma_bf16(tmem, au + ko, bd2 + ko, idesc, 1u);
            }
          }
          umma_commit(&a_empty[s]);
          umma_commit(&t_empty[ts]);
        }
        umma_commit(&tmem_full);
      }
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ epilogue
    epilogue_loop<(kND > 8 ? 16 : 32)>(S, p, tmem, warp, lane, tmem_full, tmem_empty);
  } else if (warp == 6) {
    // ------------------------------------------------------------ token rows
    // x rows (gate/up units) or H rows (down units, after every gate/up unit
    // of the expert published them) of each stage's k-block(s), kTS stages ahead
    if (lane == 0) {
      int g = 0;
      for (int u = blockIdx.x; u < S.total; u += gridDim.x) {
        const Unit x = unit_at(S, u);
        const int n_load = (x.cnt + 31) & ~31;
        const bool pair = down_pair(x, KBd);
        const int KS = x.down ? (pair ? KBd / 2 : KBd) : KBa;
        const int kb0 = x.down ? x.ks * KBd : 0;
        if (x.down) {
          const int need = ((S.off[x.e + 1] - S.off[x.e] + kTok - 1) / kTok) * S.nA;
          while (ld_acquire(p.done + x.e) < need) {
          }
          fence_proxy_async_global();
        }
        for (int kb = 0; kb < KS; ++kb, ++g) {
          const int ts = g % kTS;
          mbar_wait(&t_empty[ts], ((g / kTS) & 1) ^ 1);
          uint8_t* tt = tring + ts * kXBytes;
          if (p.dbg & 2) {
            mbar_arrive(&t_full[ts]);
            continue;
          }
          const int nkb = pair ? 2 : 1;
          mbar_arrive_expect_tx(&t_full[ts], uint32_t(nkb * (n_load / 32) * 4096));
          for (int j = 0; j < nkb; ++j) {
            const int kc = (kb0 + kb * nkb + j) * kBK;
            for (int i = 0; i < n_load / 32; ++i)
              tma_load_2d(tt + j * n_load * 128 + i * 4096, x.down ? &tm_h : &tm_x, &t_full[ts], kc, x.row0 + i * 32);
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ decoders
    const int d = warp - 7;
    int g = 0;
    for (int u = blockIdx.x; u < S.total; u += gridDim.x) {
      const Unit x = unit_at(S, u);
      const bool pair = down_pair(x, KBd);
      const int KS = x.down ? (pair ? KBd / 2 : KBd) : KBa;
      const int ntile = (!x.down || pair) ? 2 : 1;
      for (int kb = 0; kb < KS; ++kb, ++g) {
        const int sa = g % kAS, sc = g % kCS;
        uint8_t* st = smem + sa * kAStage;
        mbar_wait(&a_empty[sa], ((g / kAS) & 1) ^ 1);
        mbar_wait(&c_full[sc], (g / kCS) & 1);
        const uint8_t* code = cring + size_t(sc) * 2 * kCodeSlot;
        if (!(p.dbg & 1)) {
          // kND = 8: warp d decodes segment d of each tile; kND = 16: warp d
          // segment d % 8 of tile d / 8 (single-tile stages: warps 0..7)
#pragma unroll 1
          for (int m = kND > 8 ? d / 8 : 0; m < ntile; m += kND > 8 ? 2 : 1)
            if constexpr (kFmt == 3)
              tcode::decode_segment3(code + m * kCodeSlot, st + m * kTileA, d % 8, lane);
            else
              tcode::decode_segment(code + m * kCodeSlot, st + m * kTileA, d % 8, lane, (p.dbg & 8) ? ~0xe00u : ~0u);
        }
        fence_proxy_async();  // the stores above feed the tensor core (async proxy)
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&c_empty[sc]);
          mbar_arrive(&a_full[sa]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
  reset_done(p);
}

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

}  // namespace

// Down-projection K splits for a launch: 1 unless the unit list would not
// cover the SMs once (small models), then the smallest S that does. Measured
// at config 2 (round 1): S = 1 / 2 / 4 -> 516 / 520 / 524 us — the grid is
// already 94 % busy (ncu sm__cycles_active), so finer down units buy less
// than their extra fp32 partial traffic. SMO_MOE_SPLITS overrides (A/B runs).
int pick_moe_splits(int rows, int h, int hi, int E, int max_splits) {
  const char* env = std::getenv("SMO_MOE_SPLITS");
  const int forced = env ? std::atoi(env) : 0;
  auto ok = [&](int sp) { return sp <= max_splits && (hi / kBK) % sp == 0; };
  if (forced > 0 && ok(forced)) return forced;
  const double tiles = std::max(1.0, std::ceil(double(rows) / E / kTok));  // token tiles per expert (even routing)
  for (int sp : {1, 2, 4}) {
    const double units = E * tiles * (hi / 128 + double(h / 128) * sp);
    if (ok(sp) && units >= sm_count()) return sp;
  }
  return ok(2) ? 2 : 1;
}

// Expert block of one layer: H = SwiGLU(x_perm W1^T, x_perm W3^T) per expert,
// sum_s y[s] = H W2^T (K split in `splits` slices; 0 = pick_moe_splits;
// returned). Callers that must reproduce another launch bit for bit (expert
// parallelism vs one GPU) pass the same explicit splits. done: >= 65 ints,
// zero before the first launch; the kernel leaves them zero. x_perm bf16
// [rows, h] grouped by offsets [E+1]; pool blocks [W1 | W3 | W2]
// (w_block_stride bytes apart), w_index [E]; y has room for max_splits
// slices of [rows, h].
int moe_launch(const void* x_perm, int rows, int h, int hi, int E, const int32_t* offsets, const void* pool,
               uint64_t w_block_stride, int pool_blocks, const int32_t* w_index, void* hbuf, float* y, int splits,
               int max_splits, int* done, cudaStream_t st) {
  SMO_REQUIRE(x_perm && offsets && pool && w_index && hbuf && y && done, "moe: null pointer");
  SMO_REQUIRE(E >= 1 && E <= kMaxE, "moe: 1 <= n_expert <= 64");
  SMO_REQUIRE(h % 128 == 0 && hi % 128 == 0, "moe: h and h_i must be multiples of 128");
  SMO_REQUIRE(rows > 0 && max_splits >= 1, "moe: no rows");
  if (splits <= 0) splits = pick_moe_splits(rows, h, hi, E, max_splits);
  SMO_REQUIRE(splits <= max_splits && (hi / kBK) % splits == 0, "moe: bad down split");
  const size_t wb = size_t(hi) * h * 2;  // one matrix of a block
  CUtensorMap t1, t3, t2, tx, th;
  {
    uint64_t dims[3] = {uint64_t(h), uint64_t(hi), uint64_t(pool_blocks)};
    uint64_t strides[2] = {uint64_t(h) * 2, w_block_stride};
    uint32_t box[3] = {uint32_t(kBK), 128, 1};
    make_tmap_bf16(&t1, pool, 3, dims, strides, box, true);
    make_tmap_bf16(&t3, reinterpret_cast<const uint8_t*>(pool) + wb, 3, dims, strides, box, true);
  }
  {
    uint64_t dims[3] = {uint64_t(hi), uint64_t(h), uint64_t(pool_blocks)};
    uint64_t strides[2] = {uint64_t(hi) * 2, w_block_stride};
    uint32_t box[3] = {uint32_t(kBK), 128, 1};
    make_tmap_bf16(&t2, reinterpret_cast<const uint8_t*>(pool) + 2 * wb, 3, dims, strides, box, true);
  }
  {
    uint64_t dims[2] = {uint64_t(h), uint64_t(rows)};
    uint64_t strides[1] = {uint64_t(h) * 2};
    uint32_t box[2] = {uint32_t(kBK), 32};
    make_tmap_bf16(&tx, x_perm, 2, dims, strides, box, true);
  }
  {
    uint64_t dims[2] = {uint64_t(hi), uint64_t(rows)};
    uint64_t strides[1] = {uint64_t(hi) * 2};
    uint32_t box[2] = {uint32_t(kBK), 32};
    make_tmap_bf16(&th, hbuf, 2, dims, strides, box, true);
  }
  MoeParams p{};
  p.h = h;
  p.hi = hi;
  p.E = E;
  p.offsets = offsets;
  p.w_index = w_index;
  p.hbuf = reinterpret_cast<uint16_t*>(hbuf);
  p.y = y;
  p.y_stride = size_t(rows) * h;
  p.splits = splits;
  p.done = done;
  // one k-block (64) per stage, 256-row token tiles, 3 stages of 64 KB. (Two
  // k-blocks per stage — 256 contiguous bytes per weight row per request,
  // 128-row tiles, 2 stages — measured 510 vs 516 us at config 2: not kept.)
  auto kern = moe_fused_kernel<1, kTok, 3>;
  const size_t smem = size_t(3) * (2 * kTileA + kTok * 128) + 1024;
  static bool attr_set = false;
  if (!attr_set) {
    SMO_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr_set = true;
  }
  // one CTA per SM, co-resident (cooperative): down units wait on gate/up
  // units of other CTAs
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(sm_count()));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SMO_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, t1, t3, t2, tx, th, p));
  count_launch();
  return splits;
}

// The expert block of one layer on T2-coded experts (tcode.cuh): w_code is a
// DEVICE array of E pointers to each expert's code block (16-B aligned, e.g.
// the streamed code slots and the coded hot cache). Same unit schedule,
// split and MMA order as moe_launch, so the outputs are bit-identical to
// moe_launch on the decoded weights.
int moe_coded_launch(const void* x_perm, int rows, int h, int hi, int E, const int32_t* offsets,
                     const void* const* w_code, void* hbuf, float* y, int splits, int max_splits, int* done,
                     cudaStream_t st, int fmt) {
  SMO_REQUIRE(fmt == 2 || fmt == 3, "moe: tile code format must be 2 (T2) or 3 (T3)");
  SMO_REQUIRE(x_perm && offsets && w_code && hbuf && y && done, "moe: null pointer");
  SMO_REQUIRE(E >= 1 && E <= kMaxE, "moe: 1 <= n_expert <= 64");
  SMO_REQUIRE(h % 128 == 0 && hi % 128 == 0, "moe: h and h_i must be multiples of 128");
  SMO_REQUIRE(rows > 0 && max_splits >= 1, "moe: no rows");
  if (splits <= 0) splits = pick_moe_splits(rows, h, hi, E, max_splits);
  SMO_REQUIRE(splits <= max_splits && (hi / kBK) % splits == 0, "moe: bad down split");
  CUtensorMap tx, th;
  {
    uint64_t dims[2] = {uint64_t(h), uint64_t(rows)};
    uint64_t strides[1] = {uint64_t(h) * 2};
    uint32_t box[2] = {uint32_t(kBK), 32};
    make_tmap_bf16(&tx, x_perm, 2, dims, strides, box, true);
  }
  {
    uint64_t dims[2] = {uint64_t(hi), uint64_t(rows)};
    uint64_t strides[1] = {uint64_t(hi) * 2};
    uint32_t box[2] = {uint32_t(kBK), 32};
    make_tmap_bf16(&th, hbuf, 2, dims, strides, box, true);
  }
  MoeParams p{};
  p.h = h;
  p.hi = hi;
  p.E = E;
  p.offsets = offsets;
  p.hbuf = reinterpret_cast<uint16_t*>(hbuf);
  p.y = y;
  p.y_stride = size_t(rows) * h;
  p.splits = splits;
  p.done = done;
  p.dbg = std::getenv("SMO_MOE_CODED_DBG") ? std::atoi(std::getenv("SMO_MOE_CODED_DBG")) : 0;
  // decoder warps / A stages / code stages (SMO_MOE_CODED=<nd>,<as>,<cs> for A/B runs)
  static int variant = [] {
    const char* f = std::getenv("SMO_MOE_CODED");
    if (f && std::strcmp(f, "8,2,2") == 0) return 1;
    if (f && std::strcmp(f, "16,2,2") == 0) return 2;
    if (f && std::strcmp(f, "8,2,3") == 0) return 3;
    return 0;
  }();
  void (*kern)(const CUtensorMap, const CUtensorMap, MoeParams, const uint8_t* const*) = nullptr;
  int nd = 0, as = 0, cs = 0;
  switch (variant) {
    case 1: kern = moe_coded_kernel<8, 2, 2>, nd = 8, as = 2, cs = 2; break;
    case 2: kern = moe_coded_kernel<16, 2, 2>, nd = 16, as = 2, cs = 2; break;
    case 3: kern = moe_coded_kernel<8, 2, 3>, nd = 8, as = 2, cs = 3; break;
    default: kern = moe_coded_kernel<16, 2, 2>, nd = 16, as = 2, cs = 2; break;
  }
  int slot = variant, ts = 2;
  if (fmt == 3) {  // T3: 16 decoder warps, 2 weight / 3 token / 2 code stages (SMO_MOE_CODED=8,2,2: 8 decoders)
    static const int t3v = [] {
      const char* f = std::getenv("SMO_MOE_CODED3");
      return f ? std::atoi(f) : 0;
    }();
    if (variant == 1) kern = moe_coded_kernel<8, 2, 2, 3, 3>, nd = 8, as = 2, cs = 2, ts = 3;
    else if (t3v == 1) kern = moe_coded_kernel<16, 3, 2, 3, 2>, nd = 16, as = 3, cs = 2, ts = 2;
    else kern = moe_coded_kernel<16, 2, 2, 3, 3>, nd = 16, as = 2, cs = 2, ts = 3;
    slot = variant == 1 ? 5 : t3v == 1 ? 6 : 4;
  }
  const size_t smem = size_t(as) * 2 * kTileA + size_t(ts) * kTok * 128 + size_t(cs) * 2 * kCodeSlot + 1024;
  static bool attr_set[7] = {false, false, false, false, false, false, false};
  if (!attr_set[slot]) {
    SMO_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr_set[slot] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(sm_count()));
  cfg.blockDim = dim3(unsigned(kThreads + 32 + 32 * nd));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SMO_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, tx, th, p, reinterpret_cast<const uint8_t* const*>(w_code)));
  count_launch();
  return splits;
}

}  // namespace smo
