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
//    items. The g*n query rows sharing KV head h (row = i*g + hh) are loaded
//    R = 128/(rows rounded up to 32/64/128) times into the M=128 Q tile (TMA
//    3D box {64, g, n}); a 128-key chunk of K is the B operand of
//    S = Q K^T (N=128) and replica k owns keys [k*128/R, (k+1)*128/R) of
//    each chunk. P (hi + lo bf16 planes) is written over its S buffer in TMEM
//    and O += P V reads A from TMEM, B = V (MN-major) from shared memory.
//  * warps: w0 TMA producer, w1 TMEM alloc + MMA issuer, w2..w9 softmax (two
//    warps per TMEM lane quadrant, each owning half of its replica's keys).
//  * TMEM: S/P triple buffer cols [0,384), O accumulator [384, 384+D).
//  * shared memory: Q tile(s) + kStages K/V chunk stages (224 KB); the K tile
//    of a consumed chunk doubles as the pair max-exchange buffer and the last
//    chunk's stage as the epilogue's replica-merge scratch.
//  * HBM-bound: algorithmic bytes = 2*b*(s+n)*n_kv*d*2 (roofline.hpp:88) +
//    Q/O; FLOPs = 4*n*(s+n)*n_q*d per request.
#include <cmath>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace smo {

namespace {

constexpr int kSoftWarps = 8;                 // two per TMEM lane quadrant
constexpr int kThreads = 64 + 32 * kSoftWarps;  // + TMA producer + MMA issuer
constexpr int kChunk = 128;
static_assert(kChunk == kKvPage, "a K/V page is one K1 key chunk");

struct AttnParams {
  const uint64_t* mask;
  const int32_t* prefix;
  uint16_t* out;
  float* ws_o;    // partial pieces [grid][2][rows][D] (unnormalised, replica-merged)
  float2* ws_ml;  // their (reference max, row sum) [grid][2][rows]
  int* ws_cnt;    // per (request, KV head) pieces-finished counter, zero between launches
  int b, n, n_q, n_kv, g, rows, s_max;
  const int32_t* bt;  // paged K/V block table [b][max_pages] (null: contiguous)
  int max_pages;
  int C;          // chunk slots per (request, KV head) = ceil((max_prefix + n) / 128)
  int Q;          // chunks per CTA of the flat schedule
  int total;      // pairs * C
  float scale_log2;
};

template <int D>
struct AttnSmem {
  static constexpr int kKBlocks = D / 64;
  static constexpr int kQBytes = kKBlocks * 16384;      // 128 rows x D
  static constexpr int kKvBytes = kKBlocks * 16384;     // 128 keys x D (K or V)
  static constexpr int kQBufs = D == 128 ? 1 : 2;
  static constexpr int kStages = D == 128 ? 3 : 6;      // K/V chunk stages in flight
  static constexpr int kQOff = 0;
  static constexpr int kKvOff = kQBufs * kQBytes;
  static constexpr int kTotal = kKvOff + kStages * 2 * kKvBytes;  // 224 KB
};

#ifdef SMO_ATTN_TRACE
// Debug timeline of CTA 0 (globaltimer ns << 8 | event code) per role; the
// event counters live in shared memory so a trace point costs no global
// round trip.
__device__ unsigned long long g_trace[3][4096];
__device__ int g_trace_n[3];
__shared__ int s_trace_n[3];
__device__ __forceinline__ void trace_ev(int role, int code) {
  if (blockIdx.x != 0) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  const int i = s_trace_n[role]++;
  if (i < 4096) g_trace[role][i] = (t << 8) | unsigned(code);
  g_trace_n[role] = i + 1;
}
#define TR(role, code) trace_ev(role, code)
#define TR_INIT() \
  if (threadIdx.x < 3) s_trace_n[threadIdx.x] = 0
#else
#define TR(role, code)
#define TR_INIT()
#endif

// Flat ("stream-K") schedule: the (pair, chunk) slots of all requests and KV
// heads are laid end to end and CTA i processes slots [i*Q, (i+1)*Q). The
// run of slots a CTA holds for one pair is a piece; a piece covering a whole
// pair writes the output, otherwise it leaves a partial (O, m, l) and, once
// all of the pair's pieces are published, each of them merges one slice of
// the output (in-kernel split-KV combine, after the CTA's last item).
struct Piece {
  int pair, r, h, c0, c1, keys;  // chunks [c0, c1) of pair (r, h); keys = prefix + n
  int first_cta, npieces;        // CTAs holding the pair's non-empty pieces
  int next_f;
};

__device__ __forceinline__ Piece piece_make(const AttnParams& p, int f, int f_end, int prefix) {
  Piece pc;
  pc.pair = f / p.C;
  const int c0 = f - pc.pair * p.C;
  const int span = min(p.C - c0, f_end - f);
  pc.next_f = f + span;
  pc.r = pc.pair / p.n_kv;
  pc.h = pc.pair % p.n_kv;
  pc.keys = prefix + p.n;
  const int A = min(p.C, (pc.keys + kChunk - 1) / kChunk);  // chunks this pair really has
  pc.c0 = c0;
  pc.c1 = min(c0 + span, A);
  const int base = pc.pair * p.C;
  pc.first_cta = base / p.Q;
  pc.npieces = (base + A - 1) / p.Q - pc.first_cta + 1;
  return pc;
}
__device__ __forceinline__ int piece_request(const AttnParams& p, int f) { return (f / p.C) / p.n_kv; }
__device__ __forceinline__ Piece piece_at(const AttnParams& p, int f, int f_end) {
  return piece_make(p, f, f_end, p.prefix[piece_request(p, f)]);
}

// Partial slot of the piece CTA `cta` holds for `pair`: 0 if it is the CTA's
// first pair, else 1 (middle pieces of a CTA are always whole pairs).
__device__ __forceinline__ int partial_slot(const AttnParams& p, int cta, int pair) {
  return (cta * p.Q) / p.C == pair ? 2 * cta : 2 * cta + 1;
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

// Load this thread's C consecutive S columns (C = 16, 32 or 64) from TMEM.
template <int C>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[C]) {
  if constexpr (C == 16) {
    tmem_ld16(taddr, r);
  } else {
#pragma unroll
    for (int c = 0; c < C; c += 32) tmem_ld32(taddr + c, *reinterpret_cast<uint32_t(*)[32]>(&r[c]));
  }
}
// Store C/2 packed bf16x2 P columns (C = 16, 32 or 64 keys) to TMEM.
template <int C>
__device__ __forceinline__ void tmem_st_pcols(uint32_t taddr, const uint32_t (&r)[C / 2]) {
  if constexpr (C == 16) tmem_st8(taddr, r);
  else if constexpr (C == 32) tmem_st16(taddr, r);
  else tmem_st32(taddr, r);
}

// K1 main kernel. Template R = query-row replication: the g*n rows of a KV
// head are loaded R times into the 128-row Q tile (replica k at TMEM lanes
// [k*128/R, (k+1)*128/R)), and replica k owns key columns [k*128/R,
// (k+1)*128/R) of every chunk. Two softmax warps share each TMEM lane
// quadrant and split the replica's columns, so a softmax thread handles
// kCols = 64/R keys per chunk instead of 128 — all 8 softmax warps busy even
// for the 36 rows of a Mixtral verify. Each (lane, warp
// pair) runs its own online softmax over its key subset; the R replicas are
// merged exactly in the epilogue like split-KV partials.
//  * P never touches shared memory: it is written (hi + lo bf16 planes) over
//    its own S buffer in TMEM and PV reads its A operand from there, so P is
//    triple-buffered with S and the shared memory holds kStages K/V chunks.
//  * lazy rescale: a lane's reference max only moves when a score exceeds it
//    by more than 2^8; otherwise P(c+1) is produced without waiting for
//    PV(c), and only lanes whose reference moved rescale O in TMEM.
template <int D, int R>
__global__ void __launch_bounds__(kThreads, 1)  // 168 regs: 3 warps share an SMSP register file
    verify_attention_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kv_k,
                            const __grid_constant__ CUtensorMap tm_kv_v, const __grid_constant__ CUtensorMap tm_v8,
                            AttnParams p) {
  using L = AttnSmem<D>;
  constexpr int kStages = L::kStages;
  constexpr int kLanes = 128 / R;         // TMEM lanes per replica
  constexpr int kW = kChunk / R;          // key columns per replica
  constexpr int kCols = kW / 2;           // key columns per softmax thread per chunk
  constexpr int kOCols = D / 2;           // O columns per softmax thread (rescale / epilogue)
  // TMEM columns: S/P buffer b < kSP at [128b, 128b+128) (P hi = first 64
  // columns, P lo = next 64, two bf16 per column), O at [128*kSP, +D). Three
  // S/P buffers let S(c+1) start before PV(c-1) has drained.
  constexpr int kSP = 3;
  constexpr uint32_t kOAcc = 128 * kSP;
  extern __shared__ uint8_t smem_raw[];
  // align within the shared array (keeps the shared address space visible to
  // the compiler: LDS/STS instead of generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t q_full[2], q_empty[2];
  // K and V of a chunk stage have separate rings: a K tile is free once S
  // is in TMEM and the softmax warps have used it for the max exchange, a V
  // tile only after PV — so K loads run up to a stage ahead of V loads
  __shared__ __align__(8) uint64_t k_full[kStages], k_empty[kStages], v_full[kStages], v_empty[kStages];
  // o_full: one phase per PV (chunk); o_last: one phase per item (its last
  // PV). Softmax warps skip o_full phases (lazy rescale), so the epilogue
  // waits on o_last, which every warp observes once per item.
  __shared__ __align__(8) uint64_t s_full[kSP], s_empty[kSP], o_full, o_last, p_full[2];
  __shared__ __align__(8) uint64_t mrg_full;  // split-KV merge: bulk copies of partials landed
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  TR_INIT();
  // the producer's first piece needs its request's prefix length: issue the
  // load before the setup below so its latency hides under it
  const int pre0 = warp == 0 && int(blockIdx.x) * p.Q < p.total
                       ? __ldg(p.prefix + piece_request(p, int(blockIdx.x) * p.Q)) : 0;
  if (warp == 0 && lane == 0) {
    TR(0, 9);  // kernel entry (trace builds)
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < kSP; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 1);
    }
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], kSoftWarps);  // every softmax warp, after the max exchange
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);           // PV commit (or the epilogue, for a piece's last chunk)
    }
    mbar_init(&o_full, 1);
    mbar_init(&o_last, 1);
    mbar_init(&p_full[0], kSoftWarps);  // P of even / odd chunks: the softmax warps may finish
    mbar_init(&p_full[1], kSoftWarps);  // chunk c+1 before the MMA thread has seen P(c)
    mbar_init(&mrg_full, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_kv_k);
    tma_prefetch_desc(&tm_kv_v);
    tma_prefetch_desc(&tm_v8);
  }
  if (warp == 1) tmem_alloc<512>(&tmem_base_sh);
  if (warp >= 2) {  // V tiles start finite (a last chunk keeps older rows past its end)
    for (int st = 0; st < kStages; ++st)
      for (int i = threadIdx.x - 64; i < L::kKvBytes / 16; i += 32 * kSoftWarps)
        reinterpret_cast<uint4*>(smem + L::kKvOff + st * 2 * L::kKvBytes + L::kKvBytes)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0 && lane == 0) TR(0, 8);  // setup done (barriers, TMEM, V zero-fill)
  const uint32_t tmem = tmem_base_sh;
  const int f_begin = blockIdx.x * p.Q, f_end = min(p.total, f_begin + p.Q);

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // Two cursors over the same chunk sequence: the K cursor (which also
    // loads each piece's Q tile) and the V cursor, polled round robin so a
    // K load never waits behind a V stage that PV still holds.
    if (elect_one()) {
      struct Cursor {
        int f, c, g;
        bool first, more;
        Piece pc;
      };
      auto next_piece = [&](Cursor& u) {
        while (u.f < f_end) {
          u.pc = u.first ? piece_make(p, u.f, f_end, pre0) : piece_at(p, u.f, f_end);
          u.first = false;
          u.f = u.pc.next_f;
          if (u.pc.c1 > u.pc.c0) {
            u.c = u.pc.c0;
            return true;
          }
        }
        return false;
      };
      // first cache row of chunk c: contiguous, or its page (one page = one chunk)
      auto chunk_row = [&](const Piece& pc, int c) {
        return p.bt ? (p.bt[pc.r * p.max_pages + c] * p.n_kv + pc.h) * kChunk
                    : (pc.r * p.n_kv + pc.h) * p.s_max + c * kChunk;
      };
      Cursor ku{f_begin, 0, 0, true, false, {}}, vu{f_begin, 0, 0, true, false, {}};
      ku.more = next_piece(ku);
      vu.more = next_piece(vu);
      int used = 0;
      bool q_in = false;  // the K cursor's piece has its Q tile issued
      while (ku.more || vu.more) {
        bool progress = false;
        if (ku.more && !q_in) {
          const int qb = used % L::kQBufs;
          if (mbar_test_wait(&q_empty[qb], ((used / L::kQBufs) & 1) ^ 1)) {
            ++used;
            mbar_arrive_expect_tx(&q_full[qb], uint32_t(R * L::kKBlocks * 64 * p.g * p.n * 2));
            for (int kb = 0; kb < L::kKBlocks; ++kb)
              for (int k = 0; k < R; ++k)
                tma_load_3d(smem + L::kQOff + qb * L::kQBytes + kb * 16384 + k * kLanes * 128, &tm_q, &q_full[qb],
                            kb * 64, ku.pc.h * p.g, ku.pc.r * p.n);
            q_in = true;
            progress = true;
          }
        }
        if (ku.more && q_in) {
          const int s = ku.g % kStages;
          if (mbar_test_wait(&k_empty[s], ((ku.g / kStages) & 1) ^ 1)) {
            TR(0, 2);
            const int crow = chunk_row(ku.pc, ku.c);
            uint8_t* kdst = smem + L::kKvOff + s * 2 * L::kKvBytes;
            mbar_arrive_expect_tx(&k_full[s], uint32_t(L::kKvBytes));
            for (int kb = 0; kb < L::kKBlocks; ++kb) tma_load_2d(kdst + kb * 16384, &tm_kv_k, &k_full[s], kb * 64, crow);
            ++ku.g;
            if (++ku.c >= ku.pc.c1) {
              ku.more = next_piece(ku);
              q_in = false;
            }
            progress = true;
          }
        }
        if (vu.more && vu.g < ku.g) {
          const int s = vu.g % kStages;
          if (mbar_test_wait(&v_empty[s], ((vu.g / kStages) & 1) ^ 1)) {
            TR(0, 3);
            const int crow = chunk_row(vu.pc, vu.c);
            uint8_t* vdst = smem + L::kKvOff + s * 2 * L::kKvBytes + L::kKvBytes;
            // a request's last chunk: V rows past its end (rounded up to 8) are
            // not loaded, the tile keeps finite older rows there (P is zero)
            const int vrows = min(kChunk, (vu.pc.keys - vu.c * kChunk + 7) & ~7);
            mbar_arrive_expect_tx(&v_full[s], uint32_t(vrows * L::kKBlocks * 128));
            for (int kb = 0; kb < L::kKBlocks; ++kb) {
              if (vrows == kChunk) {
                tma_load_2d(vdst + kb * 16384, &tm_kv_v, &v_full[s], kb * 64, crow);
              } else {
                for (int r8 = 0; r8 < vrows; r8 += 8)
                  tma_load_2d(vdst + kb * 16384 + r8 * 128, &tm_v8, &v_full[s], kb * 64, crow + r8);
              }
            }
            ++vu.g;
            if (++vu.c >= vu.pc.c1) vu.more = next_piece(vu);
            progress = true;
          }
        }
        if (!progress) __nanosleep(20);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      const uint32_t id_s = make_idesc_bf16(128, kChunk);
      const uint32_t id_o = make_idesc_bf16(128, D, /*b_mn_major=*/1);
      int used = 0, gc = 0;
      for (int f = f_begin; f < f_end;) {
        const Piece pc = piece_at(p, f, f_end);
        f = pc.next_f;
        if (pc.c1 <= pc.c0) continue;
        const int qb = used % L::kQBufs;
        mbar_wait(&q_full[qb], (used / L::kQBufs) & 1);
        ++used;
        const uint64_t qd = make_sdesc_sw128(smem_u32(smem + L::kQOff + qb * L::kQBytes), 16, 1024);
        const int nch = pc.c1 - pc.c0;
        // S(ci) may be issued once its K/V stage landed and its S/P buffer
        // was consumed by PV two chunks earlier
        auto s_ready = [&](int ci) {
          const int g2 = gc + ci;
          return mbar_test_wait(&k_full[g2 % kStages], (g2 / kStages) & 1) &&
                 mbar_test_wait(&s_empty[g2 % kSP], ((g2 / kSP) & 1) ^ 1);
        };
        auto issue_s = [&](int ci) {
          const int g2 = gc + ci;
          const int s = g2 % kStages, sb = g2 % kSP;
          TR(1, 1);
          mbar_wait(&k_full[s], (g2 / kStages) & 1);
          mbar_wait(&s_empty[sb], ((g2 / kSP) & 1) ^ 1);
          tc_fence_after();
          // descriptors are built once and advanced by constants: the single
          // issuing thread must stay under the 64-cycle MMA time per step
          const uint64_t kd = make_sdesc_sw128(smem_u32(smem + L::kKvOff + s * 2 * L::kKvBytes), 16, 1024);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t off = uint64_t(((kk / 4) * 16384 + (kk % 4) * 32) >> 4);
            umma_bf16(tmem + sb * 128, qd + off, kd + off, id_s, kk > 0 ? 1u : 0u);
          }
          umma_commit(&s_full[sb]);
          if (ci == nch - 1) umma_commit(&q_empty[qb]);
          TR(1, 2);
        };
        issue_s(0);
        for (int ci = 0; ci < nch; ++ci) {
          const int g2 = gc + ci;
          const int s = g2 % kStages, sb = g2 % kSP;
          uint8_t* vbuf = smem + L::kKvOff + s * 2 * L::kKvBytes + L::kKvBytes;
          // Wait for V(ci) and P(ci); meanwhile issue S(ci+1) as soon as its K
          // landed and its S/P buffer is free (never blocking: PV(ci) must not
          // queue behind the next chunk's K load). S(j) is thus issued after
          // PV(j-2), so S(j) complete implies PV(j-2) complete (the softmax
          // warps' o_full parity wait relies on it).
          bool next_issued = ci + 1 >= nch, v_in = false;
#ifdef SMO_ATTN_TRACE
          bool tk = false, ts = false, tv = false;
#endif
          for (;;) {
#ifdef SMO_ATTN_TRACE
            if (!next_issued && !tk && mbar_test_wait(&k_full[(g2 + 1) % kStages], ((g2 + 1) / kStages) & 1)) {
              tk = true;
              TR(1, 7);
            }
            if (!next_issued && !ts && mbar_test_wait(&s_empty[(g2 + 1) % kSP], (((g2 + 1) / kSP) & 1) ^ 1)) {
              ts = true;
              TR(1, 8);
            }
            if (!tv && mbar_test_wait(&v_full[s], (g2 / kStages) & 1)) {
              tv = true;
              TR(1, 9);
            }
#endif
            if (!next_issued && s_ready(ci + 1)) {
              issue_s(ci + 1);
              next_issued = true;
            }
            v_in = v_in || mbar_test_wait(&v_full[s], (g2 / kStages) & 1);
            if (v_in && mbar_test_wait(&p_full[g2 & 1], (g2 >> 1) & 1)) break;
          }
          // last chunk: the producer loaded V only up to the request's end
          // rounded up to 8 rows; zero the loaded rows past the end (their P
          // is zero, stale cache contents may be non-finite)
          const int valid = pc.keys - (pc.c0 + ci) * kChunk;
          if (valid < kChunk && (valid & 7)) {
            for (int rr = valid; rr < ((valid + 7) & ~7); ++rr)
#pragma unroll
              for (int kb = 0; kb < L::kKBlocks; ++kb)
#pragma unroll
                for (int t = 0; t < 8; ++t)
                  *reinterpret_cast<uint4*>(vbuf + kb * 16384 + rr * 128 + t * 16) = make_uint4(0, 0, 0, 0);
            fence_proxy_async();
          }
          TR(1, 4);
          TR(1, 5);
          tc_fence_after();
          const uint64_t vd = make_sdesc_sw128(smem_u32(vbuf), 16384, 1024);
          const uint32_t pt = tmem + sb * 128;
          // O += P_hi V + P_lo V with P read from TMEM: P carried to ~16
          // mantissa bits
#pragma unroll
          for (int kk = 0; kk < kChunk / 16; ++kk) {
            umma_bf16_ts(tmem + kOAcc, pt + kk * 8, vd + uint64_t(kk * 128), id_o, (ci > 0 || kk > 0) ? 1u : 0u);
#ifndef SMO_K1_AB_NO_LO  // timing A/B only (drops the P lo plane: wrong numerics)
            umma_bf16_ts(tmem + kOAcc, pt + 64 + kk * 8, vd + uint64_t(kk * 128), id_o, 1u);
#endif
          }
          umma_commit(&o_full);
          if (ci + 1 == nch) umma_commit(&o_last);
          umma_commit(&s_empty[sb]);
          // the last chunk's stage is released by the softmax warps after the
          // epilogue (they use it as scratch)
          if (ci + 1 < nch) umma_commit(&v_empty[s]);
          TR(1, 6);
          if (!next_issued) issue_s(ci + 1);
        }
        gc += nch;
      }
    }
  } else {
    // ------------------------------------------------------------ softmax
    const int q4 = warp & 3;                    // TMEM lane quadrant of this warp
    const int half = (warp - 2) >> 2;           // which half of the replica's columns
    const int lrow = q4 * 32 + lane;            // TMEM lane = Q tile row
    const int rep = lrow / kLanes;              // warp-uniform (kLanes >= 32)
    const int row = lrow % kLanes;              // query row (i*g + hh)
    const int stid = threadIdx.x - 64;          // 0..255 over the softmax warps
    const uint32_t tlane = uint32_t(q4 * 32) << 16;
#ifdef SMO_K1_AB_NOSOFT  // timing A/B only: no softmax math (wrong results)
    const bool warp_live = false;
#else
    const bool warp_live = (q4 * 32) % kLanes < p.rows;
#endif
    const bool live = row < p.rows;
    const int qi = live ? row / p.g : 0;
    const int col0 = rep * kW + half * kCols;   // this thread's key columns in a chunk
    const int oc0 = half * kOCols;              // this thread's O columns
    const uint32_t pair_bar = 1 + q4;           // named barrier of the two warps of a quadrant
    int gc = 0, items_done = 0;
    Piece sp0{}, sp1{};  // this CTA's split pieces (at most its first and last)
    int n_split = 0;
    const uint32_t mrg_phase = 0;  // mrg_full completes once per launch (the merge pass)
    // per-row output offsets (query i, head hh of the KV group) in rows of D
    __shared__ int row_off_sh[128];
    for (int rr = stid; rr < p.rows; rr += 32 * kSoftWarps) row_off_sh[rr] = (rr / p.g) * p.n_q + rr % p.g;
    asm volatile("bar.sync 5, 256;" ::: "memory");
    // the next piece's prefix length and mask word are loaded one piece ahead
    // (pf_*), so the epilogue does not wait on them
    int f = f_begin;
    Piece pc{};
    uint64_t mword = 0;
    int pf_prefix = -1;
    uint64_t pf_mask = 0;
    auto advance = [&]() {
      bool first = true;
      while (f < f_end) {
        const int rq = piece_request(p, f);
        const int pre = first && pf_prefix >= 0 ? pf_prefix : p.prefix[rq];
        const uint64_t mw = first && pf_prefix >= 0 ? pf_mask : (live ? p.mask[rq * p.n + qi] : 0ull);
        first = false;
        pc = piece_make(p, f, f_end, pre);
        f = pc.next_f;
        if (pc.c1 > pc.c0) {
          mword = mw;
          return true;
        }
      }
      return false;
    };
    bool have = advance();
    while (have) {
      const int nch = pc.c1 - pc.c0;
      pf_prefix = -1;
      if (f < f_end) {
        const int rq = piece_request(p, f);
        pf_prefix = __ldg(p.prefix + rq);
        pf_mask = live ? __ldg(p.mask + rq * p.n + qi) : 0ull;
      }
      uint64_t mbits = mword;
      if (p.n < 64) mbits &= (1ull << p.n) - 1ull;
      const int prefix = live ? pc.keys - p.n : 0;
      float m_ref = -INFINITY, l_run = 0.f;  // reference max (log2 units), partial row sum
      if (warp == 4 && lane == 0) TR(2, 11);
      for (int ci = 0; ci < nch; ++ci) {
        const int g2 = gc + ci;
        const int sb = g2 % kSP;
        const int key0 = (pc.c0 + ci) * kChunk;
        uint8_t* kbuf = smem + L::kKvOff + (g2 % kStages) * 2 * L::kKvBytes;
        const uint32_t tsp = tmem + tlane + sb * 128;  // this quadrant's S/P buffer
        if (warp == 4 && lane == 0) TR(2, 1);
        mbar_wait(&s_full[sb], (g2 / kSP) & 1);
        if (warp == 4 && lane == 0) TR(2, 2);
        tc_fence_after();
        // this chunk's K tile is dead once S is in TMEM (it is refilled only
        // after PV of this chunk, i.e. after every warp's p_full arrival):
        // use it for the pair's max exchange
        float* xchg = reinterpret_cast<float*>(kbuf);
        uint32_t sv[kCols];
        uint32_t vb[(kCols + 31) / 32];
        float cmax = -INFINITY;
        if (warp_live) {
          tmem_ld_cols<kCols>(tsp + col0, sv);
#pragma unroll
          for (int w = 0; w < (kCols + 31) / 32; ++w) vb[w] = visible_bits(key0 + col0 + 32 * w, prefix, mbits);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < kCols; ++j)
            if ((vb[j / 32] >> (j % 32)) & 1u) cmax = fmaxf(cmax, __uint_as_float(sv[j]));
        }
        xchg[half * 128 + lrow] = cmax;
        // both warps' S columns are in registers after this barrier, so P may
        // overwrite the S buffer
        asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");
        cmax = fmaxf(cmax, xchg[(half ^ 1) * 128 + lrow]) * p.scale_log2;
        // K tile (and exchange) done: hand it to the producer, except a
        // piece's last chunk, whose stage is the epilogue's scratch
        if (ci + 1 < nch) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&k_empty[g2 % kStages]);
        }
        const bool grow = cmax > m_ref + 8.f;  // also true for the first visible score
        const float m_new = grow ? cmax : m_ref;
        const float alpha = grow ? (m_ref == -INFINITY ? 0.f : ex2_approx(m_ref - m_new)) : 1.f;
        if (warp == 4 && lane == 0) TR(2, 3);
        // p = 2^(s*scale - m) on visible keys (<= 2^8); P row = hi + lo bf16
        const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
        float psum = 0.f;
        if (warp_live) {
          // 32-key blocks keep the register footprint flat. P = hi + lo: hi is
          // the truncated bf16 pair (one PRMT), lo = p - hi is exact in fp32 and
          // rounded once (one cvt per pair): |error| <= 2^-16 p
          constexpr int kB = kCols < 32 ? kCols : 32;
#pragma unroll
          for (int c = 0; c < kCols; c += kB) {
            uint32_t phi[kB / 2], plo[kB / 2];
#pragma unroll
            for (int j = c; j < c + kB; j += 2) {
              const float a = ((vb[j / 32] >> (j % 32)) & 1u) ? ex2_approx(__uint_as_float(sv[j]) * p.scale_log2 - m_use) : 0.f;
              const float b =
                  ((vb[j / 32] >> ((j + 1) % 32)) & 1u) ? ex2_approx(__uint_as_float(sv[j + 1]) * p.scale_log2 - m_use) : 0.f;
              psum += a + b;
              const uint32_t ua = __float_as_uint(a), ub = __float_as_uint(b);
              phi[(j - c) / 2] = __byte_perm(ua, ub, 0x7632);
              plo[(j - c) / 2] = pack_bf16x2(a - __uint_as_float(ua & 0xffff0000u), b - __uint_as_float(ub & 0xffff0000u));
            }
            tmem_st_pcols<kB>(tsp + (col0 + c) / 2, phi);
            tmem_st_pcols<kB>(tsp + 64 + (col0 + c) / 2, plo);
          }
          if constexpr (R > 1) {
            // keys of other replicas: zero P for this lane (half 0 the hi
            // plane, half 1 the lo plane)
            uint32_t z[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) z[j] = 0u;
#pragma unroll
            for (int c = 0; c < 64; c += 8)
              if (c < rep * (kW / 2) || c >= (rep + 1) * (kW / 2)) tmem_st8(tsp + half * 64 + c, z);
          }
        }
        l_run = l_run * alpha + psum;
        m_ref = m_new;
        if (warp == 4 && lane == 0) TR(2, 20);
        if (warp == 4 && lane == 0) TR(2, 21);
        // lanes whose reference max moved rescale O (and only after PV(ci-1))
        if (ci > 0 && warp_live && __any_sync(0xffffffffu, live && alpha != 1.f)) {
          mbar_wait(&o_full, (g2 - 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c0 = 0; c0 < kOCols; c0 += 32) {
            uint32_t r[32];
            tmem_ld32(tmem + tlane + kOAcc + oc0 + c0, r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * alpha);
            tmem_st32(tmem + tlane + kOAcc + oc0 + c0, r);
          }
        }
        if (warp == 4 && lane == 0) TR(2, 4);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[g2 & 1]);
        if (warp == 4 && lane == 0) TR(2, 5);
      }
      mbar_wait(&o_last, items_done & 1);
      ++items_done;
      tc_fence_after();
      if (warp == 4 && lane == 0) TR(2, 6);
      const Piece cur = pc;
      const bool whole = cur.npieces == 1;
      have = advance();
      // ---- epilogue. The last chunk's K/V stage is held for us (released
      // below): first the (m, l) exchange in its V tile, then the weighted
      // replica partials [R][kLanes][D] fp32 over the stage (16-byte pieces
      // XOR-swizzled by row), summed by all softmax threads with coalesced
      // stores.
      const int s_last = (gc + nch - 1) % kStages;
      gc += nch;
      uint8_t* stage = smem + L::kKvOff + s_last * 2 * L::kKvBytes;
      float* slots = reinterpret_cast<float*>(stage);
      float* lsum = reinterpret_cast<float*>(stage + L::kKvBytes);         // [2][128]
      float2* ml = reinterpret_cast<float2*>(stage + L::kKvBytes + 1024);  // [128]
      lsum[half * 128 + lrow] = l_run;
      asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");
      const float l_tot = l_run + lsum[(half ^ 1) * 128 + lrow];
      if (half == 0) ml[lrow] = make_float2(m_ref, l_tot);
      asm volatile("bar.sync 5, 256;" ::: "memory");
      if (warp == 4 && lane == 0) TR(2, 7);
      float M = -INFINITY, Ls = 0.f;
      if (live) {
#pragma unroll
        for (int k = 0; k < R; ++k) M = fmaxf(M, ml[row + k * kLanes].x);
#pragma unroll
        for (int k = 0; k < R; ++k) {
          const float2 v = ml[row + k * kLanes];
          if (v.x != -INFINITY) Ls += v.y * ex2_approx(v.x - M);
        }
      }
      // this replica's weight in the merged row (normalised for whole pieces)
      float wgt = (live && m_ref != -INFINITY) ? ex2_approx(m_ref - M) : 0.f;
      if (whole) wgt *= Ls > 0.f ? 1.f / Ls : 0.f;
      asm volatile("bar.sync 5, 256;" ::: "memory");  // ml / lsum read: the stage becomes slots
      if (warp_live) {
#pragma unroll 1
        for (int c0 = 0; c0 < kOCols; c0 += 32) {
          uint32_t r[32];
          tmem_ld32(tmem + tlane + kOAcc + oc0 + c0, r);
          tmem_ld_wait();
          if (!live) continue;
          float4* slot = reinterpret_cast<float4*>(slots) + (rep * kLanes + row) * (D / 4);
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            slot[((oc0 + c0 + j) / 4) ^ (row & 7)] =
                make_float4(__uint_as_float(r[j]) * wgt, __uint_as_float(r[j + 1]) * wgt,
                            __uint_as_float(r[j + 2]) * wgt, __uint_as_float(r[j + 3]) * wgt);
        }
      }
      tc_fence_before();  // TMEM O reads done before the next piece's PV overwrites it
      asm volatile("bar.sync 5, 256;" ::: "memory");
      if (warp == 4 && lane == 0) TR(2, 13);
      const int my_slot = whole ? 0 : partial_slot(p, blockIdx.x, cur.pair);
      {
        // replicas summed in a fixed order; thread -> (row, 4 columns)
        const float4* s4 = reinterpret_cast<const float4*>(slots);
        for (int e = stid; e < p.rows * (D / 4); e += 32 * kSoftWarps) {
          const int rr = e / (D / 4), c4 = e % (D / 4);
          float4 a = s4[rr * (D / 4) + (c4 ^ (rr & 7))];
#pragma unroll
          for (int k = 1; k < R; ++k) {
            const float4 b = s4[(k * kLanes + rr) * (D / 4) + (c4 ^ (rr & 7))];
            a.x += b.x;
            a.y += b.y;
            a.z += b.z;
            a.w += b.w;
          }
          if (whole) {
            uint16_t* dst = p.out + (size_t(cur.r) * p.n * p.n_q + size_t(cur.h) * p.g + row_off_sh[rr]) * D;
            *reinterpret_cast<uint2*>(dst + 4 * c4) = make_uint2(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w));
          } else {
            reinterpret_cast<float4*>(p.ws_o + (size_t(my_slot) * p.rows + rr) * D)[c4] = a;
          }
        }
        if (!whole && live && rep == 0 && half == 0) p.ws_ml[size_t(my_slot) * p.rows + row] = make_float2(M, Ls);
      }
      if (warp == 4 && lane == 0) TR(2, 9);
      if (!whole) {
        // publish the partial (bar.sync orders the CTA's partial stores
        // before thread 0's release add; release is cumulative); the pair is
        // merged after this CTA's last item, a slice by each of its pieces
        asm volatile("bar.sync 5, 256;" ::: "memory");
        if (warp == 4 && lane == 0) TR(2, 30);
        if (stid == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(p.ws_cnt + cur.pair) : "memory");
        if (n_split == 0)
          sp0 = cur;
        else
          sp1 = cur;
        ++n_split;
      }
      // all stage reads done -> restore the V tile to zeros and hand the
      // stage back to the producer. The epilogue scratch above left fp32 bit
      // patterns in it; a later partial last chunk only loads V rows up to its
      // end and keeps the rest, whose P is zero — but 0 * (a bf16 NaN/Inf
      // pattern) is not zero in the PV MMA.
      // (after the CTA's last item no chunk loads follow: no zero-fill)
      asm volatile("bar.sync 5, 256;" ::: "memory");
      if (have) {
        for (int i = stid; i < L::kKvBytes / 16; i += 32 * kSoftWarps)
          reinterpret_cast<uint4*>(stage + L::kKvBytes)[i] = make_uint4(0, 0, 0, 0);
        fence_proxy_async();
        asm volatile("bar.sync 5, 256;" ::: "memory");
      }
      if (lane == 0) mbar_arrive(&k_empty[s_last]);
      if (stid == 0) mbar_arrive(&v_empty[s_last]);
      if (warp == 4 && lane == 0) TR(2, 10);
    }
    // ---- split-KV merge (deferred). A CTA's first and last pieces may be
    // parts of a pair (its middle pieces are whole pairs). Every piece of a
    // split pair merges one slice of the pair's output, out = sum_j w_j O_j
    // with w_j[row] = 2^(m_j - M) / L, once all np pieces are published:
    // the merge reads np x slice instead of one CTA reading np x the whole
    // pair, in parallel on np SMs (the grid is cooperative, so the pieces are
    // co-resident and the wait resolves). The slice's partial runs are
    // contiguous, so one thread stages them with np bulk copies into the
    // now idle K/V stages; the sums run in piece order (deterministic).
    // Both split pieces are merged in one pass (one set of barriers and
    // round trips): region k of the stages holds pair k's weights, (m, l)
    // rows and staged partials.
    if (n_split > 0) {
      // floats: w [16][128], slot_of [64], (m, l) [16][128], then the staged
      // partials: np slices of ne float4 with np * ne <= rows * D / 4 + np
      constexpr int kRegion = 16 * 128 + 64 + 16 * 128 * 2 + (128 * (D / 4) + 16) * 4;
      static_assert(2 * kRegion * 4 <= L::kStages * 2 * L::kKvBytes, "merge regions exceed the K/V stages");
      // per-pair slice geometry in shared memory (indexed by pair k below)
      __shared__ int np[2], e_lo[2], ne[2], r_lo[2], nr[2];
      if (stid < 2) {
        const int k = stid;
        const Piece& sp = k == 0 ? sp0 : sp1;
        const int jme = int(blockIdx.x) - sp.first_cta, n_e = p.rows * (D / 4);
        const int npk = k < n_split ? sp.npieces : 0;
        const int lo = k < n_split ? jme * n_e / npk : 0;
        const int nek = k < n_split ? (jme + 1) * n_e / npk - lo : 0;  // float4, >= 2
        np[k] = npk;
        e_lo[k] = lo;
        ne[k] = nek;
        r_lo[k] = lo / (D / 4);
        nr[k] = k < n_split ? (lo + nek - 1) / (D / 4) + 1 - lo / (D / 4) : 0;
      }
      asm volatile("bar.sync 5, 256;" ::: "memory");
      float* const mbase = reinterpret_cast<float*>(smem + L::kKvOff);
      auto w = [&](int k) { return mbase + k * kRegion; };
      auto slot_of = [&](int k) { return reinterpret_cast<int*>(mbase + k * kRegion + 16 * 128); };
      auto mls = [&](int k) { return reinterpret_cast<float2*>(mbase + k * kRegion + 16 * 128 + 64); };
      auto stg = [&](int k) { return reinterpret_cast<float4*>(mbase + k * kRegion + 16 * 128 + 64 + 16 * 128 * 2); };
      if (warp == 4 && lane == 0) TR(2, 31);
      if (stid == 0) {
        for (int k = 0; k < n_split; ++k) {
          const int* cnt = p.ws_cnt + (k == 0 ? sp0.pair : sp1.pair);
          int v;
          for (;;) {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
            if (v >= np[k]) break;
            __nanosleep(32);
          }
        }
      }
      if (stid < 32 && stid < np[0]) slot_of(0)[stid] = partial_slot(p, sp0.first_cta + stid, sp0.pair);
      if (stid >= 32 && stid - 32 < np[1]) slot_of(1)[stid - 32] = partial_slot(p, sp1.first_cta + stid - 32, sp1.pair);
      fence_proxy_async();  // generic accesses of the stages before the bulk copies
      asm volatile("bar.sync 5, 256;" ::: "memory");
      if (stid == 0) {
        mbar_arrive_expect_tx(&mrg_full, uint32_t((np[0] * ne[0] + np[1] * ne[1]) * 16));
        for (int k = 0; k < n_split; ++k)
          for (int j = 0; j < np[k]; ++j)
            bulk_load(stg(k) + j * ne[k],
                      reinterpret_cast<const float4*>(p.ws_o + size_t(slot_of(k)[j]) * p.rows * D) + e_lo[k],
                      uint32_t(ne[k] * 16), &mrg_full);
      }
      // (m, l) of the slices' rows, both pairs in one round trip
      for (int t = stid; t < np[0] * nr[0] + np[1] * nr[1]; t += 32 * kSoftWarps) {
        const int k = t >= np[0] * nr[0], tt = t - (k ? np[0] * nr[0] : 0);
        const int j = tt / nr[k], rl = tt - j * nr[k];
        mls(k)[j * 128 + rl] = __ldcg(&p.ws_ml[size_t(slot_of(k)[j]) * p.rows + r_lo[k] + rl]);
      }
      asm volatile("bar.sync 5, 256;" ::: "memory");
      for (int t = stid; t < nr[0] + nr[1]; t += 32 * kSoftWarps) {
        const int k = t >= nr[0], rl = t - (k ? nr[0] : 0);
        float Mx = -INFINITY, Lx = 0.f;
        for (int j = 0; j < np[k]; ++j) Mx = fmaxf(Mx, mls(k)[j * 128 + rl].x);
        for (int j = 0; j < np[k]; ++j) {
          const float2 ml = mls(k)[j * 128 + rl];
          const float e2 = ml.x == -INFINITY ? 0.f : ex2_approx(ml.x - Mx);
          w(k)[j * 128 + rl] = e2;
          Lx += ml.y * e2;
        }
        const float inv = Lx > 0.f ? 1.f / Lx : 0.f;
        for (int j = 0; j < np[k]; ++j) w(k)[j * 128 + rl] *= inv;
      }
      asm volatile("bar.sync 5, 256;" ::: "memory");
      if (warp == 4 && lane == 0) TR(2, 32);
      mbar_wait(&mrg_full, mrg_phase);
      for (int t = stid; t < ne[0] + ne[1]; t += 32 * kSoftWarps) {
        const int k = t >= ne[0], e = t - (k ? ne[0] : 0);
        const Piece& sp = k ? sp1 : sp0;
        const int E = e_lo[k] + e, rr = E / (D / 4), c4 = E % (D / 4);
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int j = 0; j < np[k]; ++j) {
          const float4 v = stg(k)[j * ne[k] + e];
          const float wj = w(k)[j * 128 + rr - r_lo[k]];
          acc.x += v.x * wj;
          acc.y += v.y * wj;
          acc.z += v.z * wj;
          acc.w += v.w * wj;
        }
        uint16_t* obase = p.out + (size_t(sp.r) * p.n * p.n_q + size_t(sp.h) * p.g) * D;
        *reinterpret_cast<uint2*>(obase + size_t(row_off_sh[rr]) * D + 4 * c4) =
            make_uint2(pack_bf16x2(acc.x, acc.y), pack_bf16x2(acc.z, acc.w));
      }
      if (warp == 4 && lane == 0) TR(2, 33);
      if (stid == 0) {  // a pair's last merge re-arms its counter for the next launch
        for (int k = 0; k < n_split; ++k) {
          int* cnt = p.ws_cnt + (k == 0 ? sp0.pair : sp1.pair);
          int old;
          asm volatile("atom.relaxed.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
          if (old == 2 * np[k] - 1) *cnt = 0;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}


struct AttnPlan {
  int C, Q, total, grid;
  size_t ws_o_off, ws_ml_off, ws_cnt_off, ws_bytes;
};

constexpr size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Flat schedule: C chunk slots per (request, KV head), Q consecutive slots per
// CTA so that the grid fills the SMs once; Q >= C/15 keeps a pair's pieces
// within 16 (the merge's weight table). Workspace: two partial slots per CTA
// (sized for a full grid, so it does not depend on the prefix lengths) and
// one counter per pair.
AttnPlan plan_attention(const smo_attn_args& a, int sms) {
  AttnPlan pl{};
  const int rows = (a.n_q / a.n_kv) * a.n;
  const int pairs = a.b * a.n_kv;
  pl.C = std::max(1, (a.max_prefix + a.n + kChunk - 1) / kChunk);
  pl.total = pairs * pl.C;
  // Q: at least total/sms (one wave). Candidates aligned with pairs (a
  // multiple or a divisor of C) avoid partial pieces; pick the lowest
  // modelled CTA time  Q*t_chunk + pieces*t_epilogue + partials*t_merge
  // (t ~ 1.6 / 4 / 3 us, measured on B200, profiles/).
  const int qmin = (pl.total + sms - 1) / sms;
  auto cost = [&](int q) {
    const bool aligned = q % pl.C == 0 || pl.C % q == 0;
    const double pieces = q >= pl.C ? double(q) / pl.C + (aligned ? 0.0 : 1.0) : (aligned ? 1.0 : 2.0);
    const double partials = aligned ? (q >= pl.C ? 0.0 : 1.0) : 2.0;
    return q * 1.6 + pieces * 4.0 + partials * 3.0;
  };
  int q = qmin;
  const int qa = qmin >= pl.C ? pl.C * ((qmin + pl.C - 1) / pl.C) : [&] {
    for (int d = qmin; d <= pl.C; ++d)
      if (pl.C % d == 0) return d;
    return pl.C;
  }();
  if (cost(qa) < cost(qmin)) q = qa;
  pl.Q = std::max(q, (pl.C + 14) / 15);
  // A/B override: never below qmin (grid <= sms: the workspace holds 2 partial slots per SM)
  if (const char* fq = std::getenv("SMO_ATTN_Q")) pl.Q = std::max(std::max(std::atoi(fq), qmin), (pl.C + 14) / 15);
  pl.grid = (pl.total + pl.Q - 1) / pl.Q;
  // the layout is sized for the largest tile (128 rows) so that the counter
  // region sits at the same offset for every n: a workspace shared by calls
  // of different shapes (verify, drafter, prefill chunks) keeps its
  // zero-between-launches counters where the next call looks for them
  (void)rows;
  pl.ws_o_off = 0;
  pl.ws_ml_off = align256(size_t(sms) * 2 * 128 * a.d * sizeof(float));
  pl.ws_cnt_off = pl.ws_ml_off + align256(size_t(sms) * 2 * 128 * sizeof(float2));
  pl.ws_bytes = pl.ws_cnt_off + align256(size_t(pairs) * sizeof(int));
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

template <int D, int R>
void launch_k1(int grid, cudaStream_t stream, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
               const CUtensorMap& tv8, const AttnParams& p) {
  constexpr size_t smem = AttnSmem<D>::kTotal + 1024;
  static bool set = false;
  if (!set) {
    SMO_CUDA_CHECK(cudaFuncSetAttribute(verify_attention_kernel<D, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(smem)));
    set = true;
  }
  // cooperative: the pieces of a split pair wait for each other before the
  // merge (grid <= SMs at one CTA per SM)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SMO_CUDA_CHECK(cudaLaunchKernelEx(&cfg, verify_attention_kernel<D, R>, tq, tk, tv, tv8, p));
}

void check_attn_args(const smo_attn_args& a) {
  SMO_REQUIRE(a.q && a.k_cache && a.v_cache && a.mask && a.prefix_len && a.out, "attention: null pointer");
  SMO_REQUIRE(a.b > 0 && a.n > 0 && a.n_q > 0 && a.n_kv > 0, "attention: shape mismatch");
  SMO_REQUIRE(a.n_q % a.n_kv == 0, "attention: shape mismatch");
  SMO_REQUIRE(a.d == 64 || a.d == 128, "attention: head_dim must be 64 or 128");
  SMO_REQUIRE(a.n <= 64, "attention: mask size mismatch");
  SMO_REQUIRE((a.n_q / a.n_kv) * a.n <= 128, "attention: n * (n_q/n_kv) must be <= 128");
  if (a.block_table) {
    SMO_REQUIRE(a.max_pages > 0 && a.num_pages > 0, "attention: paged K/V needs max_pages and num_pages");
    SMO_REQUIRE(a.max_prefix >= 0 && a.max_prefix + a.n <= a.max_pages * kChunk, "attention: shape mismatch");
  } else {
    SMO_REQUIRE(a.max_prefix >= 0 && a.max_prefix + a.n <= a.s_max, "attention: shape mismatch");
  }
}

}  // namespace

size_t attention_workspace(const smo_attn_args& a) {
  check_attn_args(a);
  return plan_attention(a, device_sms()).ws_bytes;
}

void attention_launch(const smo_attn_args& a, cudaStream_t stream) {
  check_attn_args(a);
  const AttnPlan pl = plan_attention(a, device_sms());
  SMO_REQUIRE(a.workspace && a.workspace_bytes >= pl.ws_bytes, "attention: workspace too small");
  const int g = a.n_q / a.n_kv;
  uint8_t* ws = reinterpret_cast<uint8_t*>(a.workspace);
  AttnParams p{};
  p.mask = a.mask;
  p.prefix = a.prefix_len;
  p.out = reinterpret_cast<uint16_t*>(a.out);
  p.ws_o = reinterpret_cast<float*>(ws + pl.ws_o_off);
  p.ws_ml = reinterpret_cast<float2*>(ws + pl.ws_ml_off);
  p.ws_cnt = reinterpret_cast<int*>(ws + pl.ws_cnt_off);
  p.b = a.b;
  p.n = a.n;
  p.n_q = a.n_q;
  p.n_kv = a.n_kv;
  p.g = g;
  p.rows = g * a.n;
  p.s_max = a.s_max;
  p.bt = a.block_table;
  p.max_pages = a.max_pages;
  p.C = pl.C;
  p.Q = pl.Q;
  p.total = pl.total;
  p.scale_log2 = float(1.4426950408889634 / std::sqrt(double(a.d)));

  CUtensorMap tq, tk, tv, tv8;
  {
    uint64_t dims[3] = {uint64_t(a.d), uint64_t(a.n_q), uint64_t(a.b) * a.n};
    uint64_t strides[2] = {uint64_t(a.d) * 2, uint64_t(a.n_q) * a.d * 2};
    uint32_t box[3] = {64, uint32_t(g), uint32_t(a.n)};
    make_tmap_bf16(&tq, a.q, 3, dims, strides, box, true);
  }
  {
    const uint64_t cache_rows =
        a.block_table ? uint64_t(a.num_pages) * a.n_kv * kChunk : uint64_t(a.b) * a.n_kv * a.s_max;
    uint64_t dims[2] = {uint64_t(a.d), cache_rows};
    uint64_t strides[1] = {uint64_t(a.d) * 2};
    uint32_t box[2] = {64, uint32_t(kChunk)};
    make_tmap_bf16(&tk, a.k_cache, 2, dims, strides, box, true);
    make_tmap_bf16(&tv, a.v_cache, 2, dims, strides, box, true);
    uint32_t box8[2] = {64, 8};
    make_tmap_bf16(&tv8, a.v_cache, 2, dims, strides, box8, true);
  }
  // query-row replication: as many copies of the g*n rows as fit the 128 lanes
  const int R = p.rows <= 32 ? 4 : (p.rows <= 64 ? 2 : 1);
  if (a.d == 128) {
    if (R == 4) launch_k1<128, 4>(pl.grid, stream, tq, tk, tv, tv8, p);
    else if (R == 2) launch_k1<128, 2>(pl.grid, stream, tq, tk, tv, tv8, p);
    else launch_k1<128, 1>(pl.grid, stream, tq, tk, tv, tv8, p);
  } else {
    if (R == 4) launch_k1<64, 4>(pl.grid, stream, tq, tk, tv, tv8, p);
    else if (R == 2) launch_k1<64, 2>(pl.grid, stream, tq, tk, tv, tv8, p);
    else launch_k1<64, 1>(pl.grid, stream, tq, tk, tv, tv8, p);
  }
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
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
