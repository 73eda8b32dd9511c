// ops.cu — K2 router top-k, K3 permute / unpermute-combine, K6 argmax +
// greedy accept + KV rollback, and the small support ops of a Mixtral verify
// layer (RMSNorm, embedding, RoPE + KV append, procedural fills).
// All of these are HBM/latency-bound; none is GEMM-shaped.
#include <cmath>

#include <algorithm>

#include "common.cuh"

namespace smo {

namespace {

constexpr int kMaxExperts = 64;
constexpr int kMaxTopK = 8;

// ---------------------------------------------------------------- fills
__global__ void fill_uniform_kernel(uint16_t* dst, uint64_t count, uint64_t key, uint64_t base, float s) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t x = splitmix64(splitmix64(key ^ (base + i)));
    const int32_t c = int32_t((x >> 40) << 1) - (1 << 24);
    dst[i] = f2bf(__fmul_rn(float(c), s));
  }
}

// trained-weight-like init (c_api.h smo_fill_normal_bf16): Irwin-Hall of the
// four chained draws of the same splitmix64 stream, 1/1024 outliers x8
__global__ void fill_normal_kernel(uint16_t* dst, uint64_t count, uint64_t key, uint64_t base, float s) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t x = splitmix64(splitmix64(key ^ (base + i)));
    int32_t c = int32_t(x >> 40);
#pragma unroll
    for (int k = 1; k < 4; ++k) {
      x = splitmix64(x);
      c += int32_t(x >> 40);
    }
    c -= 1 << 25;
    if ((x & 1023u) == 0) c *= 8;
    dst[i] = f2bf(__fmul_rn(__int2float_rn(c), s));
  }
}

__global__ void fill_kv_prefix_kernel(uint16_t* cache, const int32_t* prefix, int n_kv, int d, int s_max,
                                      uint64_t key, float s, const int32_t* bt, int max_pages) {
  const int rh = blockIdx.y;  // r * n_kv + h
  const int r = rh / n_kv, h = rh % n_kv;
  const int len = prefix[r];
  const uint64_t total = uint64_t(len) * d;
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < total;
       e += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t idx = (uint64_t(rh) << 32) | e;
    const uint64_t x = splitmix64(splitmix64(key ^ idx));
    const int32_t c = int32_t((x >> 40) << 1) - (1 << 24);
    const long long row = kv_row(bt, max_pages, r, h, int(e / d), n_kv, s_max);
    if (row >= 0) cache[uint64_t(row) * d + e % d] = f2bf(__fmul_rn(float(c), s));
  }
}

// ---------------------------------------------------------------- K2 router
// One warp per token. Lane l owns the 8-element chunks at 256*i + 8*l and
// accumulates them in order with fmaf; an xor-butterfly then reduces the 32
// partials (identical on every lane). This fixed order is what the oracle
// restates (oracle.c:orc_router_logits), so ids are bit-exact.
__global__ void router_topk_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ w, int T, int h,
                                   int E, int k, float* logits_out, int32_t* ids, float* weights) {
  // one block per token, warp w computes experts w, w + nwarps, ...: each
  // (token, expert) dot product keeps the fixed lane order above
  const int t = blockIdx.x;
  const int wid = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  __shared__ float lg[kMaxExperts];
  const uint16_t* xr = x + size_t(t) * h;
  for (int e = wid; e < E; e += nw) {
    const uint16_t* wr = w + size_t(e) * h;
    float a = 0.f;
    // the 16-byte loads of kU chunks are issued together, then the FMA chain
    // on `a` runs in the fixed order (bit-identical to one chunk at a time)
    constexpr int kU = 8;
    for (int b0 = lane * 8; b0 < h; b0 += 256 * kU) {
      uint4 xv[kU], wv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int base = b0 + 256 * u;
        xv[u] = base < h ? *reinterpret_cast<const uint4*>(xr + base) : make_uint4(0, 0, 0, 0);
        wv[u] = base < h ? *reinterpret_cast<const uint4*>(wr + base) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (b0 + 256 * u >= h) break;
        const uint32_t xs[4] = {xv[u].x, xv[u].y, xv[u].z, xv[u].w};
        const uint32_t ws[4] = {wv[u].x, wv[u].y, wv[u].z, wv[u].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          a = __fmaf_rn(__uint_as_float(xs[q] << 16), __uint_as_float(ws[q] << 16), a);
          a = __fmaf_rn(__uint_as_float(xs[q] & 0xffff0000u), __uint_as_float(ws[q] & 0xffff0000u), a);
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) a = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (lane == 0) lg[e] = a;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (logits_out)
    for (int e = 0; e < E; ++e) logits_out[size_t(t) * E + e] = lg[e];
  uint64_t used = 0;
  int sel[kMaxTopK];
  for (int j = 0; j < k; ++j) {
    int best = -1;
    for (int e = 0; e < E; ++e) {
      if ((used >> e) & 1ull) continue;
      if (best < 0 || lg[e] > lg[best]) best = e;
    }
    used |= 1ull << best;
    sel[j] = best;
    ids[size_t(t) * k + j] = best;
  }
  const float mx = lg[sel[0]];
  float ex[kMaxTopK], den = 0.f;
  for (int j = 0; j < k; ++j) {
    ex[j] = expf(lg[sel[j]] - mx);
    den += ex[j];
  }
  for (int j = 0; j < k; ++j) weights[size_t(t) * k + j] = ex[j] / den;
}

// ---------------------------------------------------------------- K3 permute
// Single CTA, one warp per expert (strided): ballot + popc gives each pair's
// rank among the earlier pairs of its expert -> a stable counting sort.
// The ids are staged in shared memory first (one coalesced pass by all
// threads) when they fit: the per-expert ballot loops then read shared memory
// instead of making a global round trip per 32 pairs.
constexpr int kPermuteSmemIds = 12288;  // 48 KB of dynamic shared memory
__global__ void permute_kernel(const int32_t* __restrict__ ids_g, int P, int E, int32_t* offsets, int32_t* perm,
                               int32_t* pos) {
  __shared__ int cnt[kMaxExperts + 1];
  extern __shared__ int ids_sh[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  const bool staged = P <= kPermuteSmemIds;
  if (staged) {
    for (int i = threadIdx.x; i < P; i += blockDim.x) ids_sh[i] = ids_g[i];
    __syncthreads();
  }
  const int32_t* ids = staged ? ids_sh : ids_g;
  for (int e = warp; e < E; e += nw) {
    int c = 0;
    for (int i0 = 0; i0 < P; i0 += 32) {
      const int i = i0 + lane;
      c += __popc(__ballot_sync(0xffffffffu, i < P && ids[i] == e));
    }
    if (lane == 0) cnt[e] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int e = 0; e < E; ++e) {
      const int c = cnt[e];
      cnt[e] = run;
      offsets[e] = run;
      run += c;
    }
    offsets[E] = run;
  }
  __syncthreads();
  for (int e = warp; e < E; e += nw) {
    int base = cnt[e];
    for (int i0 = 0; i0 < P; i0 += 32) {
      const int i = i0 + lane;
      const bool mine = i < P && ids[i] == e;
      const uint32_t bal = __ballot_sync(0xffffffffu, mine);
      if (mine) {
        const int at = base + __popc(bal & ((1u << lane) - 1u));
        perm[at] = i;
        pos[i] = at;
      }
      base += __popc(bal);
    }
  }
}

__global__ void gather_rows_kernel(const uint16_t* __restrict__ x, const int32_t* __restrict__ perm, int k,
                                   int h, int P, uint16_t* __restrict__ xp) {
  const int row = blockIdx.x;
  if (row >= P) return;
  const int src = perm[row] / k;
  const uint4* s = reinterpret_cast<const uint4*>(x + size_t(src) * h);
  uint4* d = reinterpret_cast<uint4*>(xp + size_t(row) * h);
  for (int c = threadIdx.x; c < h / 8; c += blockDim.x) d[c] = s[c];
}

// splits > 1: the down projection arrives as K slices y[s] (moe_tc.cu,
// split_stride elements apart), summed in slice order before the weighting.
__global__ void combine_kernel(const float* __restrict__ y, const int32_t* __restrict__ pos,
                               const float* __restrict__ w, int T, int k, int h, float* __restrict__ res,
                               int splits, size_t split_stride) {
  const int t = blockIdx.x;
  for (int c = threadIdx.x * 4; c < h; c += blockDim.x * 4) {
    float4 acc = *reinterpret_cast<float4*>(res + size_t(t) * h + c);
    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < k; ++j) {
      const float wj = w[size_t(t) * k + j];
      const size_t at = size_t(pos[size_t(t) * k + j]) * h + c;
      float4 v = *reinterpret_cast<const float4*>(y + at);
      for (int s = 1; s < splits; ++s) {
        const float4 v2 = *reinterpret_cast<const float4*>(y + size_t(s) * split_stride + at);
        v.x += v2.x;
        v.y += v2.y;
        v.z += v2.z;
        v.w += v2.w;
      }
      sum.x = __fmaf_rn(wj, v.x, sum.x);
      sum.y = __fmaf_rn(wj, v.y, sum.y);
      sum.z = __fmaf_rn(wj, v.z, sum.z);
      sum.w = __fmaf_rn(wj, v.w, sum.w);
    }
    acc.x += sum.x;
    acc.y += sum.y;
    acc.z += sum.z;
    acc.w += sum.w;
    *reinterpret_cast<float4*>(res + size_t(t) * h + c) = acc;
  }
}

// ---------------------------------------------------------------- norm / embed
// One block of 256 threads per row; the row's float4 chunks (h <= 8192) are
// loaded once, together, and kept in registers for the scaling pass. The
// per-thread sum of squares runs over the thread's chunks in increasing
// column order, as before (bit-identical).
constexpr int kRmsMaxV = 8;
__global__ void rmsnorm_kernel(const float* __restrict__ x, const uint16_t* __restrict__ gain, int h, float eps,
                               uint16_t* __restrict__ y) {
  const int t = blockIdx.x;
  const float* xr = x + size_t(t) * h;
  const int stride = blockDim.x * 4;
  float4 v[kRmsMaxV];
  uint2 gv[kRmsMaxV];
#pragma unroll
  for (int u = 0; u < kRmsMaxV; ++u) {
    const int c = threadIdx.x * 4 + u * stride;
    v[u] = c < h ? *reinterpret_cast<const float4*>(xr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    gv[u] = c < h ? *reinterpret_cast<const uint2*>(gain + c) : make_uint2(0u, 0u);
  }
  float ss = 0.f;
#pragma unroll
  for (int u = 0; u < kRmsMaxV; ++u)
    if (threadIdx.x * 4 + u * stride < h) ss += v[u].x * v[u].x + v[u].y * v[u].y + v[u].z * v[u].z + v[u].w * v[u].w;
  __shared__ float red[32];
  ss = warp_sum(ss);
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float r = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
    r = warp_sum(r);
    if (threadIdx.x == 0) red[0] = r;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / float(h) + eps);
#pragma unroll
  for (int u = 0; u < kRmsMaxV; ++u) {
    const int c = threadIdx.x * 4 + u * stride;
    if (c >= h) break;
    const float g0 = __uint_as_float(gv[u].x << 16), g1 = __uint_as_float(gv[u].x & 0xffff0000u);
    const float g2 = __uint_as_float(gv[u].y << 16), g3 = __uint_as_float(gv[u].y & 0xffff0000u);
    uint2 o;
    o.x = uint32_t(f2bf(v[u].x * inv * g0)) | (uint32_t(f2bf(v[u].y * inv * g1)) << 16);
    o.y = uint32_t(f2bf(v[u].z * inv * g2)) | (uint32_t(f2bf(v[u].w * inv * g3)) << 16);
    *reinterpret_cast<uint2*>(y + size_t(t) * h + c) = o;
  }
}

__global__ void embed_kernel(const int32_t* __restrict__ tok, const uint16_t* __restrict__ emb, int h,
                             float* __restrict__ x) {
  const int t = blockIdx.x;
  const uint16_t* src = emb + size_t(tok[t]) * h;
  for (int c = threadIdx.x; c < h; c += blockDim.x) x[size_t(t) * h + c] = bf2f(src[c]);
}

// ---------------------------------------------------------------- RoPE + append
// One block per verify row (r, i). Rotate-half RoPE at position
// prefix[r] + depth(i); angles in fp64 so long positions stay accurate.
__global__ void rope_append_kernel(const uint16_t* __restrict__ qkv, const int32_t* __restrict__ prefix,
                                   const int32_t* __restrict__ parent, int n, int n_q, int n_kv, int d, int s_max,
                                   double theta, uint16_t* __restrict__ q_out, uint16_t* __restrict__ kc,
                                   uint16_t* __restrict__ vc, const int32_t* __restrict__ bt, int max_pages) {
  const int row = blockIdx.x;
  const int r = row / n, i = row % n;
  int depth = i;
  if (parent) {
    depth = 0;
    int cur = i;
    while (cur > 0 && depth <= n) {
      cur = parent[size_t(r) * n + cur];
      ++depth;
    }
  }
  const int pos = prefix[r] + depth;
  const int slot = prefix[r] + i;
  const int half = d / 2;
  const int width = (n_q + 2 * n_kv) * d;
  const uint16_t* src = qkv + size_t(row) * width;
  // the row's rotation angles, once per frequency (fp64 angle, fp32 cos/sin)
  __shared__ float cs_sh[64], sn_sh[64];
  for (int j = threadIdx.x; j < half; j += blockDim.x) {
    const double inv = pow(theta, -2.0 * j / double(d));
    double sn, cs;
    sincos(double(pos) * inv, &sn, &cs);
    cs_sh[j] = float(cs);
    sn_sh[j] = float(sn);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < (n_q + n_kv) * half; e += blockDim.x) {
    const int head = e / half, j = e % half;
    const float c = cs_sh[j], s = sn_sh[j];
    const float a = bf2f(src[head * d + j]), b = bf2f(src[head * d + j + half]);
    const uint16_t o0 = f2bf(a * c - b * s), o1 = f2bf(b * c + a * s);
    if (head < n_q) {
      uint16_t* dst = q_out + (size_t(row) * n_q + head) * d;
      dst[j] = o0;
      dst[j + half] = o1;
    } else {
      const long long kr = kv_row(bt, max_pages, r, head - n_q, slot, n_kv, s_max);
      if (kr < 0) continue;
      uint16_t* dst = kc + size_t(kr) * d;
      dst[j] = o0;
      dst[j + half] = o1;
    }
  }
  for (int e = threadIdx.x; e < n_kv * d; e += blockDim.x) {
    const int hk = e / d, c = e % d;
    const long long vr = kv_row(bt, max_pages, r, hk, slot, n_kv, s_max);
    if (vr >= 0) vc[size_t(vr) * d + c] = src[(n_q + n_kv) * d + e];
  }
}

// ---------------------------------------------------------------- K6
__global__ void argmax_reduce_kernel(const float* __restrict__ val, const int32_t* __restrict__ idx, int rows,
                                     int parts, int32_t* target) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (warp >= rows) return;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int p = lane; p < parts; p += 32) {
    const float v = val[size_t(warp) * parts + p];
    const int i = idx[size_t(warp) * parts + p];
    if (v > best || (v == best && i < bi)) { best = v; bi = i; }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  if (lane == 0) target[warp] = bi;
}

__global__ void argmax_rows_kernel(const float* __restrict__ logits, int V, int32_t* target) {
  const int row = blockIdx.x;
  const float* l = logits + size_t(row) * V;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const float x = l[v];
    if (x > best || (x == best && v < bi)) { best = x; bi = v; }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  if (threadIdx.x % 32 == 0) { sv[threadIdx.x / 32] = best; si[threadIdx.x / 32] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < int(blockDim.x / 32); ++w)
      if (sv[w] > best || (sv[w] == best && si[w] < bi)) { best = sv[w]; bi = si[w]; }
    target[row] = bi;
  }
}

// Greedy verification, one thread per request (n <= 64). Restates
// specdec.hpp:65-76 with the draw replaced by token == argmax(parent row):
// longest accepted root path, children scanned in id order so ties resolve
// to the lower node id; committed = accepted + 1.
__global__ void greedy_accept_kernel(const int32_t* __restrict__ tokens, const int32_t* __restrict__ target,
                                     const int32_t* __restrict__ parent, int b, int n, int32_t* acc_len,
                                     int32_t* bonus, int32_t* keep) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= b) return;
  const int32_t* tok = tokens + size_t(r) * n;
  const int32_t* tgt = target + size_t(r) * n;
  int8_t best[64], depth[64];
  for (int i = n - 1; i >= 0; --i) {
    best[i] = -1;
    depth[i] = 0;
    for (int c = i + 1; c < n; ++c) {
      const int pc = parent ? parent[size_t(r) * n + c] : c - 1;
      if (pc != i || tok[c] != tgt[i]) continue;
      if (1 + depth[c] > depth[i]) {
        depth[i] = int8_t(1 + depth[c]);
        best[i] = int8_t(c);
      }
    }
  }
  int cur = 0, a = 0;
  if (keep) keep[size_t(r) * n] = 0;
  while (best[cur] >= 0) {
    cur = best[cur];
    ++a;
    if (keep) keep[size_t(r) * n + a] = cur;
  }
  if (keep)
    for (int i = a + 1; i < n; ++i) keep[size_t(r) * n + i] = -1;
  acc_len[r] = a;
  bonus[r] = tgt[cur];
}

// Tree KV compaction: row keep[r, j] -> prefix + j, j ascending (keep[j] >= j,
// so no source is overwritten before it is read). One block per (layer, r, h).
__global__ void kv_rollback_kernel(void* const* kcs, void* const* vcs, const int32_t* prefix, const int32_t* acc,
                                   const int32_t* keep, int b, int n, int n_kv, int d, int s_max, const int32_t* bt,
                                   int max_pages) {
  const int layer = blockIdx.z, r = blockIdx.y, h = blockIdx.x;
  const int a = acc[r], p = prefix[r];
  uint16_t* kc = reinterpret_cast<uint16_t*>(kcs[layer]);
  uint16_t* vc = reinterpret_cast<uint16_t*>(vcs[layer]);
  for (int j = 1; j <= a; ++j) {
    const int src = keep[size_t(r) * n + j];
    const long long rd = kv_row(bt, max_pages, r, h, p + j, n_kv, s_max);
    const long long rs = kv_row(bt, max_pages, r, h, p + src, n_kv, s_max);
    if (src != j && rd >= 0 && rs >= 0)
      for (int c = threadIdx.x; c < d; c += blockDim.x) {
        kc[size_t(rd) * d + c] = kc[size_t(rs) * d + c];
        vc[size_t(rd) * d + c] = vc[size_t(rs) * d + c];
      }
    __syncthreads();
  }
}

__global__ void kv_len_kernel(const int32_t* prefix, const int32_t* acc, int b, int32_t* kv_len) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < b) kv_len[r] = prefix[r] + acc[r] + 1;
}

// Compact draft mask: bit j of row (r,i) = draft j is an ancestor-or-self of
// draft i (chain: j <= i) — CompactMask::chain generalised to trees
// (attention.hpp:52-57).
__global__ void build_mask_kernel(const int32_t* __restrict__ parent, int b, int n, uint64_t* mask) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= b * n) return;
  const int r = row / n, i = row % n;
  uint64_t m = 0;
  if (!parent) {
    m = (i >= 63) ? ~0ull : ((1ull << (i + 1)) - 1ull);
  } else {
    int cur = i, guard = 0;
    while (cur >= 0 && guard <= n) {
      m |= 1ull << cur;
      cur = (cur == 0) ? -1 : parent[size_t(r) * n + cur];
      ++guard;
    }
  }
  mask[row] = m;
}


// ---------------------------------------------------------------- decode loop
// (draft -> verify -> accept -> commit, all on device so a
// decode iteration needs no host round trip)

// tokens[r*n] = root[r]; planted drafts (test/bench input) fill rows 1..k.
__global__ void decode_prep_kernel(const int32_t* __restrict__ root, const int32_t* __restrict__ drafts, int b,
                                   int n, int32_t* __restrict__ tokens) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b * n) return;
  const int r = i / n, j = i % n;
  if (j == 0) tokens[i] = root[r];
  else if (drafts) tokens[i] = drafts[size_t(r) * (n - 1) + (j - 1)];
}

// Draft step t: input token tokens[r*n + t] at position kv_len[r] + t.
__global__ void draft_io_kernel(const int32_t* __restrict__ tokens, const int32_t* __restrict__ kv_len, int t, int b,
                                int n, int32_t* __restrict__ tok_in, int32_t* __restrict__ pos) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= b) return;
  tok_in[r] = tokens[size_t(r) * n + t];
  pos[r] = kv_len[r] + t;
}

__global__ void draft_scatter_kernel(const int32_t* __restrict__ out, int b, int n, int t, int32_t* __restrict__ tokens) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < b) tokens[size_t(r) * n + t + 1] = out[r];
}

// Commit the greedy verdict of a chain step: accepted drafts d_1..d_a and the
// bonus token are appended to the history (committed = a + 1, config.hpp:69-70);
// the chain's K/V rows root..d_a are already in place, so kv_len += a + 1 and
// the bonus becomes the next root.
// keep (trees): the accepted root path's node ids (greedy_accept); its K/V
// rows were compacted to kv_len + j by kv_rollback before this runs.
__global__ void decode_commit_kernel(const int32_t* __restrict__ tokens, const int32_t* __restrict__ acc,
                                     const int32_t* __restrict__ bonus, const int32_t* __restrict__ keep, int b, int n,
                                     int cap, int32_t* hist, int32_t* hist_n, int32_t* kv_len, int32_t* root) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= b) return;
  const int a = acc[r];
  int h = hist_n[r];
  int32_t* dst = hist + size_t(r) * cap;
  for (int j = 1; j <= a; ++j)
    if (h < cap) dst[h++] = tokens[size_t(r) * n + (keep ? keep[size_t(r) * n + j] : j)];
  if (h < cap) dst[h++] = bonus[r];
  hist_n[r] = h;
  kv_len[r] += a + 1;
  root[r] = bonus[r];
}

// Prefill: copy the residual row of each request's last prompt token
// (position len-1; rows are chunk-major: ((c*b + r)*C + i)) to row r.
__global__ void prefill_last_kernel(const float* __restrict__ x, const int32_t* __restrict__ len, int b, int C, int h,
                                    float* __restrict__ out) {
  const int r = blockIdx.x;
  const int p = len[r] - 1, c = p / C, i = p % C;
  const float* src = x + (size_t(c * b + r) * C + i) * h;
  for (int j = threadIdx.x; j < h; j += blockDim.x) out[size_t(r) * h + j] = src[j];
}

inline int grid_for(uint64_t n, int block) {
  const uint64_t g = (n + block - 1) / block;
  return int(g > 148ull * 32 ? 148ull * 32 : (g ? g : 1));
}

}  // namespace

// ---------------------------------------------------------------- launchers
void fill_uniform(void* dst, uint64_t count, uint64_t seed, uint64_t tensor_id, uint64_t base, float scale,
                  cudaStream_t st) {
  if (!count) return;
  SMO_REQUIRE(dst, "fill: null pointer");
  const float s = std::ldexp(scale, -24);
  fill_uniform_kernel<<<grid_for(count, 256), 256, 0, st>>>(reinterpret_cast<uint16_t*>(dst), count,
                                                            seed ^ (tensor_id * 0x9e3779b97f4a7c15ULL), base, s);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void fill_normal(void* dst, uint64_t count, uint64_t seed, uint64_t tensor_id, uint64_t base, float scale,
                 cudaStream_t st) {
  if (!count) return;
  SMO_REQUIRE(dst, "fill: null pointer");
  const float s = std::ldexp(scale, -24);
  fill_normal_kernel<<<grid_for(count, 256), 256, 0, st>>>(reinterpret_cast<uint16_t*>(dst), count,
                                                           seed ^ (tensor_id * 0x9e3779b97f4a7c15ULL), base, s);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void fill_kv_prefix(void* cache, const int32_t* prefix, int b, int n_kv, int d, int s_max, uint64_t seed,
                    uint64_t tensor_id, cudaStream_t st, const int32_t* bt, int max_pages) {
  SMO_REQUIRE(cache && prefix && b > 0 && n_kv > 0 && d > 0, "fill_kv_prefix: bad arguments");
  dim3 grid(64, b * n_kv);
  fill_kv_prefix_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<uint16_t*>(cache), prefix, n_kv, d, s_max,
                                              seed ^ (tensor_id * 0x9e3779b97f4a7c15ULL), std::ldexp(1.0f, -24),
                                              bt, max_pages);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void router_topk(const void* x, const void* w, int T, int h, int E, int k, float* logits, int32_t* ids,
                 float* weights, cudaStream_t st) {
  SMO_REQUIRE(x && w && ids && weights, "router: null pointer");
  SMO_REQUIRE(h % 256 == 0, "router: h must be a multiple of 256");
  SMO_REQUIRE(E >= 1 && E <= kMaxExperts && k >= 1 && k <= kMaxTopK && k <= E, "router: bad E/k");
  if (T <= 0) return;
  const int warps = std::min(E, 8);
  router_topk_kernel<<<T, 32 * warps, 0, st>>>(reinterpret_cast<const uint16_t*>(x),
                                              reinterpret_cast<const uint16_t*>(w), T, h, E, k, logits, ids, weights);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void permute(const int32_t* ids, int T, int k, int E, const void* x, int h, int32_t* offsets, int32_t* perm,
             int32_t* pos, void* xp, cudaStream_t st) {
  SMO_REQUIRE(ids && offsets && perm && pos, "permute: null pointer");
  SMO_REQUIRE(E >= 1 && E <= kMaxExperts, "permute: bad E");
  const int P = T * k;
  permute_kernel<<<1, 1024, P <= kPermuteSmemIds ? size_t(P) * 4 : 0, st>>>(ids, P, E, offsets, perm, pos);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
  if (x && xp && P > 0) {
    SMO_REQUIRE(h % 8 == 0, "permute: h must be a multiple of 8");
    gather_rows_kernel<<<P, 128, 0, st>>>(reinterpret_cast<const uint16_t*>(x), perm, k, h, P,
                                          reinterpret_cast<uint16_t*>(xp));
    count_launch();
    SMO_CUDA_CHECK(cudaGetLastError());
  }
}

void unpermute_combine(const float* y, const int32_t* pos, const float* w, int T, int k, int h, float* res,
                       cudaStream_t st, int splits, size_t split_stride) {
  SMO_REQUIRE(y && pos && w && res, "combine: null pointer");
  SMO_REQUIRE(h % 4 == 0, "combine: h must be a multiple of 4");
  if (T <= 0) return;
  combine_kernel<<<T, 256, 0, st>>>(y, pos, w, T, k, h, res, std::max(1, splits), split_stride);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void rmsnorm(const float* x, const void* gain, int T, int h, float eps, void* y, cudaStream_t st) {
  SMO_REQUIRE(x && gain && y && h % 4 == 0 && h <= 256 * 4 * kRmsMaxV, "rmsnorm: bad arguments (h % 4 == 0, h <= 8192)");
  if (T <= 0) return;
  rmsnorm_kernel<<<T, 256, 0, st>>>(x, reinterpret_cast<const uint16_t*>(gain), h, eps,
                                    reinterpret_cast<uint16_t*>(y));
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void embed(const int32_t* tok, const void* emb, int T, int h, float* x, cudaStream_t st) {
  SMO_REQUIRE(tok && emb && x, "embed: null pointer");
  if (T <= 0) return;
  embed_kernel<<<T, 256, 0, st>>>(tok, reinterpret_cast<const uint16_t*>(emb), h, x);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

// RoPE + K/V append with the inverse frequencies theta^(-2j/d) computed once
// on the host in double (the oracle's own pow, oracle/oracle.c) and passed by
// value: a row only evaluates its 64 fp64 sincos, and the rotation / copies
// move bf16 pairs and 16-byte chunks instead of single values.
struct RopeInv {
  double inv[64];
};
__global__ void rope_append_v2_kernel(const uint16_t* __restrict__ qkv, const int32_t* __restrict__ prefix,
                                      const int32_t* __restrict__ parent, int n, int n_q, int n_kv, int d, int s_max,
                                      const __grid_constant__ RopeInv ri, uint16_t* __restrict__ q_out,
                                      uint16_t* __restrict__ kc, uint16_t* __restrict__ vc,
                                      const int32_t* __restrict__ bt, int max_pages) {
  const int row = blockIdx.x;
  const int r = row / n, i = row % n;
  int depth = i;
  if (parent) {
    depth = 0;
    int cur = i;
    while (cur > 0 && depth <= n) {
      cur = parent[size_t(r) * n + cur];
      ++depth;
    }
  }
  const int pos = prefix[r] + depth;
  const int slot = prefix[r] + i;
  const int half = d / 2;
  const int width = (n_q + 2 * n_kv) * d;
  const uint16_t* src = qkv + size_t(row) * width;
  __shared__ float cs_sh[64], sn_sh[64];
  for (int j = threadIdx.x; j < half; j += blockDim.x) {
    double sn, cs;
    sincos(double(pos) * ri.inv[j], &sn, &cs);
    cs_sh[j] = float(cs);
    sn_sh[j] = float(sn);
  }
  __syncthreads();
  const int hp = half / 2;  // bf16 pairs per half head
  for (int e = threadIdx.x; e < (n_q + n_kv) * hp; e += blockDim.x) {
    const int head = e / hp, j = 2 * (e % hp);
    const uint32_t a2 = *reinterpret_cast<const uint32_t*>(src + head * d + j);
    const uint32_t b2 = *reinterpret_cast<const uint32_t*>(src + head * d + j + half);
    const float a0 = __uint_as_float(a2 << 16), a1 = __uint_as_float(a2 & 0xffff0000u);
    const float b0 = __uint_as_float(b2 << 16), b1 = __uint_as_float(b2 & 0xffff0000u);
    const float c0 = cs_sh[j], s0 = sn_sh[j], c1 = cs_sh[j + 1], s1 = sn_sh[j + 1];
    const uint32_t o0 = uint32_t(f2bf(a0 * c0 - b0 * s0)) | (uint32_t(f2bf(a1 * c1 - b1 * s1)) << 16);
    const uint32_t o1 = uint32_t(f2bf(b0 * c0 + a0 * s0)) | (uint32_t(f2bf(b1 * c1 + a1 * s1)) << 16);
    uint16_t* dst;
    if (head < n_q) {
      dst = q_out + (size_t(row) * n_q + head) * d;
    } else {
      const long long kr = kv_row(bt, max_pages, r, head - n_q, slot, n_kv, s_max);
      if (kr < 0) continue;
      dst = kc + size_t(kr) * d;
    }
    *reinterpret_cast<uint32_t*>(dst + j) = o0;
    *reinterpret_cast<uint32_t*>(dst + j + half) = o1;
  }
  for (int e = threadIdx.x; e < n_kv * (d / 8); e += blockDim.x) {  // V rows: 16-byte chunks
    const int hk = e / (d / 8), c = 8 * (e % (d / 8));
    const long long vr = kv_row(bt, max_pages, r, hk, slot, n_kv, s_max);
    if (vr >= 0)
      *reinterpret_cast<uint4*>(vc + size_t(vr) * d + c) =
          *reinterpret_cast<const uint4*>(src + (n_q + n_kv) * d + hk * d + c);
  }
}

void rope_append(const void* qkv, const int32_t* prefix, const int32_t* parent, int b, int n, int n_q, int n_kv,
                 int d, int s_max, float theta, void* q_out, void* kc, void* vc, cudaStream_t st, const int32_t* bt,
                 int max_pages) {
  SMO_REQUIRE(qkv && prefix && q_out && kc && vc, "rope_append: null pointer");
  SMO_REQUIRE(d % 2 == 0 && d <= 128, "rope_append: head_dim must be even and <= 128");
  static const bool v1 = [] {  // A/B: SMO_ROPE_V1=1 -> the per-row fp64 pow kernel
    const char* f = std::getenv("SMO_ROPE_V1");
    return f && f[0] == '1';
  }();
  if (v1 || d % 4 != 0) {
    rope_append_kernel<<<b * n, 256, 0, st>>>(reinterpret_cast<const uint16_t*>(qkv), prefix, parent, n, n_q, n_kv,
                                              d, s_max, double(theta), reinterpret_cast<uint16_t*>(q_out),
                                              reinterpret_cast<uint16_t*>(kc), reinterpret_cast<uint16_t*>(vc), bt,
                                              max_pages);
  } else {
    RopeInv ri{};
    for (int j = 0; j < d / 2; ++j) ri.inv[j] = std::pow(double(theta), -2.0 * j / double(d));
    rope_append_v2_kernel<<<b * n, 256, 0, st>>>(reinterpret_cast<const uint16_t*>(qkv), prefix, parent, n, n_q,
                                                 n_kv, d, s_max, ri, reinterpret_cast<uint16_t*>(q_out),
                                                 reinterpret_cast<uint16_t*>(kc), reinterpret_cast<uint16_t*>(vc), bt,
                                                 max_pages);
  }
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void argmax_reduce(const float* val, const int32_t* idx, int rows, int parts, int32_t* target, cudaStream_t st) {
  SMO_REQUIRE(val && idx && target, "argmax: null pointer");
  if (rows <= 0) return;
  argmax_reduce_kernel<<<(rows * 32 + 255) / 256, 256, 0, st>>>(val, idx, rows, parts, target);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void argmax_rows(const float* logits, int rows, int V, int32_t* target, cudaStream_t st) {
  SMO_REQUIRE(logits && target, "argmax: null pointer");
  if (rows <= 0) return;
  argmax_rows_kernel<<<rows, 256, 0, st>>>(logits, V, target);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void greedy_accept(const int32_t* tokens, const int32_t* target, const int32_t* parent, int b, int n,
                   int32_t* acc_len, int32_t* bonus, int32_t* keep, cudaStream_t st) {
  SMO_REQUIRE(tokens && target && acc_len && bonus, "accept: null pointer");
  SMO_REQUIRE(n >= 1 && n <= 64, "accept: n must be in [1, 64]");
  if (b <= 0) return;
  greedy_accept_kernel<<<(b + 63) / 64, 64, 0, st>>>(tokens, target, parent, b, n, acc_len, bonus, keep);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void build_mask(const int32_t* parent, int b, int n, uint64_t* mask, cudaStream_t st) {
  SMO_REQUIRE(mask && n >= 1 && n <= 64, "build_mask: bad arguments");
  build_mask_kernel<<<(b * n + 127) / 128, 128, 0, st>>>(parent, b, n, mask);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void kv_rollback(void* const* kcs, void* const* vcs, int n_layers, const int32_t* prefix, const int32_t* acc,
                 const int32_t* keep, int b, int n, int n_kv, int d, int s_max, int32_t* kv_len, cudaStream_t st,
                 const int32_t* bt, int max_pages) {
  SMO_REQUIRE(prefix && acc, "kv_rollback: null pointer");
  if (keep && kcs && vcs && n_layers > 0) {
    dim3 grid(n_kv, b, n_layers);
    kv_rollback_kernel<<<grid, 128, 0, st>>>(kcs, vcs, prefix, acc, keep, b, n, n_kv, d, s_max, bt, max_pages);
    count_launch();
    SMO_CUDA_CHECK(cudaGetLastError());
  }
  if (kv_len) {
    kv_len_kernel<<<(b + 127) / 128, 128, 0, st>>>(prefix, acc, b, kv_len);
    count_launch();
    SMO_CUDA_CHECK(cudaGetLastError());
  }
}

void decode_prep(const int32_t* root, const int32_t* drafts, int b, int n, int32_t* tokens, cudaStream_t st) {
  decode_prep_kernel<<<(b * n + 127) / 128, 128, 0, st>>>(root, drafts, b, n, tokens);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void draft_io(const int32_t* tokens, const int32_t* kv_len, int t, int b, int n, int32_t* tok_in, int32_t* pos,
              cudaStream_t st) {
  draft_io_kernel<<<(b + 127) / 128, 128, 0, st>>>(tokens, kv_len, t, b, n, tok_in, pos);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void draft_scatter(const int32_t* out, int b, int n, int t, int32_t* tokens, cudaStream_t st) {
  draft_scatter_kernel<<<(b + 127) / 128, 128, 0, st>>>(out, b, n, t, tokens);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void decode_commit(const int32_t* tokens, const int32_t* acc, const int32_t* bonus, int b, int n, int cap,
                   int32_t* hist, int32_t* hist_n, int32_t* kv_len, int32_t* root, cudaStream_t st,
                   const int32_t* keep) {
  decode_commit_kernel<<<(b + 127) / 128, 128, 0, st>>>(tokens, acc, bonus, keep, b, n, cap, hist, hist_n, kv_len,
                                                        root);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void prefill_last(const float* x, const int32_t* len, int b, int C, int h, float* out, cudaStream_t st) {
  prefill_last_kernel<<<b, 256, 0, st>>>(x, len, b, C, h, out);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

}  // namespace smo
