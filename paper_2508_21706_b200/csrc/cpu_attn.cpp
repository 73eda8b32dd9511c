// cpu_attn.cpp — host verification attention for AttentionPlacement::CPU
// (SURVEY.md §8 f4). One work item = one (chunk, request, KV head) pair: its
// g*n query rows share every K/V row they read, so each K and V row is
// converted to fp32 once and reused by all rows (the HBM-style reuse of K1,
// here against host DRAM bandwidth). Compiled with -O3 -mavx2 -mfma (AVX2
// intrinsics, 8 x fp32 per register).
#include "cpu_attn.h"

#include <algorithm>
#include <cmath>
#include <cstring>

#include <immintrin.h>

namespace smo {

namespace {

inline uint16_t to_bf(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return uint16_t((u >> 16) | 0x40u);
  u += 0x7fffu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}

// 8 bf16 -> 8 fp32 (zero-extend to 32 bits, shift into the high half)
inline __m256 widen(const uint16_t* p) {
  const __m128i h = _mm_loadu_si128(reinterpret_cast<const __m128i*>(p));
  return _mm256_castsi256_ps(_mm256_slli_epi32(_mm256_cvtepu16_epi32(h), 16));
}

// lane k of the result = horizontal sum of a[k] (8 dot products at once)
inline __m256 hsum8(const __m256* a) {
  const __m256 h01 = _mm256_hadd_ps(a[0], a[1]), h23 = _mm256_hadd_ps(a[2], a[3]);
  const __m256 h45 = _mm256_hadd_ps(a[4], a[5]), h67 = _mm256_hadd_ps(a[6], a[7]);
  const __m256 g0 = _mm256_hadd_ps(h01, h23), g1 = _mm256_hadd_ps(h45, h67);
  return _mm256_add_ps(_mm256_permute2f128_ps(g0, g1, 0x20), _mm256_permute2f128_ps(g0, g1, 0x31));
}

// exp(x) for x <= 0 (scores minus the row maximum): 2^n * 2^f with a
// degree-6 polynomial for 2^f on [0, 1) (rel. error ~2e-7, far below the
// bf16 output rounding); x < -87 flushes to 0
inline __m256 exp_neg(__m256 x) {
  const __m256 t = _mm256_mul_ps(_mm256_max_ps(x, _mm256_set1_ps(-87.0f)), _mm256_set1_ps(1.44269504088896341f));
  const __m256 n = _mm256_floor_ps(t);
  const __m256 f = _mm256_sub_ps(t, n);
  __m256 p = _mm256_set1_ps(1.53532935e-4f);
  p = _mm256_fmadd_ps(p, f, _mm256_set1_ps(1.33989469e-3f));
  p = _mm256_fmadd_ps(p, f, _mm256_set1_ps(9.61817604e-3f));
  p = _mm256_fmadd_ps(p, f, _mm256_set1_ps(5.55036329e-2f));
  p = _mm256_fmadd_ps(p, f, _mm256_set1_ps(2.40226507e-1f));
  p = _mm256_fmadd_ps(p, f, _mm256_set1_ps(6.93147182e-1f));
  p = _mm256_fmadd_ps(p, f, _mm256_set1_ps(1.0f));
  const __m256i e = _mm256_slli_epi32(_mm256_cvtps_epi32(n), 23);
  const __m256 r = _mm256_castsi256_ps(_mm256_add_epi32(_mm256_castps_si256(p), e));
  return _mm256_and_ps(r, _mm256_cmp_ps(x, _mm256_set1_ps(-87.0f), _CMP_GT_OQ));
}

struct Scratch {
  std::vector<float> qf, kb;    // pre-scaled queries [rows][d]; 8 widened K/V rows [8][d]
  std::vector<float> s;         // scores / probabilities [rows][keys rounded up to 8]
  std::vector<float> o;         // fp32 output accumulators [rows][d]
};
thread_local Scratch tls;

// One (chunk, request, KV head) pair: its g*n query rows share every K/V row.
// S = Q K^T in blocks of 8 keys (each K row widened once per pair, 8 dot
// products reduced together by hsum8), a vectorised masked softmax, then
// O = P V as a small GEMM (4 query rows x 16 dims register tile per V row).
void pair_attention(const CpuAttnJob& a, int item) {
  const int g = a.n_q / a.n_kv;
  const int rows = g * a.n;
  const int pairs = a.b * a.n_kv;
  const int c = item / pairs, rem = item % pairs;
  const int r = rem / a.n_kv, h = rem % a.n_kv;
  const int d = a.d, dv = d / 8;
  const size_t row0 = size_t(c) * a.b * a.n;  // first q row of this chunk
  const int prefix = a.prefix[size_t(c) * a.b + r];
  const int keys = prefix + a.n;
  const int kp = (keys + 7) & ~7;
  const float scale = 1.0f / std::sqrt(float(d));
  Scratch& sc = tls;
  sc.qf.resize(size_t(rows) * d);
  sc.kb.resize(size_t(8) * d);
  sc.s.resize(size_t(rows) * kp);
  const int rp = (rows + 3) & ~3;
  sc.o.assign(size_t(rp) * d, 0.0f);
  const __m256 sv = _mm256_set1_ps(scale);
  for (int i = 0; i < a.n; ++i)
    for (int hh = 0; hh < g; ++hh) {
      const uint16_t* src = a.q + ((row0 + size_t(r) * a.n + i) * a.n_q + size_t(h) * g + hh) * d;
      float* dst = sc.qf.data() + size_t(i * g + hh) * d;
      for (int e = 0; e < dv; ++e) _mm256_storeu_ps(dst + 8 * e, _mm256_mul_ps(widen(src + 8 * e), sv));
    }
  const uint16_t* kbase = a.k_cache + (size_t(r) * a.n_kv + h) * a.s_max * d;
  const uint16_t* vbase = a.v_cache + (size_t(r) * a.n_kv + h) * a.s_max * d;
  const uint64_t* mrow = a.mask + size_t(r) * a.n;  // one [b*n] mask shared by every chunk
  float* kb = sc.kb.data();  // row k, dims [8e, 8e + 8) at kb + k*d + 8e
  // ---- S = Q K^T
  for (int j0 = 0; j0 < keys; j0 += 8) {
    const int nk = std::min(8, keys - j0);
    for (int k = 0; k < 8; ++k)
      for (int e = 0; e < dv; ++e)
        _mm256_storeu_ps(kb + k * d + 8 * e,
                         k < nk ? widen(kbase + size_t(j0 + k) * d + 8 * e) : _mm256_setzero_ps());
    for (int row = 0; row < rows; ++row) {
      const float* qv = sc.qf.data() + size_t(row) * d;
      __m256 acc[8];
      for (int k = 0; k < 8; ++k) acc[k] = _mm256_setzero_ps();
      for (int e = 0; e < dv; ++e) {
        const __m256 qe = _mm256_loadu_ps(qv + 8 * e);
        for (int k = 0; k < 8; ++k) acc[k] = _mm256_fmadd_ps(qe, _mm256_loadu_ps(kb + k * d + 8 * e), acc[k]);
      }
      _mm256_storeu_ps(sc.s.data() + size_t(row) * kp + j0, hsum8(acc));
    }
  }
  // ---- softmax per row: prefix keys are all visible; the n draft columns
  // follow the compact mask (attention.hpp:128-154); padding columns -> 0
  std::vector<float> inv(static_cast<size_t>(rows));
  const __m256 ninf = _mm256_set1_ps(-INFINITY);
  for (int row = 0; row < rows; ++row) {
    const int i = row / g;
    float* s = sc.s.data() + size_t(row) * kp;
    for (int j = prefix; j < kp; ++j) {
      const int dj = j - prefix;
      if (j >= keys || dj >= 64 || !((mrow[i] >> dj) & 1ull)) s[j] = -INFINITY;
    }
    __m256 mv = ninf;
    for (int j = 0; j < kp; j += 8) mv = _mm256_max_ps(mv, _mm256_loadu_ps(s + j));
    float m = -INFINITY;
    alignas(32) float tmp[8];
    _mm256_store_ps(tmp, mv);
    for (int t = 0; t < 8; ++t) m = std::max(m, tmp[t]);
    const __m256 mm = _mm256_set1_ps(m);
    __m256 sum = _mm256_setzero_ps();
    for (int j = 0; j < kp; j += 8) {
      const __m256 x = _mm256_loadu_ps(s + j);
      // masked (-inf) columns: x - m = -inf -> exp_neg gives exactly 0
      const __m256 p = exp_neg(_mm256_sub_ps(x, mm));
      _mm256_storeu_ps(s + j, p);
      sum = _mm256_add_ps(sum, p);
    }
    _mm256_store_ps(tmp, sum);
    float tot = 0.f;
    for (int t = 0; t < 8; ++t) tot += tmp[t];
    inv[size_t(row)] = tot > 0.f ? 1.f / tot : 0.f;
  }
  // ---- O = P V: V rows widened once per block of 8 keys; register tiles
  // of 4 query rows x 16 dims accumulate over the block
  for (int j0 = 0; j0 < keys; j0 += 8) {
    const int nk = std::min(8, keys - j0);
    for (int k = 0; k < nk; ++k)
      for (int e = 0; e < dv; ++e) _mm256_storeu_ps(kb + k * d + 8 * e, widen(vbase + size_t(j0 + k) * d + 8 * e));
    for (int r0 = 0; r0 < rows; r0 += 4) {
      const int nr = std::min(4, rows - r0);
      const float* p0 = sc.s.data() + size_t(r0) * kp + j0;
      for (int e = 0; e < dv; e += 2) {
        __m256 acc[4][2];
        for (int t = 0; t < 4; ++t) {
          float* o = sc.o.data() + size_t(r0 + t) * d + 8 * e;
          acc[t][0] = _mm256_loadu_ps(o);
          acc[t][1] = _mm256_loadu_ps(o + 8);
        }
        for (int k = 0; k < nk; ++k) {
          const __m256 v0 = _mm256_loadu_ps(kb + k * d + 8 * e), v1 = _mm256_loadu_ps(kb + k * d + 8 * e + 8);
          for (int t = 0; t < 4; ++t) {
            const __m256 pb = _mm256_set1_ps(t < nr ? p0[size_t(t) * kp + k] : 0.f);
            acc[t][0] = _mm256_fmadd_ps(pb, v0, acc[t][0]);
            acc[t][1] = _mm256_fmadd_ps(pb, v1, acc[t][1]);
          }
        }
        for (int t = 0; t < 4; ++t) {
          float* o = sc.o.data() + size_t(r0 + t) * d + 8 * e;
          _mm256_storeu_ps(o, acc[t][0]);
          _mm256_storeu_ps(o + 8, acc[t][1]);
        }
      }
    }
  }
  for (int i = 0; i < a.n; ++i)
    for (int hh = 0; hh < g; ++hh) {
      const int row = i * g + hh;
      uint16_t* dst = a.out + ((row0 + size_t(r) * a.n + i) * a.n_q + size_t(h) * g + hh) * d;
      const float* o = sc.o.data() + size_t(row) * d;
      for (int e = 0; e < d; ++e) dst[e] = to_bf(o[e] * inv[size_t(row)]);
    }
}

}  // namespace

CpuPool::CpuPool(int threads) {
  for (int t = 0; t < std::max(1, threads); ++t) workers_.emplace_back([this] { loop(); });
}

CpuPool::~CpuPool() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& w : workers_) w.join();
}

void CpuPool::loop() {
  uint64_t seen = 0;
  for (;;) {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
    if (stop_) return;
    seen = gen_;
    while (next_ < items_) {
      const int it = next_++;
      lk.unlock();
      (*fn_)(it);
      lk.lock();
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
}

void CpuPool::run(int items, const std::function<void(int)>& fn) {
  if (items <= 0) return;
  std::unique_lock<std::mutex> lk(mu_);
  fn_ = &fn;
  items_ = items;
  next_ = 0;
  pending_ = items;
  ++gen_;
  cv_.notify_all();
  done_cv_.wait(lk, [&] { return pending_ == 0; });
  fn_ = nullptr;
}

void cpu_verify_attention(const CpuAttnJob& job, CpuPool& pool) {
  const int items = job.chunks * job.b * job.n_kv;
  pool.run(items, [&](int it) { pair_attention(job, it); });
}

}  // namespace smo
