// cpu_attn.cpp — host verification attention for AttentionPlacement::CPU
// (SURVEY.md §8 f4). One work item = one (chunk, request, KV head) pair: its
// g*n query rows share every K/V row they read, so each K and V row is
// converted to fp32 once and reused by all rows (the HBM-style reuse of K1,
// here against host DRAM bandwidth). Compiled with -O3 -mavx2 -mfma; the
// inner products use GCC vector extensions (8 x fp32 = one AVX register).
#include "cpu_attn.h"

#include <algorithm>
#include <cmath>
#include <cstring>

namespace smo {

namespace {

typedef float v8f __attribute__((vector_size(32)));
typedef uint32_t v8u __attribute__((vector_size(32)));
typedef uint16_t v8h __attribute__((vector_size(16)));

inline float bf(uint16_t h) {
  uint32_t u = uint32_t(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

inline uint16_t to_bf(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return uint16_t((u >> 16) | 0x40u);
  u += 0x7fffu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}

// 8 bf16 -> 8 fp32
inline v8f widen(const uint16_t* p) {
  v8h h;
  std::memcpy(&h, p, 16);
  const v8u u = __builtin_convertvector(h, v8u) << 16;
  v8f f;
  std::memcpy(&f, &u, 32);
  return f;
}

inline float hsum(v8f v) {
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += v[i];
  return s;
}

struct Scratch {
  std::vector<v8f> qf, o, kf;  // 32-byte aligned (C++17 aligned new)
  std::vector<float> s;
};
thread_local Scratch tls;

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
  const float scale = 1.0f / std::sqrt(float(d));
  Scratch& sc = tls;
  const v8f zero = {0, 0, 0, 0, 0, 0, 0, 0};
  sc.qf.resize(size_t(rows) * dv);
  sc.o.assign(size_t(rows) * dv, zero);
  sc.s.resize(size_t(rows) * keys);
  sc.kf.resize(size_t(dv));
  // query rows (i, hh) -> row i*g + hh, pre-scaled
  const v8f sv = {scale, scale, scale, scale, scale, scale, scale, scale};
  for (int i = 0; i < a.n; ++i)
    for (int hh = 0; hh < g; ++hh) {
      const uint16_t* src = a.q + ((row0 + size_t(r) * a.n + i) * a.n_q + size_t(h) * g + hh) * d;
      v8f* dst = sc.qf.data() + size_t(i * g + hh) * dv;
      for (int e = 0; e < dv; ++e) dst[e] = widen(src + 8 * e) * sv;
    }
  const uint16_t* kbase = a.k_cache + (size_t(r) * a.n_kv + h) * a.s_max * d;
  const uint16_t* vbase = a.v_cache + (size_t(r) * a.n_kv + h) * a.s_max * d;
  const uint64_t* mrow = a.mask + size_t(r) * a.n;  // one [b*n] mask shared by every chunk
  auto visible = [&](int i, int j) {
    if (j < prefix) return true;
    const int dj = j - prefix;
    return dj < 64 && ((mrow[i] >> dj) & 1ull);
  };
  // S = Q K^T over the visible keys (key-major: each K row widened once)
  v8f* kf = sc.kf.data();
  for (int j = 0; j < keys; ++j) {
    for (int e = 0; e < dv; ++e) kf[e] = widen(kbase + size_t(j) * d + 8 * e);
    for (int row = 0; row < rows; ++row) {
      const v8f* qv = sc.qf.data() + size_t(row) * dv;
      v8f acc = zero;
      for (int e = 0; e < dv; ++e) acc += qv[e] * kf[e];
      sc.s[size_t(row) * keys + j] = hsum(acc);
    }
  }
  // softmax per row (masked keys contribute nothing)
  std::vector<float> inv(static_cast<size_t>(rows));
  for (int row = 0; row < rows; ++row) {
    const int i = row / g;
    float* s = sc.s.data() + size_t(row) * keys;
    float m = -INFINITY;
    for (int j = 0; j < keys; ++j)
      if (visible(i, j)) m = std::max(m, s[j]);
    float sum = 0.f;
    for (int j = 0; j < keys; ++j) {
      const float p = visible(i, j) ? std::exp(s[j] - m) : 0.f;
      s[j] = p;
      sum += p;
    }
    inv[size_t(row)] = sum > 0.f ? 1.f / sum : 0.f;
  }
  // O = P V (key-major: each V row widened once)
  for (int j = 0; j < keys; ++j) {
    for (int e = 0; e < dv; ++e) kf[e] = widen(vbase + size_t(j) * d + 8 * e);
    for (int row = 0; row < rows; ++row) {
      const float p = sc.s[size_t(row) * keys + j];
      if (p == 0.f) continue;
      v8f* ov = sc.o.data() + size_t(row) * dv;
      const v8f pv = {p, p, p, p, p, p, p, p};
      for (int e = 0; e < dv; ++e) ov[e] += pv * kf[e];
    }
  }
  for (int i = 0; i < a.n; ++i)
    for (int hh = 0; hh < g; ++hh) {
      const int row = i * g + hh;
      uint16_t* dst = a.out + ((row0 + size_t(r) * a.n + i) * a.n_q + size_t(h) * g + hh) * d;
      const v8f* o = sc.o.data() + size_t(row) * dv;
      for (int e = 0; e < d; ++e) dst[e] = to_bf(o[e / 8][e % 8] * inv[size_t(row)]);
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
