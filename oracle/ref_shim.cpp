// ref_shim.cpp — extern "C" wrappers around the UNMODIFIED reference headers
// (/root/reference/proj/include/moeplan/*.hpp), compiled by oracle/Makefile
// into oracle/_ref/libmoeplan_ref.so. TEST INFRASTRUCTURE ONLY: used to
// generate golden vectors (oracle/gen_golden.py), to cross-check the C
// restatement in oracle.c, and as the timed reference CPU arm in bench.py.
// Nothing here is copied from the reference; it only calls its API.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "moeplan/attention.hpp"
#include "moeplan/specdec.hpp"

namespace {
thread_local std::string g_err;

moeplan::Matrix to_matrix(const double* p, std::size_t r, std::size_t c) {
  moeplan::Matrix m(r, c);
  if (r * c) std::memcpy(m.data.data(), p, sizeof(double) * r * c);
  return m;
}

float bf16f(std::uint16_t h) {
  std::uint32_t u = std::uint32_t(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::uint64_t ref_splitmix64(std::uint64_t x) { return moeplan::detail::splitmix64(x); }

void ref_trial_stream(std::uint64_t seed, std::size_t count, double* out) {
  moeplan::detail::TrialRng rng(seed);
  for (std::size_t i = 0; i < count; ++i) out[i] = rng.uniform();
}

double ref_mask_memory_savings(std::size_t n, std::size_t p) {
  try {
    return moeplan::mask_memory_savings(n, p);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

// Returns 0 on success, 1 on std::invalid_argument (message in ref_last_error).
int ref_chunked_attention(std::size_t n, std::size_t p, std::size_t d,
                          const double* Q, const double* K, const double* V,
                          std::size_t mask_n, const std::uint8_t* mask,
                          double* out) {
  try {
    moeplan::AttentionInstance inst;
    inst.n = n;
    inst.prefix_len = p;
    inst.d = d;
    inst.Q = to_matrix(Q, n, d);
    inst.K = to_matrix(K, p + n, d);
    inst.V = to_matrix(V, p + n, d);
    moeplan::CompactMask m(mask_n);
    for (std::size_t i = 0; i < mask_n; ++i)
      for (std::size_t j = 0; j < mask_n; ++j) m.set(i, j, mask[i * mask_n + j] != 0);
    moeplan::Matrix o = moeplan::chunked_attention(inst, m);
    std::memcpy(out, o.data.data(), sizeof(double) * n * d);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int ref_naive_oracle(std::size_t n, std::size_t p, std::size_t d,
                     const double* Q, const double* K, const double* V,
                     const std::uint8_t* full, double* out) {
  try {
    moeplan::AttentionInstance inst;
    inst.n = n;
    inst.prefix_len = p;
    inst.d = d;
    inst.Q = to_matrix(Q, n, d);
    inst.K = to_matrix(K, p + n, d);
    inst.V = to_matrix(V, p + n, d);
    std::vector<bool> fm(n * (p + n));
    for (std::size_t i = 0; i < fm.size(); ++i) fm[i] = full[i] != 0;
    moeplan::Matrix o = moeplan::naive_oracle(inst, fm);
    std::memcpy(out, o.data.data(), sizeof(double) * n * d);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int ref_simulate_tokens(const double* probs, std::size_t n_probs, int k,
                        std::int64_t trials, std::uint64_t seed, double* mean,
                        double* stdev) {
  try {
    std::vector<double> p(probs, probs + n_probs);
    auto r = moeplan::simulate_tokens(p, k, trials, seed);
    *mean = r.mean_committed;
    *stdev = r.std_committed;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Reference CPU verify attention for one layer: the unmodified fp64
// moeplan::chunked_attention, one call per (request, query head) — the
// paper's CPU-attention placement — spread over `threads`
// std::threads. Inputs are the bf16 GPU-layout tensors; instances are built
// outside the timed region. Returns the seconds spent in chunked_attention
// calls (wall clock of the parallel region), or -1 on error. out may be NULL.
double ref_verify_layer_attention(const std::uint16_t* q, const std::uint16_t* kc,
                                  const std::uint16_t* vc, const std::uint64_t* mask,
                                  const std::int32_t* prefix, int b, int n, int n_q,
                                  int n_kv, int d, int s_max, int threads,
                                  double* out) {
  try {
    const int g = n_q / n_kv;
    struct Item {
      moeplan::AttentionInstance inst;
      moeplan::CompactMask mask;
      int r, hq;
    };
    std::vector<Item> items(std::size_t(b) * n_q);
    for (int r = 0; r < b; ++r)
      for (int hq = 0; hq < n_q; ++hq) {
        Item& it = items[std::size_t(r) * n_q + hq];
        it.r = r;
        it.hq = hq;
        const std::size_t p = std::size_t(prefix[r]);
        it.inst.n = std::size_t(n);
        it.inst.prefix_len = p;
        it.inst.d = std::size_t(d);
        it.inst.Q = moeplan::Matrix(std::size_t(n), std::size_t(d));
        it.inst.K = moeplan::Matrix(p + n, std::size_t(d));
        it.inst.V = moeplan::Matrix(p + n, std::size_t(d));
        for (int i = 0; i < n; ++i)
          for (int c = 0; c < d; ++c)
            it.inst.Q.at(i, c) = bf16f(q[((std::size_t(r) * n + i) * n_q + hq) * d + c]);
        const std::size_t base = (std::size_t(r) * n_kv + hq / g) * std::size_t(s_max) * d;
        for (std::size_t j = 0; j < (p + n) * std::size_t(d); ++j) {
          it.inst.K.data[j] = bf16f(kc[base + j]);
          it.inst.V.data[j] = bf16f(vc[base + j]);
        }
        it.mask = moeplan::CompactMask(std::size_t(n));
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < n; ++j)
            it.mask.set(i, j, (mask[std::size_t(r) * n + i] >> j) & 1u);
      }
    std::vector<moeplan::Matrix> outs(items.size());
    std::vector<std::string> errs(std::size_t(threads > 0 ? threads : 1));
    const int nt = threads > 0 ? threads : 1;
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int w = 0; w < nt; ++w)
      pool.emplace_back([&, w] {
        try {
          for (std::size_t i = std::size_t(w); i < items.size(); i += std::size_t(nt))
            outs[i] = moeplan::chunked_attention(items[i].inst, items[i].mask);
        } catch (const std::exception& e) {
          errs[std::size_t(w)] = e.what();
        }
      });
    for (auto& th : pool) th.join();
    auto t1 = std::chrono::steady_clock::now();
    for (auto& e : errs)
      if (!e.empty()) throw std::invalid_argument(e);
    if (out)
      for (std::size_t i = 0; i < items.size(); ++i)
        for (int row = 0; row < n; ++row)
          for (int c = 0; c < d; ++c)
            out[((std::size_t(items[i].r) * n + row) * n_q + items[i].hq) * d + c] =
                outs[i].at(std::size_t(row), std::size_t(c));
    return std::chrono::duration<double>(t1 - t0).count();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

}  // extern "C"
