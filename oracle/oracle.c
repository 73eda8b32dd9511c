/*
 * oracle.c — CPU restatement of the verify-step semantics.
 * TEST INFRASTRUCTURE ONLY (see oracle.h). Compiled with -ffp-contract=off so
 * that every fused multiply-add below is an explicit fmaf()/fma() call.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define PHI 0x9e3779b97f4a7c15ULL

/* specdec.hpp:34-39 */
uint64_t orc_splitmix64(uint64_t x) {
  uint64_t z = x + PHI;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* specdec.hpp:43-50 */
double orc_trial_uniform(uint64_t* state) {
  *state = orc_splitmix64(*state);
  return (double)(*state >> 11) * 0x1.0p-53;
}

/* ------------------------------------------------------------------------- */
/* attention.hpp:91-103: shape + finiteness checks, in the reference's order. */
static int check_finite(const double* a, size_t len) {
  for (size_t i = 0; i < len; ++i)
    if (!isfinite(a[i])) return 0;
  return 1;
}

static double row_dot(const double* a, const double* b, size_t d) {
  double s = 0.0;
  for (size_t c = 0; c < d; ++c) s += a[c] * b[c];
  return s;
}

/* attention.hpp:117-156. Visible columns are visited prefix-first, then the
 * mask-gated draft block; softmax is stabilised by the running row maximum
 * and normalised once; output accumulates w * V in column-visit order.       */
int orc_chunked_attention(size_t n, size_t p, size_t d, const double* Q,
                          const double* K, const double* V, size_t mask_n,
                          const uint8_t* mask, double* out) {
  const size_t total = p + n;
  if (!check_finite(Q, n * d)) return 2;
  if (!check_finite(K, total * d)) return 3;
  if (!check_finite(V, total * d)) return 4;
  if (mask_n != n) return 5;
  const double scale = 1.0 / sqrt((double)d);
  double* sc = (double*)malloc(sizeof(double) * (total ? total : 1));
  size_t* col = (size_t*)malloc(sizeof(size_t) * (total ? total : 1));
  memset(out, 0, sizeof(double) * n * d);
  int rc = 0;
  for (size_t i = 0; i < n && rc == 0; ++i) {
    size_t m = 0;
    double mx = -INFINITY;
    for (size_t j = 0; j < total; ++j) {
      if (j >= p && !mask[i * n + (j - p)]) continue;
      col[m] = j;
      sc[m] = row_dot(Q + i * d, K + j * d, d) * scale;
      if (sc[m] > mx) mx = sc[m];
      ++m;
    }
    if (m == 0) { rc = 6; break; }
    double den = 0.0;
    for (size_t t = 0; t < m; ++t) {
      sc[t] = exp(sc[t] - mx);
      den += sc[t];
    }
    for (size_t t = 0; t < m; ++t) {
      const double w = sc[t] / den;
      const double* vr = V + col[t] * d;
      double* o = out + i * d;
      for (size_t c = 0; c < d; ++c) o[c] += w * vr[c];
    }
  }
  free(sc);
  free(col);
  return rc;
}

/* attention.hpp:161-203: dense scores + additive 0/-inf mask. */
int orc_naive_attention(size_t n, size_t p, size_t d, const double* Q,
                        const double* K, const double* V, const uint8_t* full,
                        double* out) {
  const size_t total = p + n;
  if (!check_finite(Q, n * d)) return 2;
  if (!check_finite(K, total * d)) return 3;
  if (!check_finite(V, total * d)) return 4;
  const double scale = 1.0 / sqrt((double)d);
  double* s = (double*)malloc(sizeof(double) * (total ? total : 1));
  memset(out, 0, sizeof(double) * n * d);
  int rc = 0;
  for (size_t i = 0; i < n; ++i) {
    double mx = -INFINITY;
    for (size_t j = 0; j < total; ++j) {
      const double add = full[i * total + j] ? 0.0 : -INFINITY;
      s[j] = row_dot(Q + i * d, K + j * d, d) * scale + add;
      if (s[j] > mx) mx = s[j];
    }
    if (mx == -INFINITY) { rc = 6; break; }
    double den = 0.0;
    for (size_t j = 0; j < total; ++j) {
      s[j] = (s[j] == -INFINITY) ? 0.0 : exp(s[j] - mx);
      den += s[j];
    }
    for (size_t j = 0; j < total; ++j) {
      const double w = s[j] / den;
      if (w == 0.0) continue;
      for (size_t c = 0; c < d; ++c) out[i * d + c] += w * V[j * d + c];
    }
  }
  free(s);
  return rc;
}

/* specdec.hpp:57-85 */
int orc_simulate_tokens(const double* probs, size_t n_probs, int k,
                        int64_t trials, uint64_t seed, double* mean,
                        double* stdev) {
  if (trials < 1) return 1;
  if (k < 0 || (size_t)k > n_probs) return 2;
  double sum = 0.0, sumsq = 0.0;
  for (int64_t t = 0; t < trials; ++t) {
    uint64_t st = orc_splitmix64(seed ^ (uint64_t)t);
    int acc = 0;
    while (acc < k && orc_trial_uniform(&st) < probs[acc]) ++acc;
    const double c = (double)acc + 1.0;
    sum += c;
    sumsq += c * c;
  }
  *mean = sum / (double)trials;
  double var = sumsq / (double)trials - (*mean) * (*mean);
  *stdev = sqrt(var > 0.0 ? var : 0.0);
  return 0;
}

/* moeplan.cpp:287-311 */
void orc_random_cases(uint64_t seed, uint64_t count, int64_t* dims, double* q,
                      double* k, double* v, uint8_t* mask, size_t* q_len,
                      size_t* kv_len, size_t* mask_len) {
  uint64_t st = orc_splitmix64(seed);
  size_t qo = 0, ko = 0, mo = 0;
  for (uint64_t i = 0; i < count; ++i) {
    const size_t n = 1 + (size_t)(orc_trial_uniform(&st) * 8);
    const size_t p = (size_t)(orc_trial_uniform(&st) * 65);
    const size_t d = 1 + (size_t)(orc_trial_uniform(&st) * 32);
    if (dims) { dims[3 * i] = (int64_t)n; dims[3 * i + 1] = (int64_t)p; dims[3 * i + 2] = (int64_t)d; }
    const size_t total = p + n;
    /* Q, then K, then V, each drawn row-major as 2u-1. */
    for (size_t e = 0; e < n * d; ++e) { double x = 2.0 * orc_trial_uniform(&st) - 1.0; if (q) q[qo + e] = x; }
    for (size_t e = 0; e < total * d; ++e) { double x = 2.0 * orc_trial_uniform(&st) - 1.0; if (k) k[ko + e] = x; }
    for (size_t e = 0; e < total * d; ++e) { double x = 2.0 * orc_trial_uniform(&st) - 1.0; if (v) v[ko + e] = x; }
    for (size_t r = 0; r < n; ++r)
      for (size_t c = 0; c < n; ++c) {
        uint8_t vis = (r == c);
        if (c != r && orc_trial_uniform(&st) < 0.6) vis = 1;
        if (mask) mask[mo + r * n + c] = vis;
      }
    qo += n * d;
    ko += total * d;
    mo += n * n;
  }
  if (q_len) *q_len = qo;
  if (kv_len) *kv_len = ko;
  if (mask_len) *mask_len = mo;
}

/* ------------------------------------------------------------------------- */
uint16_t orc_f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

float orc_bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

void orc_fill_uniform_bf16(uint16_t* out, size_t count, uint64_t seed,
                           uint64_t tensor_id, uint64_t base, float scale) {
  const float s = ldexpf(scale, -24);
  const uint64_t key = seed ^ (tensor_id * PHI);
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)count; ++i) {
    const uint64_t x = orc_splitmix64(orc_splitmix64(key ^ (base + (uint64_t)i)));
    const int32_t c = (int32_t)((x >> 40) << 1) - (1 << 24);
    out[i] = orc_f32_to_bf16((float)c * s);
  }
}

/* trained-weight-like init (c_api.h smo_fill_normal_bf16 / ops.cu
 * fill_normal_kernel): Irwin-Hall of 4 chained draws, 1/1024 outliers x8 */
void orc_fill_normal_bf16(uint16_t* out, size_t count, uint64_t seed,
                          uint64_t tensor_id, uint64_t base, float scale) {
  const float s = ldexpf(scale, -24);
  const uint64_t key = seed ^ (tensor_id * PHI);
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)count; ++i) {
    uint64_t x = orc_splitmix64(orc_splitmix64(key ^ (base + (uint64_t)i)));
    int32_t c = (int32_t)(x >> 40);
    for (int k = 1; k < 4; ++k) {
      x = orc_splitmix64(x);
      c += (int32_t)(x >> 40);
    }
    c -= 1 << 25;
    if ((x & 1023u) == 0) c *= 8;
    out[i] = orc_f32_to_bf16((float)c * s);
  }
}

/* ------------------------------------------------------------------------- */
void orc_rmsnorm(const float* x, const uint16_t* gain, int T, int h, float eps,
                 uint16_t* y) {
  for (int t = 0; t < T; ++t) {
    const float* r = x + (size_t)t * h;
    double ss = 0.0;
    for (int c = 0; c < h; ++c) ss += (double)r[c] * r[c];
    const double inv = 1.0 / sqrt(ss / h + (double)eps);
    for (int c = 0; c < h; ++c)
      y[(size_t)t * h + c] = orc_f32_to_bf16((float)(r[c] * inv * orc_bf16_to_f32(gain[c])));
  }
}

void orc_gemm_xwt(const uint16_t* X, const uint16_t* W, int T, int N, int K,
                  float* out) {
  float* xf = (float*)malloc(sizeof(float) * (size_t)T * K);
  for (size_t i = 0; i < (size_t)T * K; ++i) xf[i] = orc_bf16_to_f32(X[i]);
#pragma omp parallel
  {
    float* wf = (float*)malloc(sizeof(float) * (size_t)K);
#pragma omp for schedule(static)
    for (int n = 0; n < N; ++n) {
      const uint16_t* wr = W + (size_t)n * K;
      for (int c = 0; c < K; ++c) wf[c] = orc_bf16_to_f32(wr[c]);
      for (int t = 0; t < T; ++t) {
        const float* xr = xf + (size_t)t * K;
        double acc = 0.0;
        /* products of two bf16 values are exact in fp32; sum in fp64 */
        for (int c = 0; c < K; ++c) acc += (double)(xr[c] * wf[c]);
        out[(size_t)t * N + n] = (float)acc;
      }
    }
    free(wf);
  }
  free(xf);
}

void orc_router_logits(const uint16_t* x, const uint16_t* Wr, int T, int h,
                       int E, float* logits) {
  for (int t = 0; t < T; ++t)
    for (int e = 0; e < E; ++e) {
      float part[32];
      /* lane l owns the 8-element chunks starting at 256*i + 8*l */
      for (int l = 0; l < 32; ++l) {
        float a = 0.0f;
        for (int base = 8 * l; base < h; base += 256)
          for (int j = 0; j < 8; ++j)
            a = fmaf(orc_bf16_to_f32(x[(size_t)t * h + base + j]),
                     orc_bf16_to_f32(Wr[(size_t)e * h + base + j]), a);
        part[l] = a;
      }
      for (int off = 16; off >= 1; off >>= 1)
        for (int l = 0; l < 32; ++l)
          if (l < off) part[l] = part[l] + part[l + off];
      logits[(size_t)t * E + e] = part[0];
    }
}

void orc_topk_softmax(const float* logits, int T, int E, int k, int32_t* ids,
                      float* weights) {
  for (int t = 0; t < T; ++t) {
    const float* l = logits + (size_t)t * E;
    unsigned char used[1024];
    memset(used, 0, (size_t)E);
    for (int j = 0; j < k; ++j) {
      int best = -1;
      for (int e = 0; e < E; ++e) {
        if (used[e]) continue;
        if (best < 0 || l[e] > l[best]) best = e;
      }
      used[best] = 1;
      ids[(size_t)t * k + j] = best;
    }
    const float mx = l[ids[(size_t)t * k]];
    double den = 0.0;
    double ex[64];
    for (int j = 0; j < k; ++j) {
      ex[j] = exp((double)l[ids[(size_t)t * k + j]] - mx);
      den += ex[j];
    }
    for (int j = 0; j < k; ++j) weights[(size_t)t * k + j] = (float)(ex[j] / den);
  }
}

void orc_permute(const int32_t* ids, int T, int k, int E, int32_t* offsets,
                 int32_t* perm, int32_t* pos) {
  const int P = T * k;
  for (int e = 0; e <= E; ++e) offsets[e] = 0;
  for (int i = 0; i < P; ++i) offsets[ids[i] + 1]++;
  for (int e = 0; e < E; ++e) offsets[e + 1] += offsets[e];
  int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * (size_t)(E ? E : 1));
  for (int e = 0; e < E; ++e) fill[e] = offsets[e];
  for (int i = 0; i < P; ++i) {
    const int at = fill[ids[i]]++;
    perm[at] = i;
    pos[i] = at;
  }
  free(fill);
}

void orc_expert_swiglu(const uint16_t* X, int M, int h, int h_i,
                       const uint16_t* W1, const uint16_t* W3,
                       const uint16_t* W2, float* Y) {
  if (M == 0) return;
  float* g = (float*)malloc(sizeof(float) * (size_t)M * h_i);
  float* u = (float*)malloc(sizeof(float) * (size_t)M * h_i);
  uint16_t* H = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)M * h_i);
  orc_gemm_xwt(X, W1, M, h_i, h, g);
  orc_gemm_xwt(X, W3, M, h_i, h, u);
  for (size_t i = 0; i < (size_t)M * h_i; ++i) {
    const double gv = g[i];
    const double silu = gv / (1.0 + exp(-gv));
    H[i] = orc_f32_to_bf16((float)(silu * (double)u[i]));
  }
  orc_gemm_xwt(H, W2, M, h, h_i, Y);
  free(g);
  free(u);
  free(H);
}

void orc_rope(uint16_t* x, int rows, int heads, int d, const int32_t* pos,
              float theta) {
  const int half = d / 2;
  for (int r = 0; r < rows; ++r)
    for (int hh = 0; hh < heads; ++hh) {
      uint16_t* v = x + ((size_t)r * heads + hh) * d;
      for (int i = 0; i < half; ++i) {
        const double inv = pow((double)theta, -2.0 * i / (double)d);
        const double ang = (double)pos[r] * inv;
        const double c = cos(ang), s = sin(ang);
        const double a = orc_bf16_to_f32(v[i]), b = orc_bf16_to_f32(v[i + half]);
        v[i] = orc_f32_to_bf16((float)(a * c - b * s));
        v[i + half] = orc_f32_to_bf16((float)(b * c + a * s));
      }
    }
}

int orc_verify_attention(const uint16_t* q, const uint16_t* kc,
                         const uint16_t* vc, const uint64_t* mask,
                         const int32_t* prefix, int b, int n, int n_q,
                         int n_kv, int d, int s_max, uint16_t* out) {
  const int g = n_q / n_kv;
  int rc_all = 0;
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int r = 0; r < b; ++r)
    for (int hq = 0; hq < n_q; ++hq) {
      const int hk = hq / g;
      const int p = prefix[r];
      const size_t total = (size_t)p + n;
      double* Q = (double*)malloc(sizeof(double) * (size_t)n * d);
      double* K = (double*)malloc(sizeof(double) * total * d);
      double* V = (double*)malloc(sizeof(double) * total * d);
      double* O = (double*)malloc(sizeof(double) * (size_t)n * d);
      uint8_t* m = (uint8_t*)malloc((size_t)n * n);
      for (int i = 0; i < n; ++i)
        for (int c = 0; c < d; ++c)
          Q[(size_t)i * d + c] = orc_bf16_to_f32(q[(((size_t)r * n + i) * n_q + hq) * d + c]);
      const size_t base = ((size_t)r * n_kv + hk) * (size_t)s_max * d;
      for (size_t j = 0; j < total * d; ++j) {
        K[j] = orc_bf16_to_f32(kc[base + j]);
        V[j] = orc_bf16_to_f32(vc[base + j]);
      }
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) m[i * n + j] = (uint8_t)((mask[(size_t)r * n + i] >> j) & 1u);
      const int rc = orc_chunked_attention((size_t)n, (size_t)p, (size_t)d, Q, K, V, (size_t)n, m, O);
      if (rc) {
#pragma omp critical
        rc_all = rc;
      } else {
        for (int i = 0; i < n; ++i)
          for (int c = 0; c < d; ++c)
            out[(((size_t)r * n + i) * n_q + hq) * d + c] = orc_f32_to_bf16((float)O[(size_t)i * d + c]);
      }
      free(Q); free(K); free(V); free(O); free(m);
    }
  return rc_all;
}

void orc_argmax_rows(const float* logits, int rows, int V, int32_t* idx,
                     float* top1, float* top2) {
  for (int r = 0; r < rows; ++r) {
    const float* l = logits + (size_t)r * V;
    int bi = 0;
    float b1 = l[0], b2 = -INFINITY;
    for (int v = 1; v < V; ++v) {
      if (l[v] > b1) { b2 = b1; b1 = l[v]; bi = v; }
      else if (l[v] > b2) b2 = l[v];
    }
    idx[r] = bi;
    if (top1) top1[r] = b1;
    if (top2) top2[r] = b2;
  }
}

void orc_greedy_accept(const int32_t* tokens, const int32_t* target,
                       const int32_t* parent, int b, int n, int32_t* acc_len,
                       int32_t* bonus, int32_t* keep) {
  int32_t best[64], depth[64];
  for (int r = 0; r < b; ++r) {
    const int32_t* tok = tokens + (size_t)r * n;
    const int32_t* tgt = target + (size_t)r * n;
    /* Longest accepted path below each node, children visited in id order so
     * ties resolve to the lower node id. Chain: parent(i) = i-1.            */
    for (int i = n - 1; i >= 0; --i) {
      best[i] = -1;
      depth[i] = 0;
      for (int c = i + 1; c < n; ++c) {
        const int pc = parent ? parent[(size_t)r * n + c] : c - 1;
        if (pc != i || tok[c] != tgt[i]) continue;
        if (1 + depth[c] > depth[i]) { depth[i] = 1 + depth[c]; best[i] = c; }
      }
    }
    int cur = 0, a = 0;
    keep[(size_t)r * n] = 0;
    while (best[cur] >= 0) {
      cur = best[cur];
      ++a;
      keep[(size_t)r * n + a] = cur;
    }
    for (int i = a + 1; i < n; ++i) keep[(size_t)r * n + i] = -1;
    acc_len[r] = a;
    bonus[r] = tgt[cur];
  }
}
