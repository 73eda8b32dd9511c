// c_api.cu — extern "C" entry points (include/specmoe/c_api.h): argument
// plumbing, error capture into a thread-local message, launch counting and the
// TMA tensor-map helper. No compute happens here.
#include <atomic>
#include <functional>
#include <cstring>
#include <mutex>
#include <string>

#include <thread>

#include "common.cuh"
#include "cpu_attn.h"

namespace smo {

// kernels (attention.cu, gemm_tc.cu, ops.cu)
size_t attention_workspace(const smo_attn_args& a);
void attention_launch(const smo_attn_args& a, cudaStream_t s);
void chunked_attention_f64(size_t n, size_t p, size_t d, const double* Q, const double* K, const double* V,
                           size_t mask_n, const uint8_t* mask, double* out);
void gemm_launch(const smo_gemm_args& a, cudaStream_t s);
size_t gemm_workspace(const smo_gemm_args& a);
void fill_uniform(void* dst, uint64_t count, uint64_t seed, uint64_t tensor_id, uint64_t base, float scale,
                  cudaStream_t st);
void fill_normal(void* dst, uint64_t count, uint64_t seed, uint64_t tensor_id, uint64_t base, float scale,
                 cudaStream_t st);
void fill_kv_prefix(void* cache, const int32_t* prefix, int b, int n_kv, int d, int s_max, uint64_t seed,
                    uint64_t tensor_id, cudaStream_t st, const int32_t* bt = nullptr, int max_pages = 0);
void router_topk(const void* x, const void* w, int T, int h, int E, int k, float* logits, int32_t* ids,
                 float* weights, cudaStream_t st);
void permute(const int32_t* ids, int T, int k, int E, const void* x, int h, int32_t* offsets, int32_t* perm,
             int32_t* pos, void* xp, cudaStream_t st);
void unpermute_combine(const float* y, const int32_t* pos, const float* w, int T, int k, int h, float* res,
                       cudaStream_t st, int splits = 1, size_t split_stride = 0);
int moe_launch(const void* x_perm, int rows, int h, int hi, int E, const int32_t* offsets, const void* pool,
               uint64_t w_block_stride, int pool_blocks, const int32_t* w_index, void* hbuf, float* y, int splits,
               int max_splits, int* done, cudaStream_t st);
size_t expert_code_bytes(size_t count, int bits);
size_t expert_coded_size(const void* code, size_t count, int bits);
void expert_encode(const void* src, size_t count, int bits, void* dst, int* overflow, cudaStream_t st);
void expert_decode(const void* src, size_t count, int bits, void* dst, cudaStream_t st);
size_t tcode_max_bytes(int h, int hi);
size_t tcode_encode(const void* src, int h, int hi, void* dst, cudaStream_t st, int fmt = 2);
void tcode_decode(const void* const* srcs, void* const* dsts, int n, int h, int hi, cudaStream_t st, int fmt = 2);
int moe_coded_launch(const void* x_perm, int rows, int h, int hi, int E, const int32_t* offsets,
                     const void* const* w_code, void* hbuf, float* y, int splits, int max_splits, int* done,
                     cudaStream_t st, int fmt = 2);
void rmsnorm(const float* x, const void* gain, int T, int h, float eps, void* y, cudaStream_t st);
void embed(const int32_t* tok, const void* emb, int T, int h, float* x, cudaStream_t st);
void rope_append(const void* qkv, const int32_t* prefix, const int32_t* parent, int b, int n, int n_q, int n_kv,
                 int d, int s_max, float theta, void* q_out, void* kc, void* vc, cudaStream_t st,
                 const int32_t* bt = nullptr, int max_pages = 0);
void argmax_reduce(const float* val, const int32_t* idx, int rows, int parts, int32_t* target, cudaStream_t st);
void argmax_rows(const float* logits, int rows, int V, int32_t* target, cudaStream_t st);
void greedy_accept(const int32_t* tokens, const int32_t* target, const int32_t* parent, int b, int n,
                   int32_t* acc_len, int32_t* bonus, int32_t* keep, cudaStream_t st);
void kv_rollback(void* const* kcs, void* const* vcs, int n_layers, const int32_t* prefix, const int32_t* acc,
                 const int32_t* keep, int b, int n, int n_kv, int d, int s_max, int32_t* kv_len, cudaStream_t st,
                 const int32_t* bt = nullptr, int max_pages = 0);

static std::atomic<uint64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(uint64_t(n), std::memory_order_relaxed); }

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  if (!fn) throw Error(SMO_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  return fn;
}

void make_tmap_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                    const uint64_t* strides_bytes, const uint32_t* box, bool swizzle128) {
  cuuint64_t d[5];
  cuuint64_t s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
  }
  for (int i = 0; i < rank - 1; ++i) s[i] = strides_bytes[i];
  const CUresult r = get_encode()(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, cuuint32_t(rank), const_cast<void*>(base),
                                  d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(SMO_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
}

}  // namespace smo

namespace {
thread_local std::string g_last_error;

template <class F>
smo_status guard(F&& f) {
  try {
    f();
    return SMO_OK;
  } catch (const smo::Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    return SMO_CAPACITY;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SMO_INVALID_ARG;
  }
}
inline cudaStream_t S(smo_stream s) { return reinterpret_cast<cudaStream_t>(s); }
}  // namespace

extern "C" {

const char* smo_last_error(void) { return g_last_error.c_str(); }
const char* smo_version(void) { return "specmoe-b200 0.1 (sm_100a)"; }
uint64_t smo_launch_count(void) { return smo::g_launches.load(); }

int smo_device_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return v;
}

smo_status smo_fill_normal_bf16(void* dst, uint64_t count, uint64_t seed, uint64_t tensor_id, uint64_t base,
                                float scale, smo_stream stream) {
  return guard([&] { smo::fill_normal(dst, count, seed, tensor_id, base, scale, S(stream)); });
}

smo_status smo_fill_uniform_bf16(void* dst, uint64_t count, uint64_t seed, uint64_t tensor_id, uint64_t base,
                                 float scale, smo_stream stream) {
  return guard([&] { smo::fill_uniform(dst, count, seed, tensor_id, base, scale, S(stream)); });
}

size_t smo_verify_attention_workspace(const smo_attn_args* a) {
  size_t r = 0;
  if (guard([&] {
        SMO_REQUIRE(a, "attention: null args");
        r = smo::attention_workspace(*a);
      }) != SMO_OK)
    return size_t(-1);
  return r;
}

smo_status smo_verify_attention(const smo_attn_args* a, smo_stream stream) {
  return guard([&] {
    SMO_REQUIRE(a, "attention: null args");
    smo::attention_launch(*a, S(stream));
  });
}

smo_status smo_cpu_verify_attention(const smo_attn_args* a, int32_t threads) {
  return guard([&] {
    SMO_REQUIRE(a && a->q && a->k_cache && a->v_cache && a->mask && a->prefix_len && a->out,
                "attention: null pointer");
    SMO_REQUIRE(!a->block_table, "attention: the host kernel takes contiguous K/V");
    SMO_REQUIRE(a->b > 0 && a->n > 0 && a->n <= 64 && a->n_kv > 0 && a->n_q % a->n_kv == 0 && a->d % 8 == 0,
                "attention: shape mismatch");
    for (int r = 0; r < a->b; ++r)
      SMO_REQUIRE(a->prefix_len[r] >= 0 && a->prefix_len[r] + a->n <= a->s_max, "attention: shape mismatch");
    smo::CpuPool pool(threads > 0 ? threads : int(std::max(1u, std::thread::hardware_concurrency())));
    smo::CpuAttnJob j{reinterpret_cast<const uint16_t*>(a->q), reinterpret_cast<const uint16_t*>(a->k_cache),
                      reinterpret_cast<const uint16_t*>(a->v_cache), a->mask, a->prefix_len,
                      reinterpret_cast<uint16_t*>(a->out), a->b, a->n, a->n_q, a->n_kv, a->d, a->s_max, 1};
    smo::cpu_verify_attention(j, pool);
  });
}

smo_status smo_chunked_attention_f64(size_t n, size_t p, size_t d, const double* Q, const double* K,
                                     const double* V, size_t mask_n, const uint8_t* mask, double* out) {
  return guard([&] { smo::chunked_attention_f64(n, p, d, Q, K, V, mask_n, mask, out); });
}

smo_status smo_router_topk(const void* x, const void* w, int32_t T, int32_t h, int32_t E, int32_t k,
                           float* logits_out, int32_t* ids, float* weights, smo_stream stream) {
  return guard([&] { smo::router_topk(x, w, T, h, E, k, logits_out, ids, weights, S(stream)); });
}

smo_status smo_permute(const int32_t* ids, int32_t T, int32_t k, int32_t E, const void* x, int32_t h,
                       int32_t* offsets, int32_t* perm, int32_t* pos, void* x_perm, smo_stream stream) {
  return guard([&] { smo::permute(ids, T, k, E, x, h, offsets, perm, pos, x_perm, S(stream)); });
}

smo_status smo_unpermute_combine(const float* y, const int32_t* pos, const float* w, int32_t T, int32_t k,
                                 int32_t h, float* residual, smo_stream stream) {
  return guard([&] { smo::unpermute_combine(y, pos, w, T, k, h, residual, S(stream)); });
}

smo_status smo_expert_encode(const void* src, uint64_t count, int32_t bits, void* dst, int32_t* overflow,
                             smo_stream stream) {
  return guard([&] { smo::expert_encode(src, size_t(count), bits, dst, overflow, S(stream)); });
}
smo_status smo_expert_decode(const void* src, uint64_t count, int32_t bits, void* dst, smo_stream stream) {
  return guard([&] { smo::expert_decode(src, size_t(count), bits, dst, S(stream)); });
}
size_t smo_expert_code_bytes(uint64_t count, int32_t bits) {
  return (bits == 1 || bits == 3 || bits == 4) ? smo::expert_code_bytes(size_t(count), bits) : 0;
}
uint64_t smo_expert_coded_size(const void* code, uint64_t count, int32_t bits) {
  if (!(bits == 1 || bits == 3 || bits == 4) || (bits == 1 && !code)) return 0;
  uint64_t r = 0;
  if (guard([&] { r = smo::expert_coded_size(code, size_t(count), bits); }) != SMO_OK) return 0;
  return r;
}

size_t smo_tcode_max_bytes(int32_t h, int32_t h_i) {
  return (h > 0 && h_i > 0 && h % 128 == 0 && h_i % 128 == 0) ? smo::tcode_max_bytes(h, h_i) : 0;
}
smo_status smo_tcode_encode(const void* src, int32_t h, int32_t h_i, void* dst, uint64_t* bytes, smo_stream stream) {
  return guard([&] {
    const size_t n = smo::tcode_encode(src, h, h_i, dst, S(stream));
    if (bytes) *bytes = n;
  });
}
smo_status smo_tcode_decode(const void* src, int32_t h, int32_t h_i, void* dst, smo_stream stream) {
  return guard([&] { smo::tcode_decode(&src, &dst, 1, h, h_i, S(stream)); });
}
smo_status smo_tcode3_encode(const void* src, int32_t h, int32_t h_i, void* dst, uint64_t* bytes, smo_stream stream) {
  return guard([&] {
    const size_t n = smo::tcode_encode(src, h, h_i, dst, S(stream), 3);
    if (bytes) *bytes = n;
  });
}
smo_status smo_tcode3_decode(const void* src, int32_t h, int32_t h_i, void* dst, smo_stream stream) {
  return guard([&] { smo::tcode_decode(&src, &dst, 1, h, h_i, S(stream), 3); });
}

smo_status smo_unpermute_combine_split(const float* y, int32_t splits, uint64_t split_stride, const int32_t* pos,
                                       const float* w, int32_t T, int32_t k, int32_t h, float* residual,
                                       smo_stream stream) {
  return guard([&] {
    SMO_REQUIRE(splits >= 1, "combine: splits >= 1");
    smo::unpermute_combine(y, pos, w, T, k, h, residual, S(stream), splits, size_t(split_stride));
  });
}

smo_status smo_moe_experts(const void* x_perm, int32_t rows, int32_t h, int32_t h_i, int32_t E,
                           const int32_t* offsets, const void* w_pool, uint64_t w_block_stride,
                           int32_t w_pool_blocks, const int32_t* w_index, void* h_out, float* y, int32_t splits,
                           int32_t* splits_used, int32_t* scratch, smo_stream stream) {
  return guard([&] {
    const int sp = smo::moe_launch(x_perm, rows, h, h_i, E, offsets, w_pool, w_block_stride, w_pool_blocks, w_index,
                                   h_out, y, splits, 4, scratch, S(stream));
    if (splits_used) *splits_used = sp;
  });
}

smo_status smo_moe_experts_coded(const void* x_perm, int32_t rows, int32_t h, int32_t h_i, int32_t E,
                                 const int32_t* offsets, const void* const* w_code, void* h_out, float* y,
                                 int32_t splits, int32_t* splits_used, int32_t* scratch, smo_stream stream) {
  return guard([&] {
    const int sp = smo::moe_coded_launch(x_perm, rows, h, h_i, E, offsets, w_code, h_out, y, splits, 4, scratch,
                                         S(stream));
    if (splits_used) *splits_used = sp;
  });
}
smo_status smo_moe_experts_coded3(const void* x_perm, int32_t rows, int32_t h, int32_t h_i, int32_t E,
                                  const int32_t* offsets, const void* const* w_code, void* h_out, float* y,
                                  int32_t splits, int32_t* splits_used, int32_t* scratch, smo_stream stream) {
  return guard([&] {
    const int sp = smo::moe_coded_launch(x_perm, rows, h, h_i, E, offsets, w_code, h_out, y, splits, 4, scratch,
                                         S(stream), 3);
    if (splits_used) *splits_used = sp;
  });
}

size_t smo_gemm_workspace(const smo_gemm_args* a) {
  size_t r = 0;
  if (guard([&] {
        SMO_REQUIRE(a, "gemm: null args");
        r = smo::gemm_workspace(*a);
      }) != SMO_OK)
    return size_t(-1);
  return r;
}

smo_status smo_gemm(const smo_gemm_args* a, smo_stream stream) {
  return guard([&] {
    SMO_REQUIRE(a, "gemm: null args");
    smo::gemm_launch(*a, S(stream));
  });
}

smo_status smo_rmsnorm(const float* x, const void* gain, int32_t T, int32_t h, float eps, void* y,
                       smo_stream stream) {
  return guard([&] { smo::rmsnorm(x, gain, T, h, eps, y, S(stream)); });
}

smo_status smo_embed(const int32_t* tokens, const void* emb, int32_t T, int32_t h, float* x, smo_stream stream) {
  return guard([&] { smo::embed(tokens, emb, T, h, x, S(stream)); });
}

smo_status smo_rope_append(const void* qkv, const int32_t* prefix_len, const int32_t* parent, int32_t b,
                           int32_t n, int32_t n_q, int32_t n_kv, int32_t d, int32_t s_max, float theta,
                           void* q_out, void* k_cache, void* v_cache, smo_stream stream) {
  return guard([&] {
    smo::rope_append(qkv, prefix_len, parent, b, n, n_q, n_kv, d, s_max, theta, q_out, k_cache, v_cache,
                     S(stream));
  });
}

smo_status smo_fill_kv_prefix(void* cache, const int32_t* prefix_len, int32_t b, int32_t n_kv, int32_t d,
                              int32_t s_max, uint64_t seed, uint64_t tensor_id, smo_stream stream) {
  return guard([&] { smo::fill_kv_prefix(cache, prefix_len, b, n_kv, d, s_max, seed, tensor_id, S(stream)); });
}

smo_status smo_argmax_reduce(const float* v, const int32_t* i, int32_t rows, int32_t parts, int32_t* target,
                             smo_stream stream) {
  return guard([&] { smo::argmax_reduce(v, i, rows, parts, target, S(stream)); });
}

smo_status smo_argmax_rows(const float* logits, int32_t rows, int32_t V, int32_t* target, smo_stream stream) {
  return guard([&] { smo::argmax_rows(logits, rows, V, target, S(stream)); });
}

smo_status smo_greedy_accept(const int32_t* tokens, const int32_t* target, const int32_t* parent, int32_t b,
                             int32_t n, int32_t* acc_len, int32_t* bonus, int32_t* keep, smo_stream stream) {
  return guard([&] { smo::greedy_accept(tokens, target, parent, b, n, acc_len, bonus, keep, S(stream)); });
}

smo_status smo_kv_rollback(void* const* k_caches, void* const* v_caches, int32_t n_layers,
                           const int32_t* prefix_len, const int32_t* acc_len, const int32_t* keep, int32_t b,
                           int32_t n, int32_t n_kv, int32_t d, int32_t s_max, int32_t* kv_len, smo_stream stream) {
  return guard([&] {
    smo::kv_rollback(k_caches, v_caches, n_layers, prefix_len, acc_len, keep, b, n, n_kv, d, s_max, kv_len,
                     S(stream));
  });
}

}  // extern "C"

// engine entry points live in engine.cu; they share the guard via this hook.
namespace smo {
smo_status run_guarded(const std::function<void()>& f) { return guard(f); }
}  // namespace smo
