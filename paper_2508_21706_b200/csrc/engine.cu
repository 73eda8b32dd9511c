// engine.cu — VerifyEngine: the measured realisation of the reference's
// target-verification DAG (pipeline.hpp:147-206) on one B200.
//
// Per layer l (compute stream):  RMSNorm -> QKV GEMM -> RoPE+KV append ->
//   K1 attention -> O GEMM (+residual) -> RMSNorm -> K2 router -> K3 permute
//   -> [wait slot_ready(l)] -> K4 SwiGLU gate/up -> K4 down -> K3 combine
//   -> record slot_free(l mod S).
// Copy stream (K5 expert streamer): H2D_EXPERTS(l) into HBM slot l mod S,
//   waiting slot_free of the layer that last used the slot — the reference's
//   serial-link model (pipeline.hpp:177-181) plus the real slot-release edge
//   H2D(l+S) <- GPU_MOE(l).
// After the last layer: final RMSNorm -> LM head GEMM with fused argmax
// partials -> K6 argmax reduce -> greedy accept (specdec.hpp:65-76).
//
// Experts live in pinned host DRAM as [W1 | W3 | W2] blocks (nn.Linear
// layouts: W1,W3 [h_i, h], W2 [h, h_i]); the HBM pool holds S staging slots of
// E blocks each plus the hot-expert cache (MemoryPolicy.expert_cache_bytes,
// config.hpp:103-108), filled once at creation.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <thread>
#include <string>
#include <vector>

#include "common.cuh"
#include "cpu_attn.h"

namespace smo {

smo_status run_guarded(const std::function<void()>& f);
size_t attention_workspace(const smo_attn_args& a);
void attention_launch(const smo_attn_args& a, cudaStream_t s);
void gemm_launch(const smo_gemm_args& a, cudaStream_t s);
size_t gemm_workspace(const smo_gemm_args& a);
void fill_uniform(void* dst, uint64_t count, uint64_t seed, uint64_t tensor_id, uint64_t base, float scale,
                  cudaStream_t st);
void fill_kv_prefix(void* cache, const int32_t* prefix, int b, int n_kv, int d, int s_max, uint64_t seed,
                    uint64_t tensor_id, cudaStream_t st, const int32_t* bt = nullptr, int max_pages = 0);
void router_topk(const void* x, const void* w, int T, int h, int E, int k, float* logits, int32_t* ids,
                 float* weights, cudaStream_t st);
void permute(const int32_t* ids, int T, int k, int E, const void* x, int h, int32_t* offsets, int32_t* perm,
             int32_t* pos, void* xp, cudaStream_t st);
void unpermute_combine(const float* y, const int32_t* pos, const float* w, int T, int k, int h, float* res,
                       cudaStream_t st, int splits = 1, size_t split_stride = 0);
void rmsnorm(const float* x, const void* gain, int T, int h, float eps, void* y, cudaStream_t st);
void embed(const int32_t* tok, const void* emb, int T, int h, float* x, cudaStream_t st);
void rope_append(const void* qkv, const int32_t* prefix, const int32_t* parent, int b, int n, int n_q, int n_kv,
                 int d, int s_max, float theta, void* q_out, void* kc, void* vc, cudaStream_t st,
                 const int32_t* bt = nullptr, int max_pages = 0);
void argmax_reduce(const float* val, const int32_t* idx, int rows, int parts, int32_t* target, cudaStream_t st);
void greedy_accept(const int32_t* tokens, const int32_t* target, const int32_t* parent, int b, int n,
                   int32_t* acc_len, int32_t* bonus, int32_t* keep, cudaStream_t st);
void build_mask(const int32_t* parent, int b, int n, uint64_t* mask, cudaStream_t st);
void decode_prep(const int32_t* root, const int32_t* drafts, int b, int n, int32_t* tokens, cudaStream_t st);
void draft_io(const int32_t* tokens, const int32_t* kv_len, int t, int b, int n, int32_t* tok_in, int32_t* pos,
              cudaStream_t st);
void draft_scatter(const int32_t* out, int b, int n, int t, int32_t* tokens, cudaStream_t st);
void decode_commit(const int32_t* tokens, const int32_t* acc, const int32_t* bonus, int b, int n, int cap,
                   int32_t* hist, int32_t* hist_n, int32_t* kv_len, int32_t* root, cudaStream_t st,
                   const int32_t* keep = nullptr);
void kv_rollback(void* const* kcs, void* const* vcs, int n_layers, const int32_t* prefix, const int32_t* acc,
                 const int32_t* keep, int b, int n, int n_kv, int d, int s_max, int32_t* kv_len, cudaStream_t st,
                 const int32_t* bt = nullptr, int max_pages = 0);
void prefill_last(const float* x, const int32_t* len, int b, int C, int h, float* out, cudaStream_t st);
// expert parallelism (ep.cu)
EpTransport* ep_transport(void* group);
void ep_remap(const int32_t* ids, int n, int P, int E_loc, int32_t* oid, cudaStream_t st);
void ep_pack(const void* xp, const int32_t* offsets, int P, int E_loc, int C, int h, size_t block_bytes, void* send,
             cudaStream_t st);
void ep_pos(const int32_t* oid, const int32_t* pos, const int32_t* offsets, int n, int E_loc, int C, int32_t* pos_ep,
            cudaStream_t st);
void ep_unpack(const void* recv, int P, int E_loc, int C, int h, size_t block_bytes, void* xl, int32_t* offsets_l,
               int32_t* back, cudaStream_t st);
void ep_pack_back(const float* yl, const int32_t* back, const int32_t* offsets_l, int E_loc, int h, float* sendback,
                  cudaStream_t st, int splits = 1, size_t split_stride = 0);
int moe_launch(const void* x_perm, int rows, int h, int hi, int E, const int32_t* offsets, const void* pool,
               uint64_t w_block_stride, int pool_blocks, const int32_t* w_index, void* hbuf, float* y, int splits,
               int max_splits, int* done, cudaStream_t st);
int pick_moe_splits(int rows, int h, int hi, int E, int max_splits);
size_t expert_code_bytes(size_t count, int bits);
void expert_encode(const void* src, size_t count, int bits, void* dst, int* overflow, cudaStream_t st);
void expert_decode(const void* src, size_t count, int bits, void* dst, cudaStream_t st);

// Procedural tensor ids; the oracle tests use the same ids.
namespace tid {
constexpr uint64_t kEmbed = 1, kLmHead = 2;
inline uint64_t layer(int l) { return 1000ull * uint64_t(l + 1); }
constexpr uint64_t kWqkv = 1, kWo = 2, kRouter = 4, kShared = 50, kExpert = 100;
inline uint64_t kv(int l, int which) { return 900000ull + 2ull * uint64_t(l) + uint64_t(which); }
// drafter layer l: +1 Wqkv, +2 Wo, +3 W1, +4 W3, +5 W2; its prefix K/V
inline uint64_t draft(int l) { return 700000ull + 100ull * uint64_t(l); }
inline uint64_t draft_kv(int l, int which) { return 910000ull + 2ull * uint64_t(l) + uint64_t(which); }
}  // namespace tid

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct Engine {
  smo_model_config cfg{};
  smo_engine_options opt{};
  cudaStream_t copy = nullptr;
  int h = 0, hi = 0, E = 0, K = 0, L = 0, nq = 0, nkv = 0, d = 0, V = 0;
  int qkv_w = 0;
  size_t blk_elems = 0, blk_bytes = 0;
  std::vector<DevBuf> allocs;

  // weights
  uint16_t *embed_w = nullptr, *lm_w = nullptr, *final_norm = nullptr, *ones = nullptr;
  struct Layer {
    uint16_t *wqkv, *wo, *router;
    uint16_t *ws1 = nullptr, *ws3 = nullptr, *ws2 = nullptr;  // shared expert (resident)
    uint16_t *kc, *vc;
  };
  std::vector<Layer> layers;
  // drafter: dense decoder layers, resident in HBM
  struct DLayer {
    uint16_t *wqkv, *wo, *w1, *w3, *w2, *kc, *vc;
  };
  std::vector<DLayer> dlayers;
  int dL = 0, dI = 0;
  uint16_t* dh = nullptr;  // drafter SwiGLU activations [maxT, dI]
  int32_t *d_dtok = nullptr, *d_dpos = nullptr, *d_dout = nullptr;
  uint64_t* d_mask1 = nullptr;  // single-row chain mask (bit 0) per request
  // decode state: committed K/V length, next root, history
  int dec_b = 0, hist_cap = 0;
  int64_t kv_bound = 0;  // host upper bound of kv_len (K1 split planning)
  int32_t *d_kvlen = nullptr, *d_root = nullptr, *d_hist = nullptr, *d_hist_n = nullptr, *d_dec_tok = nullptr,
          *d_drafts = nullptr, *d_dec_parent = nullptr;
  void** d_cache_ptrs = nullptr;  // [2][L + dL]: K then V caches of target + drafter layers (tree compaction)
  bool last_was_decode = false;
  // paged K/V: pool of num_pages 128-token pages per layer,
  // host-managed block table (pinned mirror + device copy), free list
  bool paged = false;
  int max_pages = 0, num_pages = 0;
  int32_t* h_bt = nullptr;  // pinned [maxB * max_pages], -1 = unmapped
  int32_t* d_bt = nullptr;
  std::vector<int> free_pages, req_pages;
  std::vector<int64_t> kv_known;  // host bound of each request's K/V length
  bool bt_dirty = false;
  // CPU attention placement: host K/V + host thread pool
  bool attn_cpu = false;
  std::unique_ptr<CpuPool> cpu_pool;
  std::vector<void*> host_allocs;         // cudaFreeHost at destruction
  uint16_t *q_host = nullptr, *attn_host = nullptr;  // pinned mapped [maxT, n_q, d]
  int32_t* prefix_host = nullptr;         // pinned [maxB]
  uint64_t* mask_host = nullptr;          // pinned [maxT]
  struct HostAttn {
    CpuPool* pool;
    CpuAttnJob job;
  };
  std::vector<HostAttn> host_jobs;        // one per target layer (enqueued ahead of execution)
  // BATCH_ONE expert streaming: stream only router-selected experts
  bool batch_one = false;
  int32_t* h_offsets = nullptr;           // pinned [E+1] routed offsets of the current layer
  cudaEvent_t route_ev = nullptr;
  std::vector<double> layer_bytes;        // bytes streamed per layer in the last step
  std::vector<double> layer_raw_bytes;    // their bf16 size (coded blocks expand)
  // lossless expert codec on the link (xfer.cu): coded blocks cross into
  // cstage and are expanded into the pool slot on the compute stream
  bool xcomp = false;
  size_t cblk_bytes = 0;                  // coded bytes of one [W1|W3|W2] block at 4 bits (staging stride)
  std::vector<uint8_t> blk_coded;         // [host_alias * E_loc] exponent bits of the host block (0 = raw)
  uint8_t* cstage = nullptr;              // [slots][E_loc][cblk_bytes]
  std::vector<std::vector<int>> coded_streamed;  // per layer: local experts streamed coded
  std::vector<cudaEvent_t> draft_ev;  // [maxN + 1]: boundaries of the drafter steps
  int last_draft_steps = 0;
  std::vector<uint16_t*> host_bufs;  // pinned, E blocks each
  int host_alias = 0;
  // expert pool in HBM
  uint16_t* pool = nullptr;
  int slots = 2, pool_blocks = 0;
  std::vector<int> cache_blk;  // [L*E] pool block of a cached expert, -1 otherwise
  int32_t* d_w_index = nullptr;  // [L*E]
  std::vector<cudaEvent_t> slot_ready, slot_free;
  // EP: experts owned by this rank
  std::vector<int> owned;
  // expert parallelism: transport, geometry and exchange buffers
  EpTransport* ept = nullptr;
  bool ep_on = false;
  int P = 1, E_loc = 0, C = 0;
  size_t blk_d = 0;  // dispatch block bytes (C bf16 rows + E_loc counts)
  int32_t *oid = nullptr, *pos_ep = nullptr, *offsets_l = nullptr, *back = nullptr, *d_w_index_loc = nullptr;
  uint8_t *ep_send = nullptr, *ep_recv = nullptr;
  uint16_t* xl = nullptr;
  float *yl = nullptr, *ep_sendback = nullptr, *ep_recvback = nullptr;

  // activations (max sizes)
  int maxT = 0, maxB = 0, maxN = 0, s_max = 0;
  float *x = nullptr, *ybuf = nullptr, *rw = nullptr, *amax_v = nullptr;
  int moe_splits = 1;      // down-projection K slices of the fused MoE kernel (from the global shapes)
  int* d_done = nullptr;   // fused MoE kernel: finished gate/up units per expert
  bool moe_fused = true;   // SMO_MOE_FUSED=0: two grouped GEMM launches instead (A/B runs)
  uint16_t *xn = nullptr, *qkv = nullptr, *q = nullptr, *attn = nullptr, *xp = nullptr, *hbuf = nullptr;
  uint16_t* hs = nullptr;  // shared-expert SwiGLU activations [T, shared_inter]
  int32_t *ids = nullptr, *offsets = nullptr, *perm = nullptr, *pos = nullptr, *amax_i = nullptr, *target = nullptr;
  int32_t *d_tokens = nullptr, *d_parent = nullptr, *d_prefix = nullptr, *d_acc = nullptr, *d_bonus = nullptr,
          *d_keep = nullptr;
  uint64_t* d_mask = nullptr;
  void* attn_ws = nullptr;
  size_t attn_ws_bytes = 0;
  void* gemm_ws = nullptr;  // split-K partials of the dense projections
  size_t gemm_ws_bytes = 0;
  int32_t* h_stage = nullptr;  // pinned staging for host inputs/outputs
  size_t h_stage_elems = 0;

  // timing
  std::vector<cudaEvent_t> ev;  // pool of timing events
  smo_stage_times last{};
  double last_h2d_bytes = 0;

  // debug snapshots
  bool debug = false;
  std::map<std::string, std::vector<DevBuf>> dbg;

  ~Engine() {
    for (auto e : slot_ready) cudaEventDestroy(e);
    for (auto e : slot_free) cudaEventDestroy(e);
    for (auto e : ev) cudaEventDestroy(e);
    for (auto e : draft_ev) cudaEventDestroy(e);
    if (route_ev) cudaEventDestroy(route_ev);
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    for (auto hb : host_bufs) cudaFreeHost(hb);
    if (h_stage) cudaFreeHost(h_stage);
    if (h_bt) cudaFreeHost(h_bt);
    cpu_pool.reset();
    for (void* hp : host_allocs) cudaFreeHost(hp);
    for (auto& a : allocs) cudaFree(a.p);
    for (auto& kv : dbg)
      for (auto& b : kv.second) cudaFree(b.p);
    if (copy) cudaStreamDestroy(copy);
  }

  template <class T>
  T* dalloc(size_t count) {
    void* p = nullptr;
    const size_t bytes = std::max<size_t>(16, count * sizeof(T));
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess)
      throw Error(SMO_CAPACITY, std::string("engine: cudaMalloc(") + std::to_string(bytes) + ") failed: " +
                                    cudaGetErrorString(e));
    allocs.push_back({p, bytes});
    return reinterpret_cast<T*>(p);
  }

  // pinned host memory the GPU reads/writes directly (UVA: same address)
  template <class T>
  T* halloc_mapped(size_t count) {
    void* hp = nullptr;
    const size_t bytes = std::max<size_t>(16, count * sizeof(T));
    cudaError_t e = cudaHostAlloc(&hp, bytes, cudaHostAllocPortable | cudaHostAllocMapped);
    if (e != cudaSuccess)
      throw Error(SMO_CAPACITY, "engine: pinned host allocation of " + std::to_string(bytes) + " bytes failed");
    host_allocs.push_back(hp);
    void* dp = nullptr;
    SMO_CUDA_CHECK(cudaHostGetDevicePointer(&dp, hp, 0));
    SMO_REQUIRE(dp == hp, "engine: mapped host memory needs unified addressing");
    std::memset(hp, 0, bytes);
    return reinterpret_cast<T*>(hp);
  }
  static void CUDART_CB host_attn_cb(void* arg) {
    auto* j = static_cast<HostAttn*>(arg);
    cpu_verify_attention(j->job, *j->pool);
  }

  size_t kv_elems() const {
    return paged ? size_t(num_pages) * nkv * kKvPage * d : size_t(maxB) * nkv * s_max * d;
  }
  const int32_t* bt() const { return paged ? d_bt : nullptr; }
  // every page back to the free list (lowest ids handed out first)
  void bt_reset() {
    if (!paged) return;
    for (size_t i = 0; i < size_t(maxB) * max_pages; ++i) h_bt[i] = -1;
    free_pages.clear();
    for (int pg = num_pages - 1; pg >= 0; --pg) free_pages.push_back(pg);
    req_pages.assign(size_t(maxB), 0);
    bt_dirty = true;
  }
  // map pages for positions [0, len) of request r
  void bt_ensure(int r, int64_t len) {
    if (!paged) return;
    const int need = int(std::min<int64_t>(max_pages, (len + kKvPage - 1) / kKvPage));
    while (req_pages[size_t(r)] < need) {
      if (free_pages.empty())
        throw Error(SMO_CAPACITY, "engine: K/V page pool exhausted (" + std::to_string(num_pages) + " pages)");
      h_bt[size_t(r) * max_pages + req_pages[size_t(r)]] = free_pages.back();
      free_pages.pop_back();
      ++req_pages[size_t(r)];
      bt_dirty = true;
    }
  }
  void bt_sync(cudaStream_t st) {
    if (!paged || !bt_dirty) return;
    SMO_CUDA_CHECK(cudaMemcpyAsync(d_bt, h_bt, size_t(maxB) * max_pages * 4, cudaMemcpyHostToDevice, st));
    bt_dirty = false;
  }

  // exponent bits of layer l's local expert le on the host (0: raw bf16)
  int code_bits(int l, int le) const { return xcomp ? blk_coded[size_t(host_layer(l)) * E_loc + size_t(le)] : 0; }
  // expand layer l's coded blocks (streamed into cstage) into its pool slot,
  // on the compute stream after slot_ready(l)
  void decode_slot(int l, cudaStream_t st) {
    const int s = l % slots;
    for (int le : coded_streamed[size_t(l)])
      expert_decode(cstage + (size_t(s) * E_loc + le) * cblk_bytes, blk_elems, code_bits(l, le),
                    pool + (size_t(s) * E_loc + le) * blk_elems, st);
  }

  int host_layer(int l) const { return host_alias > 0 ? l % host_alias : l; }
  int expert_owner(int e) const { return opt.ep_size > 1 ? e % opt.ep_size : 0; }
  bool owns(int e) const { return opt.ep_size <= 1 || expert_owner(e) == opt.ep_rank; }

  void create() {
    h = cfg.hidden;
    hi = cfg.inter;
    E = cfg.n_expert;
    K = cfg.top_k;
    L = cfg.n_layers;
    nq = cfg.n_q_heads;
    nkv = cfg.n_kv_heads;
    d = cfg.head_dim;
    V = cfg.vocab;
    SMO_REQUIRE(h > 0 && hi > 0 && E > 0 && K > 0 && K <= E && L > 0, "engine: bad model shape");
    SMO_REQUIRE(nq > 0 && nkv > 0 && nq % nkv == 0 && (d == 64 || d == 128), "engine: bad attention shape");
    SMO_REQUIRE(h % 256 == 0 && hi % 128 == 0 && V % 128 == 0 && (nq * d) % 128 == 0, "engine: unsupported dims");
    SMO_REQUIRE(cfg.shared_inter >= 0 && cfg.shared_inter % 128 == 0, "engine: shared_inter must be a multiple of 128");
    SMO_REQUIRE(opt.max_batch > 0 && opt.max_verify > 0 && opt.max_verify <= 64, "engine: bad batch options");
    // expert parallelism whenever a transport is given (ep_size 1 with a
    // 1-rank group runs the full dispatch/combine path: a 1-GPU check of it)
    if (opt.ep_size > 1 || opt.nccl_comm) {
      const int ps = std::max(1, opt.ep_size);
      SMO_REQUIRE(E % ps == 0, "engine: n_expert must be divisible by ep_size");
      SMO_REQUIRE(opt.ep_rank >= 0 && opt.ep_rank < ps, "engine: bad ep_rank");
      ept = ep_transport(opt.nccl_comm);
      SMO_REQUIRE(ept && ept->P == ps, "engine: ep_size needs an smo_ep_group of that size");
      P = ps;
      ep_on = true;
    }
    E_loc = E / P;
    qkv_w = (nq + 2 * nkv) * d;
    blk_elems = size_t(3) * h * hi;
    blk_bytes = blk_elems * 2;
    maxB = opt.max_batch;
    maxN = opt.max_verify;
    maxT = maxB * maxN;
    s_max = opt.max_seq;
    SMO_REQUIRE(s_max >= maxN + 1, "engine: max_seq too small");
    slots = std::max(2, opt.hbm_slots);
    host_alias = opt.host_alias_layers > 0 ? std::min(opt.host_alias_layers, L) : L;
    debug = (opt.flags & SMO_ENGINE_DEBUG) != 0;
    SMO_CUDA_CHECK(cudaSetDevice(opt.device));
    SMO_CUDA_CHECK(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
    if (opt.kv_pages != 0) {
      paged = true;
      max_pages = (s_max + kKvPage - 1) / kKvPage;
      num_pages = opt.kv_pages > 0 ? opt.kv_pages : maxB * max_pages;
      SMO_REQUIRE(num_pages > 0, "engine: bad kv_pages");
      SMO_CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&h_bt), size_t(maxB) * max_pages * 4,
                                   cudaHostAllocPortable));
      d_bt = dalloc<int32_t>(size_t(maxB) * max_pages);
      bt_reset();
    }
    kv_known.assign(size_t(maxB), 0);
    if (opt.moe_batching) {
      SMO_REQUIRE(!(opt.ep_size > 1 || opt.nccl_comm), "engine: BATCH_ONE streaming is not available with expert parallelism");
      batch_one = true;
      SMO_CUDA_CHECK(cudaEventCreateWithFlags(&route_ev, cudaEventDisableTiming));
    }
    if (opt.attn_cpu) {
      SMO_REQUIRE(!paged, "engine: the CPU attention placement keeps contiguous host K/V (kv_pages = 0)");
      attn_cpu = true;
      cpu_pool.reset(new CpuPool(int(std::max(1u, std::thread::hardware_concurrency()))));
    }
    cudaStream_t st = nullptr;

    // dense weights
    embed_w = dalloc<uint16_t>(size_t(V) * h);
    lm_w = dalloc<uint16_t>(size_t(V) * h);
    ones = dalloc<uint16_t>(size_t(std::max(h, 1)));
    final_norm = ones;
    fill_uniform(embed_w, size_t(V) * h, cfg.seed, tid::kEmbed, 0, 1.0f, st);
    fill_uniform(lm_w, size_t(V) * h, cfg.seed, tid::kLmHead, 0, std::sqrt(3.0f / h) * cfg.lm_scale, st);
    {
      std::vector<uint16_t> one(h, 0x3F80);  // bf16 1.0: RMSNorm gains = 1
      SMO_CUDA_CHECK(cudaMemcpy(ones, one.data(), size_t(h) * 2, cudaMemcpyHostToDevice));
    }
    layers.resize(L);
    for (int l = 0; l < L; ++l) {
      Layer& ly = layers[l];
      ly.wqkv = dalloc<uint16_t>(size_t(qkv_w) * h);
      ly.wo = dalloc<uint16_t>(size_t(h) * nq * d);
      ly.router = dalloc<uint16_t>(size_t(E) * h);
      if (attn_cpu) {  // K/V in pinned host DRAM (the GPU appends through mapped memory)
        ly.kc = halloc_mapped<uint16_t>(kv_elems());
        ly.vc = halloc_mapped<uint16_t>(kv_elems());
      } else {
        ly.kc = dalloc<uint16_t>(kv_elems());
        ly.vc = dalloc<uint16_t>(kv_elems());
        SMO_CUDA_CHECK(cudaMemset(ly.kc, 0, kv_elems() * 2));
        SMO_CUDA_CHECK(cudaMemset(ly.vc, 0, kv_elems() * 2));
      }
      fill_uniform(ly.wqkv, size_t(qkv_w) * h, cfg.seed, tid::layer(l) + tid::kWqkv, 0, std::sqrt(3.0f / h), st);
      fill_uniform(ly.wo, size_t(h) * nq * d, cfg.seed, tid::layer(l) + tid::kWo, 0, std::sqrt(3.0f / (nq * d)),
                   st);
      fill_uniform(ly.router, size_t(E) * h, cfg.seed, tid::layer(l) + tid::kRouter, 0,
                   std::sqrt(3.0f / h) * cfg.router_scale, st);
      if (cfg.shared_inter > 0) {
        const size_t n = size_t(cfg.shared_inter) * h;
        ly.ws1 = dalloc<uint16_t>(n);
        ly.ws3 = dalloc<uint16_t>(n);
        ly.ws2 = dalloc<uint16_t>(n);
        fill_uniform(ly.ws1, n, cfg.seed, tid::layer(l) + tid::kShared + 0, 0, std::sqrt(3.0f / h), st);
        fill_uniform(ly.ws3, n, cfg.seed, tid::layer(l) + tid::kShared + 1, 0, std::sqrt(3.0f / h), st);
        fill_uniform(ly.ws2, n, cfg.seed, tid::layer(l) + tid::kShared + 2, 0, std::sqrt(3.0f / cfg.shared_inter), st);
      }
    }

    // drafter: dense decoder layers with the target's attention shape,
    // sharing the target's embedding and LM head (EAGLE convention)
    dL = cfg.draft_layers;
    dI = cfg.draft_inter;
    SMO_REQUIRE(dL >= 0 && (dL == 0 || (dI > 0 && dI % 128 == 0)),
                "engine: draft_inter must be a positive multiple of 128 when draft_layers > 0");
    dlayers.resize(dL);
    for (int l = 0; l < dL; ++l) {
      DLayer& dl = dlayers[l];
      const uint64_t base = tid::draft(l);
      dl.wqkv = dalloc<uint16_t>(size_t(qkv_w) * h);
      dl.wo = dalloc<uint16_t>(size_t(h) * nq * d);
      dl.w1 = dalloc<uint16_t>(size_t(dI) * h);
      dl.w3 = dalloc<uint16_t>(size_t(dI) * h);
      dl.w2 = dalloc<uint16_t>(size_t(h) * dI);
      dl.kc = dalloc<uint16_t>(kv_elems());
      dl.vc = dalloc<uint16_t>(kv_elems());
      SMO_CUDA_CHECK(cudaMemset(dl.kc, 0, kv_elems() * 2));
      SMO_CUDA_CHECK(cudaMemset(dl.vc, 0, kv_elems() * 2));
      fill_uniform(dl.wqkv, size_t(qkv_w) * h, cfg.seed, base + 1, 0, std::sqrt(3.0f / h), st);
      fill_uniform(dl.wo, size_t(h) * nq * d, cfg.seed, base + 2, 0, std::sqrt(3.0f / (nq * d)), st);
      fill_uniform(dl.w1, size_t(dI) * h, cfg.seed, base + 3, 0, std::sqrt(3.0f / h), st);
      fill_uniform(dl.w3, size_t(dI) * h, cfg.seed, base + 4, 0, std::sqrt(3.0f / h), st);
      fill_uniform(dl.w2, size_t(h) * dI, cfg.seed, base + 5, 0, std::sqrt(3.0f / dI), st);
    }

    // experts: generate each block on the device, stage to pinned host DRAM
    for (int e = 0; e < E; ++e)
      if (owns(e)) owned.push_back(e);
    host_bufs.assign(host_alias, nullptr);
    uint16_t* stage = dalloc<uint16_t>(blk_elems);
    xcomp = opt.compress_experts != 0;
    uint8_t* cenc = nullptr;
    int* d_ovf = nullptr;
    if (xcomp) {
      cblk_bytes = expert_code_bytes(blk_elems, 4);
      cenc = dalloc<uint8_t>(cblk_bytes);
      d_ovf = dalloc<int>(1);
      blk_coded.assign(size_t(host_alias) * E_loc, 0);
    }
    for (int a = 0; a < host_alias; ++a) {
      void* hp = nullptr;
      cudaError_t err = cudaHostAlloc(&hp, blk_bytes * E_loc, cudaHostAllocPortable);
      if (err != cudaSuccess)
        throw Error(SMO_CAPACITY, "engine: pinned host allocation of " + std::to_string(blk_bytes * E) +
                                      " bytes failed (" + cudaGetErrorString(err) + "); set host_alias_layers");
      host_bufs[a] = reinterpret_cast<uint16_t*>(hp);
      for (int e : owned) {
        const uint64_t base = tid::layer(a) + tid::kExpert + 3ull * e;
        fill_uniform(stage, size_t(hi) * h, cfg.seed, base + 0, 0, std::sqrt(3.0f / h), st);
        fill_uniform(stage + size_t(hi) * h, size_t(hi) * h, cfg.seed, base + 1, 0, std::sqrt(3.0f / h), st);
        fill_uniform(stage + 2 * size_t(hi) * h, size_t(h) * hi, cfg.seed, base + 2, 0, std::sqrt(3.0f / hi), st);
        uint16_t* hdst = host_bufs[a] + size_t(local(e)) * blk_elems;
        bool coded = false;
        for (int bits = 3; xcomp && !coded && bits <= 4; ++bits) {  // the narrowest code that holds the block
          SMO_CUDA_CHECK(cudaMemset(d_ovf, 0, sizeof(int)));
          expert_encode(stage, blk_elems, bits, cenc, d_ovf, st);
          int ovf = 0;
          SMO_CUDA_CHECK(cudaMemcpy(&ovf, d_ovf, sizeof(int), cudaMemcpyDeviceToHost));
          if (!ovf) {
            SMO_CUDA_CHECK(cudaMemcpy(hdst, cenc, expert_code_bytes(blk_elems, bits), cudaMemcpyDeviceToHost));
            blk_coded[size_t(a) * E_loc + local(e)] = uint8_t(bits);
            coded = true;
          }
        }
        if (!coded) SMO_CUDA_CHECK(cudaMemcpy(hdst, stage, blk_bytes, cudaMemcpyDeviceToHost));
      }
    }

    // HBM pool: slots x E staging blocks + hot-expert cache
    const int64_t cache_blocks = opt.expert_cache_bytes > 0 ? int64_t(opt.expert_cache_bytes / int64_t(blk_bytes)) : 0;
    cache_blk.assign(size_t(L) * E, -1);
    int placed = 0;
    for (int l = 0; l < L && placed < cache_blocks; ++l)
      for (int e : owned) {
        if (placed >= cache_blocks) break;
        cache_blk[size_t(l) * E + e] = slots * E_loc + placed;
        ++placed;
      }
    pool_blocks = slots * E_loc + placed;
    pool = dalloc<uint16_t>(size_t(pool_blocks) * blk_elems);
    coded_streamed.assign(size_t(L), {});
    if (xcomp) cstage = dalloc<uint8_t>(size_t(slots) * E_loc * cblk_bytes);
    for (int l = 0; l < L; ++l)
      for (int e : owned) {
        const int cb = cache_blk[size_t(l) * E + e];
        if (cb < 0) continue;
        const uint16_t* hsrc = host_bufs[host_layer(l)] + size_t(local(e)) * blk_elems;
        if (const int bits = code_bits(l, local(e))) {
          SMO_CUDA_CHECK(cudaMemcpy(cenc, hsrc, expert_code_bytes(blk_elems, bits), cudaMemcpyHostToDevice));
          expert_decode(cenc, blk_elems, bits, pool + size_t(cb) * blk_elems, st);
        } else {
          SMO_CUDA_CHECK(cudaMemcpy(pool + size_t(cb) * blk_elems, hsrc, blk_bytes, cudaMemcpyHostToDevice));
        }
      }
    std::vector<int32_t> widx(size_t(L) * E);
    for (int l = 0; l < L; ++l)
      for (int e = 0; e < E; ++e) {
        const int cb = cache_blk[size_t(l) * E + e];
        widx[size_t(l) * E + e] = cb >= 0 ? cb : (l % slots) * E_loc + local(e);
      }
    d_w_index = dalloc<int32_t>(widx.size());
    SMO_CUDA_CHECK(cudaMemcpy(d_w_index, widx.data(), widx.size() * 4, cudaMemcpyHostToDevice));
    if (ep_on) {  // local expert le of this rank = global expert le*P + rank
      std::vector<int32_t> wl(size_t(L) * E_loc);
      for (int l = 0; l < L; ++l)
        for (int le = 0; le < E_loc; ++le) wl[size_t(l) * E_loc + le] = widx[size_t(l) * E + le * P + opt.ep_rank];
      d_w_index_loc = dalloc<int32_t>(wl.size());
      SMO_CUDA_CHECK(cudaMemcpy(d_w_index_loc, wl.data(), wl.size() * 4, cudaMemcpyHostToDevice));
    }
    slot_ready.resize(slots);
    slot_free.resize(slots);
    for (int s = 0; s < slots; ++s) {
      SMO_CUDA_CHECK(cudaEventCreateWithFlags(&slot_ready[s], cudaEventDisableTiming));
      SMO_CUDA_CHECK(cudaEventCreateWithFlags(&slot_free[s], cudaEventDisableTiming));
    }

    // activations
    const int P = maxT * K;
    x = dalloc<float>(size_t(maxT) * h);
    xn = dalloc<uint16_t>(size_t(maxT) * h);
    qkv = dalloc<uint16_t>(size_t(maxT) * qkv_w);
    q = dalloc<uint16_t>(size_t(maxT) * nq * d);
    attn = dalloc<uint16_t>(size_t(maxT) * nq * d);
    ids = dalloc<int32_t>(P);
    rw = dalloc<float>(P);
    offsets = dalloc<int32_t>(E + 1);
    perm = dalloc<int32_t>(P);
    pos = dalloc<int32_t>(P);
    xp = dalloc<uint16_t>(size_t(P) * h);
    if (cfg.shared_inter > 0) hs = dalloc<uint16_t>(size_t(maxT) * cfg.shared_inter);
    if (ep_on) {
      // fixed capacity per destination: every local (token, slot) pair could
      // target one owner; identical on all ranks (same options)
      C = P;
      const int PR = this->P;
      blk_d = (size_t(C) * h * 2 + size_t(E_loc) * 4 + 15) & ~size_t(15);
      oid = dalloc<int32_t>(P);
      pos_ep = dalloc<int32_t>(P);
      offsets_l = dalloc<int32_t>(E_loc + 1);
      back = dalloc<int32_t>(size_t(PR) * C);
      ep_send = dalloc<uint8_t>(size_t(PR) * blk_d);
      ep_recv = dalloc<uint8_t>(size_t(PR) * blk_d);
      xl = dalloc<uint16_t>(size_t(PR) * C * h);
      yl = dalloc<float>(size_t(4) * PR * C * h);  // room for the fused kernel's down slices
      ep_sendback = dalloc<float>(size_t(PR) * C * h);
      ep_recvback = dalloc<float>(size_t(PR) * C * h);
      hbuf = dalloc<uint16_t>(size_t(PR) * C * hi);
    } else {
      hbuf = dalloc<uint16_t>(size_t(P) * hi);
    }
    {
      const char* f = std::getenv("SMO_MOE_FUSED");
      moe_fused = !(f && f[0] == '0');
    }
    // fused MoE down splits from the GLOBAL shapes (every EP rank uses the
    // same S, so expert parallelism reproduces one GPU bit for bit)
    moe_splits = moe_fused ? pick_moe_splits(maxT * K, h, hi, E, 4) : 1;
    ybuf = dalloc<float>(size_t(moe_splits) * P * h);
    d_done = dalloc<int>(64);
    amax_v = dalloc<float>(size_t(maxT) * (V / 128));
    amax_i = dalloc<int32_t>(size_t(maxT) * (V / 128));
    target = dalloc<int32_t>(maxT);
    d_tokens = dalloc<int32_t>(maxT);
    d_parent = dalloc<int32_t>(maxT);
    d_prefix = dalloc<int32_t>(maxB);
    d_acc = dalloc<int32_t>(maxB);
    d_bonus = dalloc<int32_t>(maxB);
    d_keep = dalloc<int32_t>(maxT);
    d_mask = dalloc<uint64_t>(maxT);
    smo_attn_args wa{};
    wa.b = maxB;
    wa.n = maxN;
    wa.n_q = nq;
    wa.n_kv = nkv;
    wa.d = d;
    wa.s_max = s_max;
    wa.max_prefix = s_max - maxN;
    wa.q = wa.k_cache = wa.v_cache = wa.out = reinterpret_cast<void*>(1);
    wa.mask = reinterpret_cast<const uint64_t*>(1);
    wa.prefix_len = reinterpret_cast<const int32_t*>(1);
    attn_ws_bytes = attention_workspace(wa);
    // (the flat-schedule workspace is sized for a full grid at maxB, any prefix)
    attn_ws = dalloc<uint8_t>(attn_ws_bytes);
    SMO_CUDA_CHECK(cudaMemset(attn_ws, 0, attn_ws_bytes));  // K1's pair counters start at zero
    {
      smo_gemm_args g{};
      g.rows = maxT;
      g.groups = 1;
      g.max_rows_per_group = maxT;
      g.epilogue = SMO_EPI_BF16;
      g.K = h;
      g.N = qkv_w;
      gemm_ws_bytes = gemm_workspace(g);
      g.K = nq * d;
      g.N = h;
      g.epilogue = SMO_EPI_F32_ADD;
      gemm_ws_bytes = std::max(gemm_ws_bytes, gemm_workspace(g));
      // smaller batches plan more splits: bound by 8 splits of the widest output
      gemm_ws_bytes = std::max(gemm_ws_bytes, size_t(8) * maxT * std::max(qkv_w, h) * sizeof(float));
      gemm_ws = dalloc<uint8_t>(gemm_ws_bytes);
    }
    layer_bytes.assign(size_t(L), 0.0);
    layer_raw_bytes.assign(size_t(L), 0.0);
    if (batch_one) h_offsets = halloc_mapped<int32_t>(size_t(E) + 1);
    if (attn_cpu) {
      q_host = halloc_mapped<uint16_t>(size_t(maxT) * nq * d);
      attn_host = halloc_mapped<uint16_t>(size_t(maxT) * nq * d);
      prefix_host = halloc_mapped<int32_t>(maxB);
      mask_host = halloc_mapped<uint64_t>(maxT);
      host_jobs.resize(size_t(L));
    }
    // drafter + decode-loop state
    if (dL > 0) dh = dalloc<uint16_t>(size_t(maxT) * dI);
    d_dtok = dalloc<int32_t>(maxB);
    d_dpos = dalloc<int32_t>(maxB);
    d_dout = dalloc<int32_t>(maxB);
    d_mask1 = dalloc<uint64_t>(maxB);
    {
      std::vector<uint64_t> one(maxB, 1ull);
      SMO_CUDA_CHECK(cudaMemcpy(d_mask1, one.data(), size_t(maxB) * 8, cudaMemcpyHostToDevice));
    }
    hist_cap = s_max;
    d_kvlen = dalloc<int32_t>(maxB);
    d_root = dalloc<int32_t>(maxB);
    d_hist = dalloc<int32_t>(size_t(maxB) * hist_cap);
    d_hist_n = dalloc<int32_t>(maxB);
    d_dec_tok = dalloc<int32_t>(maxT);
    d_drafts = dalloc<int32_t>(maxT);
    d_dec_parent = dalloc<int32_t>(maxT);
    {
      std::vector<void*> ptrs;
      for (int l = 0; l < L; ++l) ptrs.push_back(layers[l].kc);
      for (int l = 0; l < dL; ++l) ptrs.push_back(dlayers[l].kc);
      for (int l = 0; l < L; ++l) ptrs.push_back(layers[l].vc);
      for (int l = 0; l < dL; ++l) ptrs.push_back(dlayers[l].vc);
      d_cache_ptrs = dalloc<void*>(ptrs.size());
      SMO_CUDA_CHECK(cudaMemcpy(d_cache_ptrs, ptrs.data(), ptrs.size() * sizeof(void*), cudaMemcpyHostToDevice));
    }
    h_stage_elems = size_t(maxT) * 4 + maxB * 4;
    SMO_CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&h_stage), h_stage_elems * 4, cudaHostAllocPortable));
    ev.resize(8 + size_t(L) * 8);
    for (auto& e : ev) SMO_CUDA_CHECK(cudaEventCreate(&e));
    draft_ev.resize(size_t(maxN) + 1);
    for (auto& e : draft_ev) SMO_CUDA_CHECK(cudaEventCreate(&e));
    SMO_CUDA_CHECK(cudaDeviceSynchronize());
  }

  void fill_prefix(const int32_t* prefix_host, int b) {
    SMO_REQUIRE(b > 0 && b <= maxB, "fill_prefix: bad batch");
    for (int r = 0; r < b; ++r)
      SMO_REQUIRE(prefix_host[r] >= 0 && prefix_host[r] + maxN <= s_max, "fill_prefix: prefix exceeds max_seq");
    SMO_CUDA_CHECK(cudaDeviceSynchronize());
    SMO_CUDA_CHECK(cudaMemcpy(d_prefix, prefix_host, size_t(b) * 4, cudaMemcpyHostToDevice));
    bt_reset();
    for (int r = 0; r < b; ++r) {
      bt_ensure(r, int64_t(prefix_host[r]) + maxN);
      kv_known[size_t(r)] = prefix_host[r];
    }
    bt_sync(nullptr);
    for (int l = 0; l < L; ++l) {
      fill_kv_prefix(layers[l].kc, d_prefix, b, nkv, d, s_max, cfg.seed, tid::kv(l, 0), nullptr, bt(), max_pages);
      fill_kv_prefix(layers[l].vc, d_prefix, b, nkv, d, s_max, cfg.seed, tid::kv(l, 1), nullptr, bt(), max_pages);
    }
    for (int l = 0; l < dL; ++l) {
      fill_kv_prefix(dlayers[l].kc, d_prefix, b, nkv, d, s_max, cfg.seed, tid::draft_kv(l, 0), nullptr, bt(),
                     max_pages);
      fill_kv_prefix(dlayers[l].vc, d_prefix, b, nkv, d, s_max, cfg.seed, tid::draft_kv(l, 1), nullptr, bt(),
                     max_pages);
    }
    SMO_CUDA_CHECK(cudaDeviceSynchronize());
  }

  // Stream layer l's non-cached owned experts into slot l % slots.
  // owned expert e -> its local index (host block / staging slot position)
  int local(int e) const { return P > 1 ? e / P : e; }

  // Stream layer l's non-cached owned experts into slot l % slots. Host and
  // slot blocks are in local order, so runs of consecutive local experts go
  // out as one copy (a whole layer when nothing is cached: 2.8 GB for 8x7B).
  // active (optional, BATCH_ONE): per local expert, 0 = not routed to -> not streamed
  double enqueue_h2d(int l, cudaEvent_t t0, cudaEvent_t t1, const uint8_t* active = nullptr) {
    const int s = l % slots;
    // while capturing a graph the first `slots` layers' release events belong
    // to the previous iteration (outside the graph; replays are serialised)
    if (!(capturing && l < slots)) SMO_CUDA_CHECK(cudaStreamWaitEvent(copy, slot_free[s], 0));
    if (t0) SMO_CUDA_CHECK(cudaEventRecord(t0, copy));
    double bytes = 0;
    const uint16_t* hb = host_bufs[host_layer(l)];
    auto streamed = [&](int le) {
      return cache_blk[size_t(l) * E + owned[size_t(le)]] < 0 && (!active || active[le]);
    };
    coded_streamed[size_t(l)].clear();
    if (xcomp) {
      // coded blocks into cstage (expanded by decode_slot), raw ones straight into the slot
      for (int q = 0; q < E_loc; ++q) {
        if (!streamed(q)) continue;
        if (const int bits = code_bits(l, q)) {
          const size_t cb = expert_code_bytes(blk_elems, bits);
          SMO_CUDA_CHECK(cudaMemcpyAsync(cstage + (size_t(s) * E_loc + q) * cblk_bytes, hb + size_t(q) * blk_elems,
                                         cb, cudaMemcpyHostToDevice, copy));
          bytes += double(cb);
          coded_streamed[size_t(l)].push_back(q);
        } else {
          SMO_CUDA_CHECK(cudaMemcpyAsync(pool + (size_t(s) * E_loc + q) * blk_elems, hb + size_t(q) * blk_elems,
                                         blk_bytes, cudaMemcpyHostToDevice, copy));
          bytes += double(blk_bytes);
        }
      }
    }
    int le = xcomp ? E_loc : 0;
    while (le < E_loc) {
      if (!streamed(le)) {
        ++le;
        continue;
      }
      int le2 = le;
      while (le2 + 1 < E_loc && streamed(le2 + 1)) ++le2;
      const size_t nbytes = size_t(le2 - le + 1) * blk_bytes;
      SMO_CUDA_CHECK(cudaMemcpyAsync(pool + (size_t(s) * E_loc + le) * blk_elems, hb + size_t(le) * blk_elems, nbytes,
                                     cudaMemcpyHostToDevice, copy));
      bytes += double(nbytes);
      le = le2 + 1;
    }
    if (t1) SMO_CUDA_CHECK(cudaEventRecord(t1, copy));
    SMO_CUDA_CHECK(cudaEventRecord(slot_ready[s], copy));
    layer_bytes[size_t(l)] = bytes;
    int nstreamed = 0;
    for (int q = 0; q < E_loc; ++q) nstreamed += streamed(q) ? 1 : 0;
    layer_raw_bytes[size_t(l)] = double(nstreamed) * double(blk_bytes);
    return bytes;
  }

  void snap(const char* name, int layer, const void* src, size_t bytes, cudaStream_t st) {
    if (!debug) return;
    auto& v = dbg[name];
    const size_t idx = size_t(layer + 1);
    if (v.size() <= idx) v.resize(idx + 1);
    if (v[idx].bytes < bytes) {
      if (v[idx].p) cudaFree(v[idx].p);
      SMO_CUDA_CHECK(cudaMalloc(&v[idx].p, bytes));
      v[idx].bytes = bytes;
    }
    SMO_CUDA_CHECK(cudaMemcpyAsync(v[idx].p, src, bytes, cudaMemcpyDeviceToDevice, st));
  }

  // Expert-parallel MoE of layer l (ep.cu): dispatch, local shard, combine.
  void moe_ep(int l, int T, cudaStream_t st) {
    const int PT = T * K;
    const int rank = opt.ep_rank;
    ep_pack(xp, offsets, P, E_loc, C, h, blk_d, ep_send, st);
    ep_pos(oid, pos, offsets, PT, E_loc, C, pos_ep, st);
    ept->alltoall(rank, ep_send, ep_recv, blk_d, st);
    ep_unpack(ep_recv, P, E_loc, C, h, blk_d, xl, offsets_l, back, st);
    SMO_CUDA_CHECK(cudaEventRecord(tev(l * 8 + 7), st));
    SMO_CUDA_CHECK(cudaStreamWaitEvent(st, slot_ready[l % slots], 0));
    decode_slot(l, st);
    SMO_CUDA_CHECK(cudaEventRecord(tev(l * 8 + 4), st));
    if (moe_fused) {
      moe_launch(xl, P * C, h, hi, E_loc, offsets_l, pool, blk_bytes, pool_blocks, d_w_index_loc + size_t(l) * E_loc,
                 hbuf, yl, moe_splits, 4, d_done, st);
      SMO_CUDA_CHECK(cudaEventRecord(slot_free[l % slots], st));
      ep_pack_back(yl, back, offsets_l, E_loc, h, ep_sendback, st, moe_splits, size_t(P) * C * h);
      ept->alltoall(rank, ep_sendback, ep_recvback, size_t(C) * h * sizeof(float), st);
      unpermute_combine(ep_recvback, pos_ep, rw, T, K, h, x, st);
      return;
    }
    smo_gemm_args g{};
    g.x = xl;
    g.rows = P * C;
    g.K = h;
    g.N = hi;
    g.groups = E_loc;
    g.row_offsets = offsets_l;
    g.max_rows_per_group = P * maxT;
    g.w = pool;
    g.w_up = pool + size_t(hi) * h;
    g.w_block_stride = blk_bytes;
    g.w_pool_blocks = pool_blocks;
    g.w_index = d_w_index_loc + size_t(l) * E_loc;
    g.epilogue = SMO_EPI_SWIGLU;
    g.out = hbuf;
    g.ldo = hi;
    gemm_launch(g, st);
    g = smo_gemm_args{};
    g.x = hbuf;
    g.rows = P * C;
    g.K = hi;
    g.N = h;
    g.groups = E_loc;
    g.row_offsets = offsets_l;
    g.max_rows_per_group = P * maxT;
    g.w = pool + 2 * size_t(hi) * h;
    g.w_block_stride = blk_bytes;
    g.w_pool_blocks = pool_blocks;
    g.w_index = d_w_index_loc + size_t(l) * E_loc;
    g.epilogue = SMO_EPI_F32;
    g.out = yl;
    g.ldo = h;
    gemm_launch(g, st);
    SMO_CUDA_CHECK(cudaEventRecord(slot_free[l % slots], st));
    ep_pack_back(yl, back, offsets_l, E_loc, h, ep_sendback, st);
    ept->alltoall(rank, ep_sendback, ep_recvback, size_t(C) * h * sizeof(float), st);
    unpermute_combine(ep_recvback, pos_ep, rw, T, K, h, x, st);
  }

  cudaEvent_t tev(int i) const { return ev[8 + size_t(i)]; }

  void verify(const smo_verify_batch& in, smo_verify_output& out, cudaStream_t st) {
    const int b = in.b, n = in.n, T = b * n;
    SMO_REQUIRE(b > 0 && b <= maxB && n > 0 && n <= maxN, "verify: batch exceeds engine capacity");
    SMO_REQUIRE(in.tokens && in.prefix_len, "verify: null tokens/prefix_len");
    SMO_REQUIRE(out.acc_len && out.bonus, "verify: null outputs");
    const uint64_t l0 = 0;
    (void)l0;
    // ---- inputs
    int max_prefix = s_max - n;
    if (in.on_device) {
      SMO_CUDA_CHECK(cudaMemcpyAsync(d_tokens, in.tokens, size_t(T) * 4, cudaMemcpyDeviceToDevice, st));
      SMO_CUDA_CHECK(cudaMemcpyAsync(d_prefix, in.prefix_len, size_t(b) * 4, cudaMemcpyDeviceToDevice, st));
      if (in.parent)
        SMO_CUDA_CHECK(cudaMemcpyAsync(d_parent, in.parent, size_t(T) * 4, cudaMemcpyDeviceToDevice, st));
    } else {
      max_prefix = 0;
      for (int r = 0; r < b; ++r) {
        SMO_REQUIRE(in.prefix_len[r] >= 0 && in.prefix_len[r] + n <= s_max, "verify: prefix exceeds max_seq");
        max_prefix = std::max(max_prefix, in.prefix_len[r]);
      }
      SMO_CUDA_CHECK(cudaStreamSynchronize(st));  // staging buffer reuse
      int32_t* hs = h_stage;
      std::memcpy(hs, in.tokens, size_t(T) * 4);
      std::memcpy(hs + T, in.prefix_len, size_t(b) * 4);
      if (in.parent) std::memcpy(hs + T + b, in.parent, size_t(T) * 4);
      SMO_CUDA_CHECK(cudaMemcpyAsync(d_tokens, hs, size_t(T) * 4, cudaMemcpyHostToDevice, st));
      SMO_CUDA_CHECK(cudaMemcpyAsync(d_prefix, hs + T, size_t(b) * 4, cudaMemcpyHostToDevice, st));
      if (in.parent)
        SMO_CUDA_CHECK(cudaMemcpyAsync(d_parent, hs + T + b, size_t(T) * 4, cudaMemcpyHostToDevice, st));
    }
    const int32_t* parent = in.parent ? d_parent : nullptr;
    // pages for the appended rows (device inputs: up to the known lengths)
    for (int r = 0; r < b; ++r) {
      const int64_t pre = in.on_device ? kv_known[size_t(r)] : int64_t(in.prefix_len[r]);
      if (!in.on_device) kv_known[size_t(r)] = pre;
      bt_ensure(r, pre + n);
    }
    bt_sync(st);
    last_was_decode = false;
    begin_step(st, !batch_one);
    verify_core(b, n, d_tokens, parent, d_prefix, max_prefix, st);
    // ---- outputs
    if (out.on_device) {
      SMO_CUDA_CHECK(cudaMemcpyAsync(out.acc_len, d_acc, size_t(b) * 4, cudaMemcpyDeviceToDevice, st));
      SMO_CUDA_CHECK(cudaMemcpyAsync(out.bonus, d_bonus, size_t(b) * 4, cudaMemcpyDeviceToDevice, st));
      if (out.keep) SMO_CUDA_CHECK(cudaMemcpyAsync(out.keep, d_keep, size_t(T) * 4, cudaMemcpyDeviceToDevice, st));
      if (out.target)
        SMO_CUDA_CHECK(cudaMemcpyAsync(out.target, target, size_t(T) * 4, cudaMemcpyDeviceToDevice, st));
    } else {
      int32_t* hs = h_stage + 2 * size_t(T) + b;
      SMO_CUDA_CHECK(cudaMemcpyAsync(hs, d_acc, size_t(b) * 4, cudaMemcpyDeviceToHost, st));
      SMO_CUDA_CHECK(cudaMemcpyAsync(hs + b, d_bonus, size_t(b) * 4, cudaMemcpyDeviceToHost, st));
      SMO_CUDA_CHECK(cudaMemcpyAsync(hs + 2 * b, d_keep, size_t(T) * 4, cudaMemcpyDeviceToHost, st));
      SMO_CUDA_CHECK(cudaMemcpyAsync(hs + 2 * b + T, target, size_t(T) * 4, cudaMemcpyDeviceToHost, st));
      SMO_CUDA_CHECK(cudaStreamSynchronize(st));
      std::memcpy(out.acc_len, hs, size_t(b) * 4);
      std::memcpy(out.bonus, hs + b, size_t(b) * 4);
      if (out.keep) std::memcpy(out.keep, hs + 2 * b, size_t(T) * 4);
      if (out.target) std::memcpy(out.target, hs + 2 * b + T, size_t(T) * 4);
    }
  }

  // Step start: event 0, then the copy engine starts streaming the first
  // `slots` layers (it only waits for the slot-release edges). Called before
  // the drafter in a decode step so that the first transfers overlap drafting.
  double step_h2d_bytes = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> step_h2d_ev;
  void begin_step(cudaStream_t st, bool prefetch = true) {
    SMO_CUDA_CHECK(cudaEventRecord(ev[0], st));
    // order the copy stream after the step start (so H2D timing is step-relative)
    SMO_CUDA_CHECK(cudaStreamWaitEvent(copy, ev[0], 0));
    step_h2d_bytes = 0;
    step_h2d_ev.clear();
    std::fill(layer_bytes.begin(), layer_bytes.end(), 0.0);
    std::fill(layer_raw_bytes.begin(), layer_raw_bytes.end(), 0.0);
    for (int l = 0; prefetch && l < std::min(slots, L); ++l) {
      step_h2d_bytes += enqueue_h2d(l, tev(l * 8 + 0), tev(l * 8 + 1));
      step_h2d_ev.push_back({tev(l * 8 + 0), tev(l * 8 + 1)});
    }
  }

  // The target verification DAG on device inputs: tokens [b*n], parent
  // [b*n] or null, prefix [b]; results in d_acc / d_bonus / d_keep / target.
  void verify_core(int b, int n, const int32_t* tokens, const int32_t* parent, const int32_t* prefix, int max_prefix,
                   cudaStream_t st) {
    const int T = b * n;
    cudaEvent_t e_end = ev[1];
    double h2d_bytes = step_h2d_bytes;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> h2d_ev = step_h2d_ev, attn_ev, moe_ev;
    build_mask(parent, b, n, d_mask, st);
    embed(tokens, embed_w, T, h, x, st);

    const int PT = T * K;  // (token, slot) pairs
    for (int l = 0; l < L; ++l) {
      Layer& ly = layers[l];
      SMO_CUDA_CHECK(cudaEventRecord(tev(l * 8 + 6), st));
      snap("x_in", l, x, size_t(T) * h * 4, st);
      rmsnorm(x, ones, T, h, cfg.rms_eps, xn, st);
      snap("xn1", l, xn, size_t(T) * h * 2, st);
      smo_gemm_args g{};
      g.x = xn;
      g.rows = T;
      g.K = h;
      g.N = qkv_w;
      g.groups = 1;
      g.max_rows_per_group = T;
      g.w = ly.wqkv;
      g.w_pool_blocks = 1;
      g.epilogue = SMO_EPI_BF16;
      g.out = qkv;
      g.ldo = qkv_w;
      g.workspace = gemm_ws;
      g.workspace_bytes = gemm_ws_bytes;
      gemm_launch(g, st);
      uint16_t* q_dst = attn_cpu ? q_host : q;  // CPU placement: q straight into pinned host memory
      rope_append(qkv, prefix, parent, b, n, nq, nkv, d, s_max, cfg.rope_theta, q_dst, ly.kc, ly.vc, st, bt(),
                  max_pages);
      snap("q", l, q_dst, size_t(T) * nq * d * 2, st);
      smo_attn_args a{};
      a.q = q;
      a.k_cache = ly.kc;
      a.v_cache = ly.vc;
      a.block_table = bt();
      a.max_pages = max_pages;
      a.num_pages = num_pages;
      a.mask = d_mask;
      a.prefix_len = prefix;
      a.out = attn;
      a.b = b;
      a.n = n;
      a.n_q = nq;
      a.n_kv = nkv;
      a.d = d;
      a.s_max = s_max;
      a.max_prefix = max_prefix;
      a.workspace = attn_ws;
      a.workspace_bytes = attn_ws_bytes;
      SMO_CUDA_CHECK(cudaEventRecord(tev(l * 8 + 2), st));
      if (attn_cpu) {
        // the paper's CPU attention: prefix lengths and mask to the host, the
        // host pool attends over the host K/V, the output goes back for O-proj
        SMO_CUDA_CHECK(cudaMemcpyAsync(prefix_host, prefix, size_t(b) * 4, cudaMemcpyDeviceToHost, st));
        SMO_CUDA_CHECK(cudaMemcpyAsync(mask_host, d_mask, size_t(T) * 8, cudaMemcpyDeviceToHost, st));
        HostAttn& hj = host_jobs[size_t(l)];
        hj.pool = cpu_pool.get();
        hj.job = CpuAttnJob{q_host, ly.kc, ly.vc, mask_host, prefix_host, attn_host, b, n, nq, nkv, d, s_max, 1};
        SMO_CUDA_CHECK(cudaLaunchHostFunc(st, host_attn_cb, &hj));
        SMO_CUDA_CHECK(cudaMemcpyAsync(attn, attn_host, size_t(T) * nq * d * 2, cudaMemcpyHostToDevice, st));
      } else {
        attention_launch(a, st);
      }
      SMO_CUDA_CHECK(cudaEventRecord(tev(l * 8 + 3), st));
      attn_ev.push_back({tev(l * 8 + 2), tev(l * 8 + 3)});
      snap("attn", l, attn, size_t(T) * nq * d * 2, st);
      g = smo_gemm_args{};
      g.x = attn;
      g.rows = T;
      g.K = nq * d;
      g.N = h;
      g.groups = 1;
      g.max_rows_per_group = T;
      g.w = ly.wo;
      g.w_pool_blocks = 1;
      g.epilogue = SMO_EPI_F32_ADD;
      g.out = x;
      g.ldo = h;
      g.workspace = gemm_ws;
      g.workspace_bytes = gemm_ws_bytes;
      gemm_launch(g, st);
      rmsnorm(x, ones, T, h, cfg.rms_eps, xn, st);
      snap("xn2", l, xn, size_t(T) * h * 2, st);
      float* rlog = nullptr;
      if (debug) {
        auto& v = dbg["logits_r"];
        if (v.size() <= size_t(l + 1)) v.resize(l + 2);
        if (!v[l + 1].p) {
          SMO_CUDA_CHECK(cudaMalloc(&v[l + 1].p, size_t(maxT) * E * 4));
          v[l + 1].bytes = size_t(maxT) * E * 4;
        }
        rlog = reinterpret_cast<float*>(v[l + 1].p);
      }
      router_topk(xn, ly.router, T, h, E, K, rlog, ids, rw, st);
      if (ep_on) {  // owner-major order: rows bound for one rank are contiguous
        ep_remap(ids, T * K, P, E_loc, oid, st);
        permute(oid, T, K, E, xn, h, offsets, perm, pos, xp, st);
      } else {
        permute(ids, T, K, E, xn, h, offsets, perm, pos, xp, st);
      }
      snap("ids", l, ids, size_t(PT) * 4, st);
      snap("weights", l, rw, size_t(PT) * 4, st);
      snap("offsets", l, offsets, size_t(E + 1) * 4, st);
      snap("pos", l, pos, size_t(PT) * 4, st);
      if (batch_one) {
        // BATCH_ONE (optimizer.hpp:81-96): wait for this layer's routing, then
        // stream only the experts its tokens selected
        SMO_CUDA_CHECK(cudaMemcpyAsync(h_offsets, offsets, size_t(E + 1) * 4, cudaMemcpyDeviceToHost, st));
        SMO_CUDA_CHECK(cudaEventRecord(route_ev, st));
        SMO_CUDA_CHECK(cudaEventSynchronize(route_ev));
        std::vector<uint8_t> act(size_t(E_loc), 0);
        for (int e = 0; e < E; ++e) act[size_t(local(e))] = h_offsets[e + 1] > h_offsets[e] ? 1 : 0;
        h2d_bytes += enqueue_h2d(l, tev(l * 8 + 0), tev(l * 8 + 1), act.data());
        h2d_ev.push_back({tev(l * 8 + 0), tev(l * 8 + 1)});
      }
      if (cfg.shared_inter > 0) {
        // always-on shared expert (config 4): x += SwiGLU_shared(xn2); its
        // weights are resident, so it runs before the wait for streamed experts
        smo_gemm_args gs{};
        gs.x = xn;
        gs.rows = T;
        gs.K = h;
        gs.N = cfg.shared_inter;
        gs.groups = 1;
        gs.max_rows_per_group = T;
        gs.w = ly.ws1;
        gs.w_up = ly.ws3;
        gs.w_pool_blocks = 1;
        gs.epilogue = SMO_EPI_SWIGLU;
        gs.out = hs;
        gs.ldo = cfg.shared_inter;
        gemm_launch(gs, st);
        gs = smo_gemm_args{};
        gs.x = hs;
        gs.rows = T;
        gs.K = cfg.shared_inter;
        gs.N = h;
        gs.groups = 1;
        gs.max_rows_per_group = T;
        gs.w = ly.ws2;
        gs.w_pool_blocks = 1;
        gs.epilogue = SMO_EPI_F32_ADD;
        gs.out = x;
        gs.ldo = h;
        gs.workspace = gemm_ws;
        gs.workspace_bytes = gemm_ws_bytes;
        gemm_launch(gs, st);
      }
      // ---- MoE: wait for this layer's experts
      if (ep_on) {
        moe_ep(l, T, st);
      } else {
        SMO_CUDA_CHECK(cudaEventRecord(tev(l * 8 + 7), st));
        SMO_CUDA_CHECK(cudaStreamWaitEvent(st, slot_ready[l % slots], 0));
        decode_slot(l, st);  // coded expert blocks -> bf16 slot (compress_experts)
        SMO_CUDA_CHECK(cudaEventRecord(tev(l * 8 + 4), st));
        if (moe_fused) {
          moe_launch(xp, PT, h, hi, E, offsets, pool, blk_bytes, pool_blocks, d_w_index + size_t(l) * E, hbuf, ybuf,
                     moe_splits, moe_splits, d_done, st);
          SMO_CUDA_CHECK(cudaEventRecord(slot_free[l % slots], st));
          unpermute_combine(ybuf, pos, rw, T, K, h, x, st, moe_splits, size_t(PT) * h);
        } else {
        g = smo_gemm_args{};
        g.x = xp;
        g.rows = PT;
        g.K = h;
        g.N = hi;
        g.groups = E;
        g.row_offsets = offsets;
        g.max_rows_per_group = T;  // a token selects an expert at most once
        g.w = pool;
        g.w_up = pool + size_t(hi) * h;
        g.w_block_stride = blk_bytes;
        g.w_pool_blocks = pool_blocks;
        g.w_index = d_w_index + size_t(l) * E;
        g.epilogue = SMO_EPI_SWIGLU;
        g.out = hbuf;
        g.ldo = hi;
        gemm_launch(g, st);
        g = smo_gemm_args{};
        g.x = hbuf;
        g.rows = PT;
        g.K = hi;
        g.N = h;
        g.groups = E;
        g.row_offsets = offsets;
        g.max_rows_per_group = T;
        g.w = pool + 2 * size_t(hi) * h;
        g.w_block_stride = blk_bytes;
        g.w_pool_blocks = pool_blocks;
        g.w_index = d_w_index + size_t(l) * E;
        g.epilogue = SMO_EPI_F32;
        g.out = ybuf;
        g.ldo = h;
        gemm_launch(g, st);
        SMO_CUDA_CHECK(cudaEventRecord(slot_free[l % slots], st));
        unpermute_combine(ybuf, pos, rw, T, K, h, x, st);
        }
      }
      SMO_CUDA_CHECK(cudaEventRecord(tev(l * 8 + 5), st));
      moe_ev.push_back({tev(l * 8 + 4), tev(l * 8 + 5)});
      snap("x_out", l, x, size_t(T) * h * 4, st);
      if (!batch_one && l + slots < L) {
        const int ln = l + slots;
        h2d_bytes += enqueue_h2d(ln, tev(ln * 8 + 0), tev(ln * 8 + 1));
        h2d_ev.push_back({tev(ln * 8 + 0), tev(ln * 8 + 1)});
      }
    }
    // ---- LM head with fused argmax partials, then K6
    rmsnorm(x, final_norm, T, h, cfg.rms_eps, xn, st);
    snap("xf", -1, xn, size_t(T) * h * 2, st);
    smo_gemm_args g{};
    g.x = xn;
    g.rows = T;
    g.K = h;
    g.N = V;
    g.groups = 1;
    g.max_rows_per_group = T;
    g.w = lm_w;
    g.w_pool_blocks = 1;
    g.epilogue = SMO_EPI_ARGMAX;
    g.argmax_val = amax_v;
    g.argmax_idx = amax_i;
    gemm_launch(g, st);
    if (debug) {
      auto& v = dbg["logits"];
      if (v.empty()) v.resize(1);
      if (!v[0].p) {
        SMO_CUDA_CHECK(cudaMalloc(&v[0].p, size_t(maxT) * V * 4));
        v[0].bytes = size_t(maxT) * V * 4;
      }
      g.epilogue = SMO_EPI_F32;
      g.out = v[0].p;
      g.ldo = V;
      gemm_launch(g, st);
    }
    argmax_reduce(amax_v, amax_i, T, V / 128, target, st);
    greedy_accept(tokens, target, parent, b, n, d_acc, d_bonus, d_keep, st);
    SMO_CUDA_CHECK(cudaEventRecord(e_end, st));
    // the step is complete only when the copy engine is idle too
    SMO_CUDA_CHECK(cudaStreamWaitEvent(st, slot_ready[(L - 1) % slots], 0));
    pending_attn = attn_ev;
    pending_moe = moe_ev;
    pending_h2d = h2d_ev;
    last_h2d_bytes = h2d_bytes;
  }

  // ------------------------------------------------------------------ dense
  // building blocks shared by the drafter and the prefill
  struct Scratch {
    float* x;
    uint16_t *xn, *qkv, *q, *attn;
    void* attn_ws;
    size_t attn_ws_bytes;
    int split;  // 0: auto split-K (engine workspace), 1: off
  };

  void dense_gemm(const void* xin, int rows, int Kd, int N, const void* w, const void* w_up, int epi, void* out,
                  int split, cudaStream_t st) {
    smo_gemm_args g{};
    g.x = xin;
    g.rows = rows;
    g.K = Kd;
    g.N = N;
    g.groups = 1;
    g.max_rows_per_group = rows;
    g.w = w;
    g.w_up = w_up;
    g.w_pool_blocks = 1;
    g.epilogue = epi;
    g.out = out;
    g.ldo = N;
    g.split_k = split;
    if (split != 1) {
      g.workspace = gemm_ws;
      g.workspace_bytes = gemm_ws_bytes;
    }
    gemm_launch(g, st);
  }

  // x += Wo . attn(RoPE(Wqkv . rmsnorm(x))) for rows organised as `nch`
  // chunks of b*n verify rows; chunk c's row (r, i) sits at position
  // prefix[c*b + r] + i and sees the prefix plus the chain `mask`. K/V rows
  // are appended to kc/vc (the K1 contract of smo_verify_attention).
  void attn_sublayer(const Scratch& sc, const uint16_t* wqkv, const uint16_t* wo, uint16_t* kc, uint16_t* vc, int b,
                     int n, int nch, const int32_t* prefix, const std::vector<int>& max_prefix, const uint64_t* mask,
                     cudaStream_t st, const int32_t* parent = nullptr) {
    const int rows = b * n * nch;
    rmsnorm(sc.x, ones, rows, h, cfg.rms_eps, sc.xn, st);
    dense_gemm(sc.xn, rows, h, qkv_w, wqkv, nullptr, SMO_EPI_BF16, sc.qkv, sc.split, st);
    for (int c = 0; c < nch; ++c) {
      const size_t r0 = size_t(c) * b * n;
      rope_append(sc.qkv + r0 * qkv_w, prefix + size_t(c) * b, parent, b, n, nq, nkv, d, s_max, cfg.rope_theta,
                  sc.q + r0 * nq * d, kc, vc, st, bt(), max_pages);
      smo_attn_args a{};
      a.q = sc.q + r0 * nq * d;
      a.k_cache = kc;
      a.v_cache = vc;
      a.block_table = bt();
      a.max_pages = max_pages;
      a.num_pages = num_pages;
      a.mask = mask;
      a.prefix_len = prefix + size_t(c) * b;
      a.out = sc.attn + r0 * nq * d;
      a.b = b;
      a.n = n;
      a.n_q = nq;
      a.n_kv = nkv;
      a.d = d;
      a.s_max = s_max;
      a.max_prefix = max_prefix[size_t(c)];
      a.workspace = sc.attn_ws;
      a.workspace_bytes = sc.attn_ws_bytes;
      attention_launch(a, st);
    }
    dense_gemm(sc.attn, rows, nq * d, h, wo, nullptr, SMO_EPI_F32_ADD, sc.x, sc.split, st);
  }

  // attn_sublayer with the CPU placement: q and the appended K/V rows go to
  // pinned host memory, one host job attends over all `nch` chunks (chunk c
  // only sees its prefix + own rows), the output comes back for O-proj.
  // qh/ah: pinned mapped [b*n*nch, n_q, d]; pre_h [nch*b], mask_h [b*n] host.
  void attn_sublayer_cpu(const Scratch& sc, const uint16_t* wqkv, const uint16_t* wo, uint16_t* kc, uint16_t* vc,
                         int b, int n, int nch, const int32_t* prefix, uint16_t* qh, uint16_t* ah,
                         const int32_t* pre_h, const uint64_t* mask_h, HostAttn& job, cudaStream_t st) {
    const int rows = b * n * nch;
    rmsnorm(sc.x, ones, rows, h, cfg.rms_eps, sc.xn, st);
    dense_gemm(sc.xn, rows, h, qkv_w, wqkv, nullptr, SMO_EPI_BF16, sc.qkv, sc.split, st);
    for (int c = 0; c < nch; ++c) {
      const size_t r0 = size_t(c) * b * n;
      rope_append(sc.qkv + r0 * qkv_w, prefix + size_t(c) * b, nullptr, b, n, nq, nkv, d, s_max, cfg.rope_theta,
                  qh + r0 * nq * d, kc, vc, st);
    }
    job.pool = cpu_pool.get();
    job.job = CpuAttnJob{qh, kc, vc, mask_h, pre_h, ah, b, n, nq, nkv, d, s_max, nch};
    SMO_CUDA_CHECK(cudaLaunchHostFunc(st, host_attn_cb, &job));
    SMO_CUDA_CHECK(cudaMemcpyAsync(sc.attn, ah, size_t(rows) * nq * d * 2, cudaMemcpyHostToDevice, st));
    dense_gemm(sc.attn, rows, nq * d, h, wo, nullptr, SMO_EPI_F32_ADD, sc.x, sc.split, st);
  }

  // x += W2 . (silu(W1 . rmsnorm(x)) * W3 . rmsnorm(x))  (dense SwiGLU)
  void ffn_dense(const Scratch& sc, uint16_t* hb, int rows, const uint16_t* w1, const uint16_t* w3,
                 const uint16_t* w2, int inter, cudaStream_t st) {
    rmsnorm(sc.x, ones, rows, h, cfg.rms_eps, sc.xn, st);
    dense_gemm(sc.xn, rows, h, inter, w1, w3, SMO_EPI_SWIGLU, hb, 0, st);
    dense_gemm(hb, rows, inter, h, w2, nullptr, SMO_EPI_F32_ADD, sc.x, sc.split, st);
  }

  // final RMSNorm -> LM head with fused argmax partials -> per-row argmax
  void lm_argmax(const float* xr, int rows, int32_t* out, cudaStream_t st) {
    rmsnorm(xr, final_norm, rows, h, cfg.rms_eps, xn, st);
    smo_gemm_args g{};
    g.x = xn;
    g.rows = rows;
    g.K = h;
    g.N = V;
    g.groups = 1;
    g.max_rows_per_group = rows;
    g.w = lm_w;
    g.w_pool_blocks = 1;
    g.epilogue = SMO_EPI_ARGMAX;
    g.argmax_val = amax_v;
    g.argmax_idx = amax_i;
    gemm_launch(g, st);
    argmax_reduce(amax_v, amax_i, rows, V / 128, out, st);
  }

  // One drafter step for b requests: token tok_in[r] at position pos[r]
  // (its K/V appended there), greedy next token into out_tok[r].
  void draft_forward(int b, const int32_t* tok_in, const int32_t* pos, int max_pos, int32_t* out_tok,
                     cudaStream_t st) {
    const Scratch sc{x, xn, qkv, q, attn, attn_ws, attn_ws_bytes, 0};
    embed(tok_in, embed_w, b, h, x, st);
    const std::vector<int> mp{max_pos};
    for (auto& dl : dlayers) {
      attn_sublayer(sc, dl.wqkv, dl.wo, dl.kc, dl.vc, b, 1, 1, pos, mp, d_mask1, st);
      ffn_dense(sc, dh, b, dl.w1, dl.w3, dl.w2, dI, st);
    }
    lm_argmax(x, b, out_tok, st);
  }

  // ------------------------------------------------------------------ decode
  void decode_begin(const int32_t* root_h, const int32_t* kv_h, int b) {
    SMO_REQUIRE(b > 0 && b <= maxB, "decode_begin: batch exceeds engine capacity");
    int64_t mx = 0;
    for (int r = 0; r < b; ++r) {
      SMO_REQUIRE(kv_h[r] >= 0 && kv_h[r] < s_max, "decode_begin: kv_len out of range");
      SMO_REQUIRE(root_h[r] >= 0 && root_h[r] < V, "decode_begin: root token out of range");
      mx = std::max<int64_t>(mx, kv_h[r]);
    }
    SMO_CUDA_CHECK(cudaDeviceSynchronize());
    SMO_CUDA_CHECK(cudaMemcpy(d_root, root_h, size_t(b) * 4, cudaMemcpyHostToDevice));
    SMO_CUDA_CHECK(cudaMemcpy(d_kvlen, kv_h, size_t(b) * 4, cudaMemcpyHostToDevice));
    SMO_CUDA_CHECK(cudaMemset(d_hist_n, 0, size_t(maxB) * 4));
    SMO_CUDA_CHECK(cudaMemset(d_hist, 0xFF, size_t(maxB) * hist_cap * 4));
    for (int r = 0; r < b; ++r) {
      bt_ensure(r, int64_t(kv_h[r]) + 1);
      kv_known[size_t(r)] = kv_h[r];
    }
    bt_sync(nullptr);
    SMO_CUDA_CHECK(cudaDeviceSynchronize());
    dec_b = b;
    kv_bound = mx;
  }

  // draft (k+1 drafter steps) -> verify -> greedy accept -> commit, on device
  void decode_step(int k, const int32_t* drafts_h, cudaStream_t st, const int32_t* parents_h = nullptr) {
    const int b = dec_b, n = k + 1;
    SMO_REQUIRE(!parents_h || (drafts_h && k > 0), "decode: a draft tree needs planted drafts");
    SMO_REQUIRE(b > 0, "decode: call smo_engine_prefill or smo_engine_decode_begin first");
    SMO_REQUIRE(k >= 0 && n <= maxN, "decode: k + 1 exceeds max_verify");
    SMO_REQUIRE(kv_bound + n <= s_max, "decode: KV capacity (max_seq) exhausted");
    SMO_REQUIRE(drafts_h || k == 0 || dL > 0, "decode: k > 0 needs a drafter (draft_layers) or planted drafts");
    const bool planted = drafts_h && k > 0;
    for (int r = 0; r < b; ++r) {
      bt_ensure(r, kv_bound + n);
      kv_known[size_t(r)] = kv_bound + n;  // upper bound (the device holds the exact length)
    }
    bt_sync(st);
    if (planted) {
      SMO_CUDA_CHECK(cudaStreamSynchronize(st));  // staging buffer reuse
      std::memcpy(h_stage, drafts_h, size_t(b) * k * 4);
      SMO_CUDA_CHECK(cudaMemcpyAsync(d_drafts, h_stage, size_t(b) * k * 4, cudaMemcpyHostToDevice, st));
    }
    if (parents_h) {
      for (int r = 0; r < b; ++r) {
        SMO_REQUIRE(parents_h[size_t(r) * n] == -1, "decode: tree node 0 is the root (parent -1)");
        for (int i = 1; i < n; ++i)
          SMO_REQUIRE(parents_h[size_t(r) * n + i] >= 0 && parents_h[size_t(r) * n + i] < i,
                      "decode: tree parents must precede their children");
      }
      int32_t* hp = h_stage + size_t(b) * k;
      std::memcpy(hp, parents_h, size_t(b) * n * 4);
      SMO_CUDA_CHECK(cudaMemcpyAsync(d_dec_parent, hp, size_t(b) * n * 4, cudaMemcpyHostToDevice, st));
    }
    decode_device(k, planted, int(kv_bound), st, parents_h != nullptr);
    kv_bound += n;
  }

  // The device part of a decode step (capturable into a CUDA graph): every
  // argument is fixed at enqueue time; bound = host bound of kv_len used for
  // K1 split planning and the drafter's positions.
  void decode_device(int k, bool planted, int bound, cudaStream_t st, bool tree = false) {
    const int b = dec_b, n = k + 1;
    last_was_decode = true;
    begin_step(st, !batch_one);  // the first layers' experts stream while the drafter runs
    decode_prep(d_root, planted ? d_drafts : nullptr, b, n, d_dec_tok, st);
    if (tree) {
      // planted draft tree: the drafter runs its layers over all n nodes at
      // once (tree positions and mask) so its K/V covers every node; verify
      // with the tree mask; the accepted root path's K/V rows of every target
      // and drafter layer are compacted to kv_len + j; commit along it
      last_draft_steps = dL > 0 ? 1 : 0;
      if (dL > 0) SMO_CUDA_CHECK(cudaEventRecord(draft_ev[0], st));
      if (dL > 0) {
        build_mask(d_dec_parent, b, n, d_mask, st);
        const Scratch sc{x, xn, qkv, q, attn, attn_ws, attn_ws_bytes, 0};
        embed(d_dec_tok, embed_w, b * n, h, x, st);
        const std::vector<int> mp{bound};
        for (auto& dl : dlayers) {
          attn_sublayer(sc, dl.wqkv, dl.wo, dl.kc, dl.vc, b, n, 1, d_kvlen, mp, d_mask, st, d_dec_parent);
          ffn_dense(sc, dh, b * n, dl.w1, dl.w3, dl.w2, dI, st);
        }
      }
      SMO_CUDA_CHECK(cudaEventRecord(ev[3], st));
      if (dL > 0) SMO_CUDA_CHECK(cudaEventRecord(draft_ev[1], st));
      verify_core(b, n, d_dec_tok, d_dec_parent, d_kvlen, bound, st);
      void* const* kp = d_cache_ptrs;
      void* const* vp = d_cache_ptrs + (L + dL);
      kv_rollback(kp, vp, L + dL, d_kvlen, d_acc, d_keep, b, n, nkv, d, s_max, nullptr, st, bt(), max_pages);
      decode_commit(d_dec_tok, d_acc, d_bonus, b, n, hist_cap, d_hist, d_hist_n, d_kvlen, d_root, st, d_keep);
      return;
    }
    // drafter: step t consumes row t (root, d_1, ..., d_k) at kv_len + t and
    // proposes d_{t+1}; the extra step t = k only appends d_k's draft K/V so
    // that a fully accepted chain leaves no hole in the drafter's cache
    last_draft_steps = dL > 0 ? k + 1 : 0;
    for (int t = 0; dL > 0 && t <= k; ++t) {
      SMO_CUDA_CHECK(cudaEventRecord(draft_ev[size_t(t)], st));
      draft_io(d_dec_tok, d_kvlen, t, b, n, d_dtok, d_dpos, st);
      draft_forward(b, d_dtok, d_dpos, bound + t, d_dout, st);
      if (!planted && t < k) draft_scatter(d_dout, b, n, t, d_dec_tok, st);
    }
    SMO_CUDA_CHECK(cudaEventRecord(ev[3], st));
    if (last_draft_steps > 0) SMO_CUDA_CHECK(cudaEventRecord(draft_ev[size_t(last_draft_steps)], st));
    verify_core(b, n, d_dec_tok, nullptr, d_kvlen, bound, st);
    decode_commit(d_dec_tok, d_acc, d_bonus, b, n, hist_cap, d_hist, d_hist_n, d_kvlen, d_root, st);
  }

  // `steps` decode iterations with k drafts. graph: the device part of one
  // iteration is captured once into a CUDA graph (keyed on k, batch and the
  // kv bound it was planned for) and replayed — one launch per iteration
  // instead of ~15 per layer. Graph replays on one stream are serialised, so
  // the cross-iteration slot-release edges hold without the in-graph waits.
  cudaGraphExec_t graph_exec = nullptr;
  int graph_k = -1, graph_b = -1;
  int64_t graph_bound = -1;
  uint64_t graph_launches = 0;
  bool capturing = false;
  void decode_run(int k, int steps, bool graph, cudaStream_t st) {
    if (!graph) {
      for (int i = 0; i < steps; ++i) decode_step(k, nullptr, st);
      return;
    }
    const int b = dec_b, n = k + 1;
    SMO_REQUIRE(b > 0, "decode: call smo_engine_prefill or smo_engine_decode_begin first");
    SMO_REQUIRE(k >= 0 && n <= maxN, "decode: k + 1 exceeds max_verify");
    SMO_REQUIRE(k == 0 || dL > 0, "decode: k > 0 needs a drafter (draft_layers)");
    SMO_REQUIRE(!batch_one && !attn_cpu && !ep_on && !debug,
                "decode graph: not with BATCH_ONE, CPU attention, expert parallelism or debug snapshots");
    SMO_REQUIRE(st != nullptr, "decode graph: needs a non-default stream");
    const int64_t end = kv_bound + int64_t(steps) * n;  // kv bound after the last iteration
    SMO_REQUIRE(end <= s_max, "decode: KV capacity (max_seq) exhausted");
    for (int r = 0; r < b; ++r) {  // pages for every iteration of the run, outside the graph
      bt_ensure(r, end);
      kv_known[size_t(r)] = end;
    }
    bt_sync(st);
    // one graph serves any run whose positions stay under the bound it was planned for
    const int64_t plan = std::max<int64_t>(end - n, graph_bound);
    if (!graph_exec || graph_k != k || graph_b != b || graph_bound < end - n) {
      if (graph_exec) SMO_CUDA_CHECK(cudaGraphExecDestroy(graph_exec));
      graph_exec = nullptr;
      const int64_t bound = std::min<int64_t>(plan, s_max - n);
      const uint64_t l0 = smo_launch_count();
      cudaGraph_t g = nullptr;
      SMO_CUDA_CHECK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      capturing = true;
      try {
        decode_device(k, false, int(bound), st);
      } catch (...) {
        capturing = false;
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      capturing = false;
      SMO_CUDA_CHECK(cudaStreamEndCapture(st, &g));
      SMO_CUDA_CHECK(cudaGraphInstantiate(&graph_exec, g, 0));
      SMO_CUDA_CHECK(cudaGraphDestroy(g));
      graph_launches = smo_launch_count() - l0;
      count_launch(-int(graph_launches));  // captured, not launched: counted per replay below
      graph_k = k;
      graph_b = b;
      graph_bound = bound;
    }
    for (int i = 0; i < steps; ++i) {
      SMO_CUDA_CHECK(cudaGraphLaunch(graph_exec, st));
      count_launch(int(graph_launches));
    }
    last_was_decode = true;
    last_draft_steps = dL > 0 ? k + 1 : 0;
    kv_bound = end;
  }

  // durations (s) of the drafter steps of the last decode step; returns count
  int draft_times(double* out, size_t n) {
    SMO_CUDA_CHECK(cudaDeviceSynchronize());
    if (!last_was_decode) return 0;
    const int m = last_draft_steps;
    SMO_REQUIRE(n >= size_t(m), "draft_times: output too small");
    for (int t = 0; t < m; ++t) {
      float ms = 0;
      SMO_CUDA_CHECK(cudaEventElapsedTime(&ms, draft_ev[size_t(t)], draft_ev[size_t(t) + 1]));
      out[t] = ms * 1e-3;
    }
    return m;
  }

  void decode_read(int32_t* committed, int cap, int32_t* n_committed, int32_t* kv_len, int32_t* root) {
    SMO_REQUIRE(dec_b > 0, "decode_read: no decode state");
    const int b = dec_b;
    SMO_CUDA_CHECK(cudaDeviceSynchronize());
    if (committed) {
      SMO_REQUIRE(cap > 0, "decode_read: bad capacity");
      std::vector<int32_t> hh(size_t(b) * hist_cap);
      SMO_CUDA_CHECK(cudaMemcpy(hh.data(), d_hist, hh.size() * 4, cudaMemcpyDeviceToHost));
      for (int r = 0; r < b; ++r)
        for (int j = 0; j < cap; ++j) committed[size_t(r) * cap + j] = j < hist_cap ? hh[size_t(r) * hist_cap + j] : -1;
    }
    if (n_committed) SMO_CUDA_CHECK(cudaMemcpy(n_committed, d_hist_n, size_t(b) * 4, cudaMemcpyDeviceToHost));
    if (kv_len) SMO_CUDA_CHECK(cudaMemcpy(kv_len, d_kvlen, size_t(b) * 4, cudaMemcpyDeviceToHost));
    if (root) SMO_CUDA_CHECK(cudaMemcpy(root, d_root, size_t(b) * 4, cudaMemcpyDeviceToHost));
  }

  // SMO_PREFILL_CHECK=1: host scan for non-finite values after each prefill
  // stage (diagnostics only; synchronises)
  static bool prefill_check_on() {
    const char* e = std::getenv("SMO_PREFILL_CHECK");
    return e && e[0] == '1';
  }
  void check_finite(const char* what, int layer, const void* p, size_t count, bool bf16, cudaStream_t st) {
    SMO_CUDA_CHECK(cudaStreamSynchronize(st));
    std::vector<uint16_t> hb;
    std::vector<float> hf;
    size_t bad = 0, first = 0;
    if (bf16) {
      hb.resize(count);
      SMO_CUDA_CHECK(cudaMemcpy(hb.data(), p, count * 2, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < count; ++i)
        if (!std::isfinite(bf2f(hb[i])) && !bad++) first = i;
    } else {
      hf.resize(count);
      SMO_CUDA_CHECK(cudaMemcpy(hf.data(), p, count * 4, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < count; ++i)
        if (!std::isfinite(hf[i]) && !bad++) first = i;
    }
    std::fprintf(stderr, "[prefill-check] L%d %-8s %zu non-finite of %zu (first at %zu)\n", layer, what, bad, count,
                 first);
  }

  // ------------------------------------------------------------------ prefill
  // Layer-major prefill: every layer's experts are streamed once for the
  // whole prompt batch; attention runs the prompt as causal chunks of C rows.
  void prefill(const int32_t* tok_h, const int32_t* len_h, int b, int Lmax, int32_t* next_h, cudaStream_t st) {
    SMO_REQUIRE(!ep_on, "prefill: not available with expert parallelism");
    SMO_REQUIRE(b > 0 && b <= maxB && Lmax > 0, "prefill: bad batch");
    SMO_REQUIRE(tok_h && len_h && next_h, "prefill: null argument");
    const int g = nq / nkv;
    const int C = std::max(1, std::min(64, 128 / g));
    const int nch = (Lmax + C - 1) / C;
    SMO_REQUIRE(int64_t(nch) * C + maxN <= s_max, "prefill: prompt exceeds max_seq");
    for (int r = 0; r < b; ++r) SMO_REQUIRE(len_h[r] >= 1 && len_h[r] <= Lmax, "prefill: len out of range");
    const int Tp = b * nch * C;
    std::vector<int32_t> tok(size_t(Tp), 0), pre(size_t(nch) * b);
    for (int c = 0; c < nch; ++c)
      for (int r = 0; r < b; ++r) {
        pre[size_t(c) * b + r] = c * C;
        for (int i = 0; i < C; ++i) {
          const int p = c * C + i;
          const int32_t t = p < len_h[r] ? tok_h[size_t(r) * Lmax + p] : 0;
          SMO_REQUIRE(t >= 0 && t < V, "prefill: token out of range");
          tok[(size_t(c) * b + r) * C + i] = t;
        }
      }
    std::vector<int> maxpre(static_cast<size_t>(nch));
    for (int c = 0; c < nch; ++c) maxpre[size_t(c)] = c * C;
    // prompt-sized scratch (freed at the end: prefill is not a per-step call)
    std::vector<void*> tmp;
    auto talloc = [&](size_t bytes) {
      void* p = nullptr;
      cudaError_t e = cudaMalloc(&p, std::max<size_t>(bytes, 16));
      if (e != cudaSuccess) {
        for (void* q2 : tmp) cudaFree(q2);
        throw Error(SMO_CAPACITY, "prefill: cudaMalloc(" + std::to_string(bytes) + ") failed");
      }
      tmp.push_back(p);
      return p;
    };
    const int PT = Tp * K;
    auto* p_tok = static_cast<int32_t*>(talloc(size_t(Tp) * 4));
    auto* p_pre = static_cast<int32_t*>(talloc(pre.size() * 4));
    auto* p_len = static_cast<int32_t*>(talloc(size_t(b) * 4));
    auto* p_mask = static_cast<uint64_t*>(talloc(size_t(b) * C * 8));
    Scratch sc{};
    sc.x = static_cast<float*>(talloc(size_t(Tp) * h * 4));
    sc.xn = static_cast<uint16_t*>(talloc(size_t(Tp) * h * 2));
    sc.qkv = static_cast<uint16_t*>(talloc(size_t(Tp) * qkv_w * 2));
    sc.q = static_cast<uint16_t*>(talloc(size_t(Tp) * nq * d * 2));
    sc.attn = static_cast<uint16_t*>(talloc(size_t(Tp) * nq * d * 2));
    sc.split = 1;  // prompt-sized row counts fill the SMs without split-K
    {
      smo_attn_args wa{};
      wa.b = b;
      wa.n = C;
      wa.n_q = nq;
      wa.n_kv = nkv;
      wa.d = d;
      wa.s_max = s_max;
      wa.max_prefix = (nch - 1) * C;
      wa.q = wa.k_cache = wa.v_cache = wa.out = reinterpret_cast<void*>(1);
      wa.mask = reinterpret_cast<const uint64_t*>(1);
      wa.prefix_len = reinterpret_cast<const int32_t*>(1);
      sc.attn_ws_bytes = attention_workspace(wa);
      sc.attn_ws = talloc(sc.attn_ws_bytes);
      SMO_CUDA_CHECK(cudaMemsetAsync(sc.attn_ws, 0, sc.attn_ws_bytes, st));
    }
    auto* p_ids = static_cast<int32_t*>(talloc(size_t(PT) * 4));
    auto* p_rw = static_cast<float*>(talloc(size_t(PT) * 4));
    auto* p_off = static_cast<int32_t*>(talloc(size_t(E + 1) * 4));
    auto* p_perm = static_cast<int32_t*>(talloc(size_t(PT) * 4));
    auto* p_pos = static_cast<int32_t*>(talloc(size_t(PT) * 4));
    auto* p_xp = static_cast<uint16_t*>(talloc(size_t(PT) * h * 2));
    auto* p_hb = static_cast<uint16_t*>(talloc(size_t(PT) * hi * 2));
    const int pf_splits = moe_fused ? pick_moe_splits(PT, h, hi, E, 2) : 1;
    auto* p_y = static_cast<float*>(talloc(size_t(pf_splits) * PT * h * 4));
    uint16_t* p_hs = cfg.shared_inter > 0 ? static_cast<uint16_t*>(talloc(size_t(Tp) * cfg.shared_inter * 2)) : nullptr;
    uint16_t* p_dh = dL > 0 ? static_cast<uint16_t*>(talloc(size_t(Tp) * dI * 2)) : nullptr;
    // CPU placement: pinned host q / attention rows, prefix and chain mask
    std::vector<void*> htmp;
    std::vector<HostAttn> pf_jobs(attn_cpu ? size_t(L) : 0);
    uint16_t *pq_h = nullptr, *pa_h = nullptr;
    int32_t* ppre_h = nullptr;
    uint64_t* pmask_h = nullptr;
    if (attn_cpu) {
      auto hal = [&](size_t bytes) {
        void* hp = nullptr;
        if (cudaHostAlloc(&hp, std::max<size_t>(bytes, 16), cudaHostAllocPortable | cudaHostAllocMapped) !=
            cudaSuccess) {
          for (void* q2 : htmp) cudaFreeHost(q2);
          for (void* q2 : tmp) cudaFree(q2);
          throw Error(SMO_CAPACITY, "prefill: pinned host allocation failed");
        }
        htmp.push_back(hp);
        return hp;
      };
      pq_h = static_cast<uint16_t*>(hal(size_t(Tp) * nq * d * 2));
      pa_h = static_cast<uint16_t*>(hal(size_t(Tp) * nq * d * 2));
      ppre_h = static_cast<int32_t*>(hal(pre.size() * 4));
      pmask_h = static_cast<uint64_t*>(hal(size_t(b) * C * 8));
      std::memcpy(ppre_h, pre.data(), pre.size() * 4);
      for (int r = 0; r < b; ++r)
        for (int i = 0; i < C; ++i) pmask_h[size_t(r) * C + i] = i >= 63 ? ~0ull : ((1ull << (i + 1)) - 1ull);
    }
    SMO_CUDA_CHECK(cudaStreamSynchronize(st));
    bt_reset();
    for (int r = 0; r < b; ++r) {
      bt_ensure(r, int64_t(nch) * C);  // the padded chunk rows are appended too
      kv_known[size_t(r)] = len_h[r];
    }
    bt_sync(st);
    SMO_CUDA_CHECK(cudaMemcpyAsync(p_tok, tok.data(), tok.size() * 4, cudaMemcpyHostToDevice, st));
    SMO_CUDA_CHECK(cudaMemcpyAsync(p_pre, pre.data(), pre.size() * 4, cudaMemcpyHostToDevice, st));
    SMO_CUDA_CHECK(cudaMemcpyAsync(p_len, len_h, size_t(b) * 4, cudaMemcpyHostToDevice, st));
    build_mask(nullptr, b, C, p_mask, st);

    // target: layer-major, experts streamed once per layer
    last_was_decode = false;
    begin_step(st);
    double h2d_bytes = step_h2d_bytes;
    embed(p_tok, embed_w, Tp, h, sc.x, st);
    for (int l = 0; l < L; ++l) {
      Layer& ly = layers[l];
      const bool chk = prefill_check_on();
      if (chk) check_finite("x_in", l, sc.x, size_t(Tp) * h, false, st);
      if (attn_cpu)
        attn_sublayer_cpu(sc, ly.wqkv, ly.wo, ly.kc, ly.vc, b, C, nch, p_pre, pq_h, pa_h, ppre_h, pmask_h,
                          pf_jobs[size_t(l)], st);
      else
        attn_sublayer(sc, ly.wqkv, ly.wo, ly.kc, ly.vc, b, C, nch, p_pre, maxpre, p_mask, st);
      if (chk) {
        check_finite("qkv", l, sc.qkv, size_t(Tp) * qkv_w, true, st);
        check_finite("q", l, sc.q, size_t(Tp) * nq * d, true, st);
        check_finite("attn", l, sc.attn, size_t(Tp) * nq * d, true, st);
        check_finite("x_mid", l, sc.x, size_t(Tp) * h, false, st);
      }
      rmsnorm(sc.x, ones, Tp, h, cfg.rms_eps, sc.xn, st);
      router_topk(sc.xn, ly.router, Tp, h, E, K, nullptr, p_ids, p_rw, st);
      permute(p_ids, Tp, K, E, sc.xn, h, p_off, p_perm, p_pos, p_xp, st);
      if (chk) check_finite("xp", l, p_xp, size_t(PT) * h, true, st);
      if (cfg.shared_inter > 0) {
        dense_gemm(sc.xn, Tp, h, cfg.shared_inter, ly.ws1, ly.ws3, SMO_EPI_SWIGLU, p_hs, 1, st);
        dense_gemm(p_hs, Tp, cfg.shared_inter, h, ly.ws2, nullptr, SMO_EPI_F32_ADD, sc.x, 1, st);
      }
      SMO_CUDA_CHECK(cudaStreamWaitEvent(st, slot_ready[l % slots], 0));
      decode_slot(l, st);
      if (moe_fused) {
        moe_launch(p_xp, PT, h, hi, E, p_off, pool, blk_bytes, pool_blocks, d_w_index + size_t(l) * E, p_hb, p_y,
                   pf_splits, pf_splits, d_done, st);
      } else {
      smo_gemm_args g2{};
      g2.x = p_xp;
      g2.rows = PT;
      g2.K = h;
      g2.N = hi;
      g2.groups = E;
      g2.row_offsets = p_off;
      g2.max_rows_per_group = Tp;
      g2.w = pool;
      g2.w_up = pool + size_t(hi) * h;
      g2.w_block_stride = blk_bytes;
      g2.w_pool_blocks = pool_blocks;
      g2.w_index = d_w_index + size_t(l) * E;
      g2.epilogue = SMO_EPI_SWIGLU;
      g2.out = p_hb;
      g2.ldo = hi;
      gemm_launch(g2, st);
      g2 = smo_gemm_args{};
      g2.x = p_hb;
      g2.rows = PT;
      g2.K = hi;
      g2.N = h;
      g2.groups = E;
      g2.row_offsets = p_off;
      g2.max_rows_per_group = Tp;
      g2.w = pool + 2 * size_t(hi) * h;
      g2.w_block_stride = blk_bytes;
      g2.w_pool_blocks = pool_blocks;
      g2.w_index = d_w_index + size_t(l) * E;
      g2.epilogue = SMO_EPI_F32;
      g2.out = p_y;
      g2.ldo = h;
      gemm_launch(g2, st);
      }
      SMO_CUDA_CHECK(cudaEventRecord(slot_free[l % slots], st));
      if (chk) {
        check_finite("h_swiglu", l, p_hb, size_t(PT) * hi, true, st);
        check_finite("y_down", l, p_y, size_t(PT) * h, false, st);
      }
      unpermute_combine(p_y, p_pos, p_rw, Tp, K, h, sc.x, st, pf_splits, size_t(PT) * h);
      if (l + slots < L) h2d_bytes += enqueue_h2d(l + slots, nullptr, nullptr);
    }
    SMO_CUDA_CHECK(cudaStreamWaitEvent(st, slot_ready[(L - 1) % slots], 0));
    prefill_last(sc.x, p_len, b, C, h, x, st);
    lm_argmax(x, b, d_root, st);
    // drafter: its own residual stream over the same prompt
    if (dL > 0) {
      embed(p_tok, embed_w, Tp, h, sc.x, st);
      for (auto& dl : dlayers) {
        attn_sublayer(sc, dl.wqkv, dl.wo, dl.kc, dl.vc, b, C, nch, p_pre, maxpre, p_mask, st);
        ffn_dense(sc, p_dh, Tp, dl.w1, dl.w3, dl.w2, dI, st);
      }
    }
    SMO_CUDA_CHECK(cudaEventRecord(ev[1], st));
    SMO_CUDA_CHECK(cudaMemcpyAsync(d_kvlen, p_len, size_t(b) * 4, cudaMemcpyDeviceToDevice, st));
    SMO_CUDA_CHECK(cudaMemsetAsync(d_hist_n, 0, size_t(maxB) * 4, st));
    SMO_CUDA_CHECK(cudaMemsetAsync(d_hist, 0xFF, size_t(maxB) * hist_cap * 4, st));
    SMO_CUDA_CHECK(cudaMemcpyAsync(next_h, d_root, size_t(b) * 4, cudaMemcpyDeviceToHost, st));
    SMO_CUDA_CHECK(cudaStreamSynchronize(st));
    for (void* p : tmp) cudaFree(p);
    for (void* p : htmp) cudaFreeHost(p);
    pending_attn.clear();
    pending_moe.clear();
    pending_h2d.clear();
    last_h2d_bytes = h2d_bytes;
    dec_b = b;
    kv_bound = Lmax;
  }

  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending_attn, pending_moe, pending_h2d;

  // Per layer: [h2d_start, h2d_end, attn_start, attn_end, moe_start, moe_end,
  // layer_start, pre_moe] in seconds from the step's start event.
  void layer_times(double* out, size_t n) {
    SMO_REQUIRE(n >= size_t(L) * 9, "layer_times: output too small");
    SMO_CUDA_CHECK(cudaDeviceSynchronize());
    for (int l = 0; l < L; ++l) {
      for (int k = 0; k < 8; ++k) {
        float ms = 0;
        SMO_CUDA_CHECK(cudaEventElapsedTime(&ms, ev[0], ev[8 + size_t(l) * 8 + k]));
        out[size_t(l) * 9 + k] = ms * 1e-3;
      }
      out[size_t(l) * 9 + 8] = layer_bytes[size_t(l)];
    }
  }

  void times(smo_stage_times* t) {
    SMO_CUDA_CHECK(cudaDeviceSynchronize());
    auto span = [](const std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v) {
      double s = 0;
      for (auto& p : v) {
        float ms = 0;
        if (cudaEventElapsedTime(&ms, p.first, p.second) == cudaSuccess) s += ms * 1e-3;
      }
      return s;
    };
    smo_stage_times r{};
    float ms = 0;
    if (last_was_decode) {  // iteration = draft (ev0 -> ev3) + target (ev3 -> ev1)
      float md = 0;
      cudaEventElapsedTime(&md, ev[0], ev[3]);
      cudaEventElapsedTime(&ms, ev[3], ev[1]);
      r.draft = md * 1e-3;
    } else {
      cudaEventElapsedTime(&ms, ev[0], ev[1]);
    }
    r.target_total = ms * 1e-3;
    r.attention = span(pending_attn);
    r.gpu_moe = span(pending_moe);
    r.h2d_transfer = span(pending_h2d);
    r.h2d_bytes = last_h2d_bytes;
    for (double v : layer_raw_bytes) r.h2d_raw_bytes += v;
    r.others = std::max(0.0, r.target_total - r.attention - r.gpu_moe);
    *t = r;
  }
};

}  // namespace smo

struct smo_engine {
  smo::Engine impl;
};

extern "C" {

smo_status smo_engine_create(const smo_model_config* cfg, const smo_engine_options* opt, smo_engine** out) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(cfg && opt && out, "engine: null argument");
    auto* e = new smo_engine();
    e->impl.cfg = *cfg;
    e->impl.opt = *opt;
    try {
      e->impl.create();
    } catch (...) {
      delete e;
      throw;
    }
    *out = e;
  });
}

smo_status smo_engine_destroy(smo_engine* e) {
  return smo::run_guarded([&] { delete e; });
}

smo_status smo_engine_fill_prefix(smo_engine* e, const int32_t* prefix_len_host, int32_t b) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(e && prefix_len_host, "engine: null argument");
    e->impl.fill_prefix(prefix_len_host, b);
  });
}

smo_status smo_engine_verify(smo_engine* e, const smo_verify_batch* in, smo_verify_output* out,
                             smo_stream stream) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(e && in && out, "engine: null argument");
    e->impl.verify(*in, *out, reinterpret_cast<cudaStream_t>(stream));
  });
}

smo_status smo_engine_prefill(smo_engine* e, const int32_t* tokens, const int32_t* len, int32_t b, int32_t max_len,
                              int32_t* next_token, smo_stream stream) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(e, "engine: null argument");
    e->impl.prefill(tokens, len, b, max_len, next_token, reinterpret_cast<cudaStream_t>(stream));
  });
}

smo_status smo_engine_decode_begin(smo_engine* e, const int32_t* root, const int32_t* kv_len, int32_t b) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(e && root && kv_len, "engine: null argument");
    e->impl.decode_begin(root, kv_len, b);
  });
}

smo_status smo_engine_decode_step(smo_engine* e, int32_t k, const int32_t* drafts, smo_stream stream) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(e, "engine: null argument");
    e->impl.decode_step(k, drafts, reinterpret_cast<cudaStream_t>(stream));
  });
}

smo_status smo_engine_decode_step_tree(smo_engine* e, int32_t n, const int32_t* tokens, const int32_t* parents,
                                       smo_stream stream) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(e && tokens && parents && n >= 2, "engine: bad argument");
    e->impl.decode_step(n - 1, tokens, reinterpret_cast<cudaStream_t>(stream), parents);
  });
}

smo_status smo_engine_decode_run(smo_engine* e, int32_t k, int32_t steps, int32_t use_graph, smo_stream stream) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(e && steps >= 0, "engine: bad argument");
    e->impl.decode_run(k, steps, use_graph != 0, reinterpret_cast<cudaStream_t>(stream));
  });
}

smo_status smo_engine_decode_read(smo_engine* e, int32_t* committed, int32_t cap, int32_t* n_committed,
                                  int32_t* kv_len, int32_t* root) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(e, "engine: null argument");
    e->impl.decode_read(committed, cap, n_committed, kv_len, root);
  });
}

smo_status smo_engine_draft_times(smo_engine* e, double* out, size_t n, int32_t* steps) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(e && out && steps, "engine: null argument");
    *steps = e->impl.draft_times(out, n);
  });
}

smo_status smo_engine_last_times(smo_engine* e, smo_stage_times* t) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(e && t, "engine: null argument");
    e->impl.times(t);
  });
}

smo_status smo_engine_layer_times(smo_engine* e, double* out, size_t n) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(e && out, "engine: null argument");
    e->impl.layer_times(out, n);
  });
}

smo_status smo_engine_debug_tensor(smo_engine* e, const char* name, int32_t layer, void* dst, size_t bytes) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(e && name && dst, "engine: null argument");
    SMO_REQUIRE(e->impl.debug, "engine: created without SMO_ENGINE_DEBUG");
    const std::string nm(name);
    if (nm == "k_cache" || nm == "v_cache" || nm == "draft_k_cache" || nm == "draft_v_cache") {
      // live cache contents of a (target or drafter) layer
      smo::Engine& g = e->impl;
      const bool dr = nm.rfind("draft_", 0) == 0;
      SMO_REQUIRE(layer >= 0 && layer < (dr ? g.dL : g.L), "engine: layer out of range");
      const size_t cb = g.kv_elems() * 2;
      SMO_REQUIRE(bytes <= cb, "engine: debug tensor smaller than requested");
      SMO_CUDA_CHECK(cudaDeviceSynchronize());
      const bool kk = nm == "k_cache" || nm == "draft_k_cache";
      const void* src = dr ? (kk ? g.dlayers[layer].kc : g.dlayers[layer].vc)
                           : (kk ? g.layers[layer].kc : g.layers[layer].vc);
      SMO_CUDA_CHECK(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
      return;
    }
    auto it = e->impl.dbg.find(name);
    SMO_REQUIRE(it != e->impl.dbg.end(), std::string("engine: unknown debug tensor ") + name);
    const size_t idx = size_t(layer + 1);
    SMO_REQUIRE(idx < it->second.size() && it->second[idx].p, "engine: debug tensor not captured for layer");
    SMO_REQUIRE(bytes <= it->second[idx].bytes, "engine: debug tensor smaller than requested");
    SMO_CUDA_CHECK(cudaDeviceSynchronize());
    SMO_CUDA_CHECK(cudaMemcpy(dst, it->second[idx].p, bytes, cudaMemcpyDeviceToHost));
  });
}

smo_status smo_engine_tensor_ptr(smo_engine* e, const char* name, int32_t layer, int32_t expert, void** ptr,
                                 size_t* bytes) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(e && name && ptr && bytes, "engine: null argument");
    smo::Engine& g = e->impl;
    const std::string n(name);
    auto need_layer = [&] { SMO_REQUIRE(layer >= 0 && layer < g.L, "engine: layer out of range"); };
    if (n == "embed") {
      *ptr = g.embed_w;
      *bytes = size_t(g.V) * g.h * 2;
    } else if (n == "lm_head") {
      *ptr = g.lm_w;
      *bytes = size_t(g.V) * g.h * 2;
    } else if (n == "wqkv") {
      need_layer();
      *ptr = g.layers[layer].wqkv;
      *bytes = size_t(g.qkv_w) * g.h * 2;
    } else if (n == "wo") {
      need_layer();
      *ptr = g.layers[layer].wo;
      *bytes = size_t(g.h) * g.nq * g.d * 2;
    } else if (n == "router") {
      need_layer();
      *ptr = g.layers[layer].router;
      *bytes = size_t(g.E) * g.h * 2;
    } else if (n == "k_cache" || n == "v_cache") {
      need_layer();
      *ptr = n == "k_cache" ? g.layers[layer].kc : g.layers[layer].vc;
      *bytes = g.kv_elems() * 2;
    } else if (n == "expert_host") {
      need_layer();
      SMO_REQUIRE(expert >= 0 && expert < g.E, "engine: expert out of range");
      SMO_REQUIRE(g.owns(expert), "engine: expert not owned by this rank");
      *ptr = g.host_bufs[g.host_layer(layer)] + size_t(g.local(expert)) * g.blk_elems;
      *bytes = g.blk_bytes;
    } else {
      throw smo::Error(SMO_INVALID_ARG, "engine: unknown tensor " + n);
    }
  });
}

}  // extern "C"
