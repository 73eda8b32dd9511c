// engine.cuh — the Engine behind the smo_engine_* C-ABI (definitions in
// engine.cu: creation, expert streaming, the verify DAG; decode.cu: dense
// blocks, drafter, decode loop; prefill.cu: layer-major prefill).
#pragma once
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <functional>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
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
             cudaStream_t st, uint8_t* const* dests = nullptr);
void ep_pos(const int32_t* oid, const int32_t* pos, const int32_t* offsets, int n, int E_loc, int C, int32_t* pos_ep,
            cudaStream_t st);
void ep_unpack(const void* recv, int P, int E_loc, int C, int h, size_t block_bytes, void* xl, int32_t* offsets_l,
               int32_t* back, cudaStream_t st);
void ep_pack_back(const float* yl, const int32_t* back, const int32_t* offsets_l, int E_loc, int h, float* sendback,
                  cudaStream_t st, int splits = 1, size_t split_stride = 0, uint8_t* const* dests = nullptr,
                  int C = 1);
int moe_launch(const void* x_perm, int rows, int h, int hi, int E, const int32_t* offsets, const void* pool,
               uint64_t w_block_stride, int pool_blocks, const int32_t* w_index, void* hbuf, float* y, int splits,
               int max_splits, int* done, cudaStream_t st);
int pick_moe_splits(int rows, int h, int hi, int E, int max_splits);
size_t expert_code_bytes(size_t count, int bits);
size_t expert_coded_size(const void* code, size_t count, int bits);
void expert_encode(const void* src, size_t count, int bits, void* dst, int* overflow, cudaStream_t st);
void expert_decode(const void* src, size_t count, int bits, void* dst, cudaStream_t st);
void expert_decode_blocks(const void* const* srcs, void* const* dsts, int n, size_t count, int bits, cudaStream_t st);
size_t tcode_max_bytes(int h, int hi);
size_t tcode_encode(const void* src, int h, int hi, void* dst, cudaStream_t st, int fmt = 2);
void tcode_decode(const void* const* srcs, void* const* dsts, int n, int h, int hi, cudaStream_t st, int fmt = 2);
int moe_coded_launch(const void* x_perm, int rows, int h, int hi, int E, const int32_t* offsets,
                     const void* const* w_code, void* hbuf, float* y, int splits, int max_splits, int* done,
                     cudaStream_t st, int fmt = 2);

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

// Pinned host memory for the expert blocks, placed on a NUMA node (the
// GPU's own, so each rank's shard crosses only its local root complex):
// mmap + mbind(MPOL_BIND) + cudaHostRegister; bytes_out = 0 when it fell
// back to cudaHostAlloc (single-node hosts, SMO_HOST_NUMA=-1, any failure).
int device_numa_node(int device);
void* pinned_alloc(size_t bytes, int node, size_t* bytes_out);
void pinned_free(void* p, size_t numa_bytes);

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
  // drafter GPU-part / CPU-part split (build_draft_dag
  // pipeline.hpp:217-253): requests [draft_g, dec_b) keep their drafter K/V
  // in pinned host memory (dkc_h / dvc_h, contiguous [maxB][n_kv][s_max][d])
  // and attend on the host pool while the GPU part runs K1
  bool draft_cpu = false;
  int draft_g = -1;  // GPU-part requests; -1: all
  std::vector<uint16_t*> dkc_h, dvc_h;
  uint16_t *dq_h = nullptr, *da_h = nullptr;  // pinned mapped [maxB, n_q, d]: CPU-part q / attention out
  int32_t* dpos_h = nullptr;                  // pinned mapped [maxB]: CPU-part positions (= prefix)
  uint64_t* dmask_h = nullptr;                // pinned [maxB]: bit 0 (the row sees itself)
  std::vector<cudaEvent_t> join_ev;           // [maxN]: host join of each drafter step
  std::vector<std::vector<uint32_t>> step_seqs;  // host job sequence numbers of each drafter step
  bool last_split = false;
  void set_draft_split(int g);
  int draft_split_times(double* out, size_t n);
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
  std::vector<HostAttn> host_jobs;        // [L][kMaxMb] (enqueued ahead of execution)
  // Asynchronous host attention (verify steps outside graph capture): the
  // GPU publishes "job seq's q rows are written" in pinned mapped memory
  // (ready_flag); a dispatcher thread takes the jobs in order, waits for
  // that, runs the job on the pool, then publishes "job seq done"
  // (done_flag); the compute stream only waits for done right before the
  // job's output is consumed (wait_host_flag), so the GPU keeps running the
  // other micro-batches' stages while the host attends (no stream-blocking
  // host function). Jobs are queued by value with monotonically increasing
  // sequence numbers, so steps may be issued ahead without reusing state.
  struct AsyncHost {
    struct Item {
      CpuAttnJob job;
      CpuPool* pool;
      uint32_t seq;
    };
    std::thread th;
    std::mutex mu;
    std::atomic<uint64_t> dur_ns[256];  // wall time of job seq (ring by seq & 255)
    std::condition_variable cv;
    std::vector<Item> q;
    size_t head = 0;
    bool stop = false;
    volatile uint32_t* ready_flag = nullptr;  // written by the GPU
    volatile uint32_t* done_flag = nullptr;   // written by the dispatcher
    void start(volatile uint32_t* ready, volatile uint32_t* done);
    void push(const Item& it);
    void shutdown();
    ~AsyncHost() { shutdown(); }
  };
  AsyncHost async_host;
  uint32_t* host_flags = nullptr;  // pinned mapped [2]: GPU-ready seq, host-done seq
  uint32_t host_seq = 0;           // last enqueued host job
  void signal_host_ready(uint32_t seq, cudaStream_t st);
  void copy_from_mapped(void* dst, const void* src, size_t bytes, cudaStream_t st);
  void wait_host_flag(uint32_t seq, cudaStream_t st);
  // BATCH_ONE expert streaming: stream only router-selected experts
  bool batch_one = false;
  int32_t* h_offsets = nullptr;           // pinned [E+1] routed offsets of the current layer
  cudaEvent_t route_ev = nullptr;
  // BATCH_ONE link-gap prefetch: while layer l+1's routing is computed the
  // link would idle; it carries (prefixes of) the experts most routed at
  // layer l into layer l+1's staging instead, sized from the previous step's
  // measured gap (SMO_B1_PREFETCH=0 disables)
  bool b1_prefetch = true;
  bool b1_measured = false;                // the last step left a gap timeline
  std::vector<double> b1_budget;          // [L] bytes to prefetch after layer l's copies
  std::vector<size_t> spec_done;          // [E_loc] bytes of layer spec_layer already staged
  int spec_layer = -1;
  double b1_prefetch_step(int l, cudaStream_t copy_st);
  void b1_update_budget();
  std::vector<double> layer_bytes;        // bytes streamed per layer in the last step
  std::vector<double> layer_raw_bytes;    // their bf16 size (coded blocks expand)
  // lossless expert codec on the link (xfer.cu): coded blocks cross into
  // cstage and are expanded into the pool slot on the compute stream
  bool xcomp = false;
  // T2 tile code (tcode.cuh; compress_experts = 2 or SMO_CODEC=tile): every
  // block crosses the link and sits in HBM (staging and hot cache) in the
  // tile code, and K4-MoE decodes it in shared memory (moe_coded_launch):
  // no expansion launch, no bf16 copy of an expert in HBM
  bool tmode = false;
  int tfmt = 2;  // the tile code: 2 (T2) or 3 (T3, fixed 3-bit exponents)
  const void** d_w_code = nullptr;      // [L*E] code block of (layer, expert)
  const void** d_w_code_loc = nullptr;  // [L*E_loc] (expert parallelism)
  size_t cblk_bytes = 0;                  // coded bytes of one [W1|W3|W2] block at 4 bits (staging stride)
  std::vector<uint8_t> blk_coded;         // [host_alias * E_loc] code of the host block: 0 raw, 1 unary, 3 / 4 bits
  std::vector<size_t> blk_csize;          // [host_alias * E_loc] coded bytes of the host block
  uint8_t* cstage = nullptr;              // [slots][E_loc][cblk_bytes]
  std::vector<std::vector<int>> coded_streamed;  // per layer: local experts streamed coded
  std::vector<cudaEvent_t> dec_ev;        // [2L] around each layer's block expansion
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> step_dec_ev;
  std::vector<cudaEvent_t> draft_ev;  // [maxN + 1]: boundaries of the drafter steps
  int last_draft_steps = 0;
  std::vector<uint16_t*> host_bufs;  // pinned, E blocks each
  std::vector<size_t> host_numa_bytes;  // > 0: placed on the GPU's NUMA node (mmap + mbind + cudaHostRegister)
  int host_numa = -1;                   // NUMA node of the expert buffers (-1: default placement)
  int host_alias = 0;
  // expert pool in HBM
  uint16_t* pool = nullptr;
  int slots = 2, pool_blocks = 0;
  std::vector<int> cache_blk;  // [L*E] pool block of a cached expert, kCachedCoded, -1 = streamed
  double step_codec_bytes = 0;                  // code read + bf16 written by this step's expansions
  static constexpr int kCachedCoded = -2;       // cached in its link code in `ccache`, expanded per step
  uint8_t* ccache = nullptr;                    // coded hot cache
  std::vector<size_t> ccache_off;               // [L*E] byte offset in ccache
  std::vector<std::vector<int>> coded_cached;   // per layer: local experts cached coded
  int32_t* d_w_index = nullptr;  // [L*E]
  std::vector<cudaEvent_t> slot_ready, slot_free;
  // EP: experts owned by this rank
  std::vector<int> owned;
  // expert parallelism: transport, geometry and exchange buffers
  EpTransport* ept = nullptr;
  bool ep_on = false;
  bool ep_direct = false;  // dispatch/combine kernels store into the peers' mailboxes
  int ep_rows = 0;         // rows per returned block in the combine input (C, or the mailbox stride)
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
    cudaDeviceSynchronize();  // in-flight copies (e.g. a cross-step prefetch) read the host buffers freed below
    async_host.shutdown();  // before the pool and the host buffers it uses go away
    for (auto e : slot_ready) cudaEventDestroy(e);
    for (auto e : slot_free) cudaEventDestroy(e);
    for (auto e : ev) cudaEventDestroy(e);
    for (auto e : draft_ev) cudaEventDestroy(e);
    for (auto e : dec_ev) cudaEventDestroy(e);
    for (auto e : pf_ev) cudaEventDestroy(e);
    for (auto e : join_ev) cudaEventDestroy(e);
    if (route_ev) cudaEventDestroy(route_ev);
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    for (size_t i = 0; i < host_bufs.size(); ++i) pinned_free(host_bufs[i], i < host_numa_bytes.size() ? host_numa_bytes[i] : 0);
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
  void bt_reset();
  // map pages for positions [0, len) of request r
  void bt_ensure(int r, int64_t len);
  void bt_sync(cudaStream_t st);

  // exponent bits of layer l's local expert le on the host (0: raw bf16)
  int code_bits(int l, int le) const { return xcomp ? blk_coded[size_t(host_layer(l)) * E_loc + size_t(le)] : 0; }
  // expand layer l's coded blocks (streamed into cstage) into its pool slot,
  // on the compute stream after slot_ready(l)
  void decode_slot(int l, cudaStream_t st);
  // the expert block of layer l: K4-MoE on the bf16 pool slot, or on the
  // tile-coded blocks (tmode); returns the down-projection splits
  int expert_block(int l, const void* x_perm, int rows, int nexp, const int32_t* offsets, const int32_t* w_index,
                   const void* const* w_code, void* hb, float* y, int splits, int max_splits, cudaStream_t st);

  int host_layer(int l) const { return host_alias > 0 ? l % host_alias : l; }
  int expert_owner(int e) const { return opt.ep_size > 1 ? e % opt.ep_size : 0; }
  bool owns(int e) const { return opt.ep_size <= 1 || expert_owner(e) == opt.ep_rank; }

  void create();

  void fill_prefix(const int32_t* prefix_host, int b);

  // Stream layer l's non-cached owned experts into slot l % slots.
  // owned expert e -> its local index (host block / staging slot position)
  int local(int e) const { return P > 1 ? e / P : e; }

  // Stream layer l's non-cached owned experts into slot l % slots. Host and
  // slot blocks are in local order, so runs of consecutive local experts go
  // out as one copy (a whole layer when nothing is cached: 2.8 GB for 8x7B).
  // active (optional, BATCH_ONE): per local expert, 0 = not routed to -> not streamed
  double enqueue_h2d(int l, cudaEvent_t t0, cudaEvent_t t1, const uint8_t* active = nullptr);

  void snap(const char* name, int layer, const void* src, size_t bytes, cudaStream_t st);

  // Expert-parallel MoE of layer l (ep.cu): dispatch, local shard, combine.
  double moe_ep(int l, int T, cudaStream_t st, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* h2d_ev = nullptr);

  cudaEvent_t tev(int i) const { return ev[8 + size_t(i)]; }

  void verify(const smo_verify_batch& in, smo_verify_output& out, cudaStream_t st);

  // Step start: event 0, then the copy engine starts streaming the first
  // `slots` layers (it only waits for the slot-release edges). Called before
  // the drafter in a decode step so that the first transfers overlap drafting.
  double step_h2d_bytes = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> step_h2d_ev;
  void begin_step(cudaStream_t st, bool prefetch = true);

  // The target verification DAG on device inputs: tokens [b*n], parent
  // [b*n] or null, prefix [b]; results in d_acc / d_bonus / d_keep / target.
  void verify_core(int b, int n, const int32_t* tokens, const int32_t* parent, const int32_t* prefix, int max_prefix,
                   cudaStream_t st);

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
                  int split, cudaStream_t st);

  // x += Wo . attn(RoPE(Wqkv . rmsnorm(x))) for rows organised as `nch`
  // chunks of b*n verify rows; chunk c's row (r, i) sits at position
  // prefix[c*b + r] + i and sees the prefix plus the chain `mask`. K/V rows
  // are appended to kc/vc (the K1 contract of smo_verify_attention).
  void attn_sublayer(const Scratch& sc, const uint16_t* wqkv, const uint16_t* wo, uint16_t* kc, uint16_t* vc, int b,
                     int n, int nch, const int32_t* prefix, const std::vector<int>& max_prefix, const uint64_t* mask,
                     cudaStream_t st, const int32_t* parent = nullptr);

  // attn_sublayer with the CPU placement: q and the appended K/V rows go to
  // pinned host memory, one host job attends over all `nch` chunks (chunk c
  // only sees its prefix + own rows), the output comes back for O-proj.
  // qh/ah: pinned mapped [b*n*nch, n_q, d]; pre_h [nch*b], mask_h [b*n] host.
  void attn_sublayer_cpu(const Scratch& sc, const uint16_t* wqkv, const uint16_t* wo, uint16_t* kc, uint16_t* vc,
                         int b, int n, int nch, const int32_t* prefix, uint16_t* qh, uint16_t* ah,
                         const int32_t* pre_h, const uint64_t* mask_h, HostAttn& job, cudaStream_t st);

  // x += W2 . (silu(W1 . rmsnorm(x)) * W3 . rmsnorm(x))  (dense SwiGLU)
  void ffn_dense(const Scratch& sc, uint16_t* hb, int rows, const uint16_t* w1, const uint16_t* w3,
                 const uint16_t* w2, int inter, cudaStream_t st);

  // final RMSNorm -> LM head with fused argmax partials -> per-row argmax
  void lm_argmax(const float* xr, int rows, int32_t* out, cudaStream_t st);

  // One drafter step for b requests: token tok_in[r] at position pos[r]
  // (its K/V appended there), greedy next token into out_tok[r].
  void draft_forward(int b, const int32_t* tok_in, const int32_t* pos, int max_pos, int32_t* out_tok, cudaStream_t st,
                     int step = -1);

  // ------------------------------------------------------------------ decode
  void decode_begin(const int32_t* root_h, const int32_t* kv_h, int b);

  // draft (k+1 drafter steps) -> verify -> greedy accept -> commit, on device
  void decode_step(int k, const int32_t* drafts_h, cudaStream_t st, const int32_t* parents_h = nullptr);

  // The device part of a decode step (capturable into a CUDA graph): every
  // argument is fixed at enqueue time; bound = host bound of kv_len used for
  // K1 split planning and the drafter's positions.
  void decode_device(int k, bool planted, int bound, cudaStream_t st, bool tree = false);

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
  // Cross-step prefetch (LARGE_BATCH): the experts are the same every step,
  // so once a step has enqueued its last layer's copy, layers [0, slots) of
  // the NEXT step start streaming into their freed slots — the link does not
  // idle through the step's tail (last layer, LM head, accept) and the host
  // round trip of a synchronous API call. SMO_STEP_PREFETCH=0 disables.
  bool step_pf = true;
  bool next_pf = false;
  std::vector<cudaEvent_t> pf_ev;           // [2*slots] copy start / end per prefetched layer
  std::vector<double> pf_bytes, pf_raw;     // [slots]
  void prefetch_next_step();
  void decode_run(int k, int steps, bool graph, cudaStream_t st);

  // durations (s) of the drafter steps of the last decode step; returns count
  int draft_times(double* out, size_t n);
  void ensure_async_host();

  void decode_read(int32_t* committed, int cap, int32_t* n_committed, int32_t* kv_len, int32_t* root);

  // SMO_PREFILL_CHECK=1: host scan for non-finite values after each prefill
  // stage (diagnostics only; synchronises)
  static bool prefill_check_on() {
    const char* e = std::getenv("SMO_PREFILL_CHECK");
    return e && e[0] == '1';
  }
  void check_finite(const char* what, int layer, const void* p, size_t count, bool bf16, cudaStream_t st);

  // ------------------------------------------------------------------ prefill
  // Layer-major prefill: every layer's experts are streamed once for the
  // whole prompt batch; attention runs the prompt as causal chunks of C rows.
  void prefill(const int32_t* tok_h, const int32_t* len_h, int b, int Lmax, int32_t* next_h, cudaStream_t st);

  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending_attn, pending_moe, pending_h2d;

  // micro-batching (Hyperparameters.m, pipeline.hpp:147-206)
  static constexpr int kMaxMb = 8;
  int mb = 1;       // micro-batches of the next steps
  int last_mb = 1;  // of the last step (layer_times layout)
  // timing event k of micro-batch j of layer l (j = 0: the per-layer events tev)
  cudaEvent_t mev(int l, int j, int k) const {
    return j == 0 ? tev(l * 8 + k) : ev[8 + size_t(L) * 8 + (size_t(l) * (kMaxMb - 1) + size_t(j - 1)) * 8 + k];
  }
  void set_micro_batches(int m);

    // Per layer (4 + 6 * last_mb doubles, c_api.h smo_engine_layer_times).
  void layer_times(double* out, size_t n);

  void times(smo_stage_times* t);
};

}  // namespace smo
