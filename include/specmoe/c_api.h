/*
 * specmoe/c_api.h — the C-ABI drop-in boundary of the B200 verify step.
 *
 * Plain pointers and sizes only (no torch / CUDA types in the signatures):
 * streams are passed as `smo_stream` (a cudaStream_t, NULL = legacy default).
 * Every call is asynchronous on the given stream unless stated otherwise and
 * returns an smo_status; the message of the last failure on the calling host
 * thread is available from smo_last_error(). The caller owns every tensor
 * passed in; the library owns only handle-scoped resources (engine, streamer).
 *
 * Each entry cites the reference interface it realises (file:line into
 * /root/reference/proj). The reference has no FFI of its own: its boundary is
 * the header-only C++ API `moeplan::*`; INTEGRATION.md shows the binding a
 * maintainer adds on that side.
 */
#ifndef SPECMOE_C_API_H
#define SPECMOE_C_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SMO_OK = 0,
  SMO_INVALID_ARG = 1, /* std::invalid_argument in the reference (attention.hpp:92-144) */
  SMO_CAPACITY = 2,    /* moeplan::CapacityError (memory.hpp:15) */
  SMO_CUDA = 3,
  SMO_NCCL = 4,
  SMO_UNSUPPORTED = 5
} smo_status;

typedef void* smo_stream;

const char* smo_last_error(void);
const char* smo_version(void);
/* Number of kernels this library has launched since it was loaded. */
uint64_t smo_launch_count(void);
int smo_device_sm_count(int device);

/* ---- procedural synthetic tensors -------------------------
 * dst[i] = bf16(fl(float(2*u24 - 2^24) * fl(scale*2^-24))),
 * u24 = splitmix64(splitmix64(seed ^ tensor_id*0x9e3779b97f4a7c15 ^ (base+i)))>>40
 * — the reference RNG family (specdec.hpp:34-39).                           */
/* Trained-weight-like procedural init with the same variance as the uniform
 * one (std = scale / sqrt(3)): c = sum of the 4 chained splitmix64 draws
 * u_k = x_k >> 40 of the same stream minus 2^25 (Irwin-Hall, near-gaussian),
 * times 8 for one value in 1024 (outliers: x_4 & 1023 == 0), out[i] =
 * bf16(fl(float(c) * fl(scale * 2^-24))) — integer-exact on CPU and GPU
 * (oracle: orc_fill_normal_bf16).                                           */
smo_status smo_fill_normal_bf16(void* dst, uint64_t count, uint64_t seed, uint64_t tensor_id, uint64_t base,
                                float scale, smo_stream stream);
smo_status smo_fill_uniform_bf16(void* dst, uint64_t count, uint64_t seed, uint64_t tensor_id,
                                 uint64_t base, float scale, smo_stream stream);

/* ---- K1: chunked verification attention ------------------------------------
 * Realises moeplan::chunked_attention (attention.hpp:117-156) batched over
 * requests and GQA heads in bf16: prefix keys implicitly visible, the n x n
 * draft block gated by a bit-packed compact mask (attention.hpp:41-58).
 *   q       bf16 [b*n, n_q, d]          (row r*n+i = draft i of request r)
 *   k_cache bf16 [b, n_kv, s_max, d]    (draft rows already at prefix_r + i)
 *   v_cache bf16 [b, n_kv, s_max, d]
 *   mask    u64  [b*n]  bit j of row (r,i) = draft j visible to draft i
 *   prefix  i32  [b]
 *   out     bf16 [b*n, n_q, d]
 * n <= 64, n*(n_q/n_kv) <= 128, d in {64,128}. Errors: SMO_INVALID_ARG with
 * the reference's messages.                                                 */
typedef struct {
  const void* q;
  const void* k_cache;
  const void* v_cache;
  const uint64_t* mask;
  const int32_t* prefix_len;
  void* out;
  int32_t b, n, n_q, n_kv, d, s_max;
  int32_t max_prefix; /* host upper bound of prefix_len (split planning) */
  void* workspace;    /* >= smo_verify_attention_workspace() bytes, zero-filled
                         before its first use (the kernel leaves it so) */
  size_t workspace_bytes;
  /* Paged K/V: when block_table is non-NULL the caches are
   * page pools [num_pages, n_kv, 128, d] and position pos of request r lives
   * in page block_table[r * max_pages + pos / 128] (one page = one 128-key
   * chunk); s_max is then ignored and max_prefix + n <= 128 * max_pages.  */
  const int32_t* block_table;
  int32_t max_pages, num_pages;
} smo_attn_args;
size_t smo_verify_attention_workspace(const smo_attn_args* a);
smo_status smo_verify_attention(const smo_attn_args* a, smo_stream stream);

/* Host verification attention (the CPU placement's kernel, fp32 on bf16
 * inputs): same arguments as smo_verify_attention but every pointer is HOST
 * memory (contiguous K/V only; workspace unused); synchronous, `threads`
 * host threads (0 = all cores).                                           */
smo_status smo_cpu_verify_attention(const smo_attn_args* a, int32_t threads);

/* The reference's desk-scale fp64 operator, one head of one request, host
 * buffers in and out, computed by an fp64 CUDA kernel (synchronous).
 * Same contract as moeplan::chunked_attention (attention.hpp:117); the
 * messages of attention.hpp:96-144 are reported through smo_last_error().
 * Q n x d, K/V (p+n) x d row-major, mask n x n bytes (1 = visible).        */
smo_status smo_chunked_attention_f64(size_t n, size_t p, size_t d, const double* Q,
                                     const double* K, const double* V, size_t mask_n,
                                     const uint8_t* mask, double* out);

/* ---- K2: router top-k -------------------------------------------------------
 * logits[t,e] = fp32 x[t,:].w[e,:] in the fixed order of DESIGN.md §3.3 (so
 * ids are bit-exact vs the oracle); top-k ties to the lower expert id; weights
 * = softmax over the k selected logits. x bf16 [T,h], w bf16 [E,h]; h%256==0,
 * E <= 64, k <= 8. logits_out may be NULL. (n_activate: config.hpp:51)     */
smo_status smo_router_topk(const void* x, const void* w_router, int32_t T, int32_t h, int32_t E,
                           int32_t k, float* logits_out, int32_t* ids, float* weights,
                           smo_stream stream);

/* ---- K3: permute / unpermute-combine ---------------------------------------
 * Stable counting sort of the T*k (token,slot) pairs by expert id:
 * offsets i32 [E+1], perm i32 [T*k] (source pair at each sorted position),
 * pos i32 [T*k] (sorted position of each pair), x_perm bf16 [T*k, h] rows
 * gathered from x bf16 [T,h] (x/x_perm may be NULL to skip the gather).    */
smo_status smo_permute(const int32_t* ids, int32_t T, int32_t k, int32_t E, const void* x, int32_t h,
                       int32_t* offsets, int32_t* perm, int32_t* pos, void* x_perm,
                       smo_stream stream);
/* residual[t,:] += sum_{j<k} weights[t,j] * y_perm[pos[t*k+j], :]  (fp32,
 * j order fixed, no atomics). y_perm fp32 [T*k, h].                         */
smo_status smo_unpermute_combine(const float* y_perm, const int32_t* pos, const float* weights,
                                 int32_t T, int32_t k, int32_t h, float* residual, smo_stream stream);
/* Same with the down projection in K slices y_perm[s] (split_stride
 * elements apart, s < splits), summed in slice order per (token, slot), as
 * produced by smo_moe_experts.                                             */
smo_status smo_unpermute_combine_split(const float* y_perm, int32_t splits, uint64_t split_stride,
                                       const int32_t* pos, const float* weights, int32_t T, int32_t k, int32_t h,
                                       float* residual, smo_stream stream);

/* ---- K4: tcgen05 GEMMs ------------------------------------------------------
 * out[t, n] = sum_c x[t,c] * W_g[n,c] for the rows t of group g
 * (row_offsets[g] <= t < row_offsets[g+1]); W_g = pool block w_index[g].
 * SWIGLU: out = bf16(silu(x W_g^T) * (x U_g^T)) with U from w_up.
 * ARGMAX: no output matrix; (max, index) partials per 128-row weight tile
 * into argmax_val/argmax_idx [rows, N/128] (the LM-head epilogue of K6).
 * Weights are row-major [N, K] per block (nn.Linear layout) — the MMA's
 * 128-row A operand ("swap-AB": tokens are the small N side).              */
enum {
  SMO_EPI_BF16 = 0,
  SMO_EPI_F32 = 1,
  SMO_EPI_F32_ADD = 2,
  SMO_EPI_SWIGLU = 3,
  SMO_EPI_ARGMAX = 4
};
typedef struct {
  const void* x;              /* bf16 [rows, K] */
  int32_t rows, K, N, groups;
  const int32_t* row_offsets; /* device [groups+1]; NULL: one group = all rows */
  int32_t max_rows_per_group; /* host bound (grid sizing); <= rows */
  const void* w;              /* bf16 pool, block b at w + b*w_block_stride */
  const void* w_up;           /* SWIGLU second weight (same pool layout) */
  uint64_t w_block_stride;    /* bytes between pool blocks */
  int32_t w_pool_blocks;
  const int32_t* w_index;     /* device [groups] pool block per group; NULL = g */
  int32_t epilogue;
  void* out;                  /* bf16 or f32 [rows, ldo] */
  int64_t ldo;
  float* argmax_val;          /* [rows, N/128] */
  int32_t* argmax_idx;
  int32_t split_k;            /* 0 = auto (dense GEMMs split K to cover the SMs), 1 = off, S */
  void* workspace;            /* >= smo_gemm_workspace() bytes (fp32 split-K partials) */
  size_t workspace_bytes;
} smo_gemm_args;
/* Split-K partials are reduced in fixed order (deterministic) and fused with
 * the epilogue. Returns the workspace the call needs (0: none).            */
size_t smo_gemm_workspace(const smo_gemm_args* a);
smo_status smo_gemm(const smo_gemm_args* a, smo_stream stream);

/* ---- K4-MoE: the whole expert block of one layer in ONE persistent kernel
 * (grouped SwiGLU gate/up, then the down projection; moe_tc.cu):
 *   h_out bf16 [rows, h_i] = silu(x W1_e^T) * (x W3_e^T)   for the rows of e
 *   sum_s y[s] f32 [rows, h] = h_out W2_e^T, the K dimension cut into `splits`
 *            slices (1, 2 or 4; 0 = chosen by a waves model, written to
 *            *splits_used); y holds [splits][rows][h] (room for 4 when 0);
 *            sum them with smo_unpermute_combine_split.
 * x_perm bf16 [rows, h] grouped by offsets [E+1] (device); expert e uses pool
 * block w_index[e] = [W1 | W3 | W2] (nn.Linear layouts), blocks
 * w_block_stride bytes apart. scratch: >= 65 int32 (device), zero before the
 * first call (every call leaves it zero). E <= 64,
 * h and h_i multiples of 128. The roofline.hpp:56-64 expert cost.          */
smo_status smo_moe_experts(const void* x_perm, int32_t rows, int32_t h, int32_t h_i, int32_t E,
                           const int32_t* offsets, const void* w_pool, uint64_t w_block_stride,
                           int32_t w_pool_blocks, const int32_t* w_index, void* h_out, float* y, int32_t splits,
                           int32_t* splits_used, int32_t* scratch, smo_stream stream);

/* ---- K5 codec: lossless expert-weight packing for the host link (xfer.cu)
 * bf16 values in segments of 1024: sign + mantissa verbatim (1 byte), the
 * exponent as a `bits`-bit code (3 or 4) against a per-segment base with up
 * to 32 escaped exponents per segment — 1456 (3 bits: 11.4 bits/value) or
 * 1584 (4 bits: 12.4 bits/value) bytes per 1024 values. count % 1024 == 0.
 * encode sets *overflow (device int) to 1 when a segment needs more than 32
 * escapes (retry with 4 bits or keep the block raw). Decode is the exact
 * inverse (bit-identical bf16).
 * bits = 1: the variable-length UNARY exponent code (xfer.cu header: j = E - e
 * ones then a zero, per-segment table; ~10.2 bits/value on uniform-init
 * weights). smo_expert_code_bytes(count, 1) is its capacity (worst case);
 * encode is synchronous on `stream` for bits = 1 and never overflows;
 * smo_expert_coded_size gives the bytes actually used (reads the device
 * code's table; 3 / 4 bits: the fixed size).                               */
size_t smo_expert_code_bytes(uint64_t count, int32_t bits);
uint64_t smo_expert_coded_size(const void* code, uint64_t count, int32_t bits);
smo_status smo_expert_encode(const void* src, uint64_t count, int32_t bits, void* dst, int32_t* overflow,
                             smo_stream stream);
smo_status smo_expert_decode(const void* src, uint64_t count, int32_t bits, void* dst, smo_stream stream);

/* ---- K5 tile code T2 (tcode.cuh; format restated in tests/tcode_ref.py) ----
 * The link code the fused expert kernel decodes in shared memory: one expert
 * block [W1 | W3 | W2] (bf16, device; W1/W3 [h_i, h], W2 [h, h_i]) in tiles of
 * 128 x 64 (= the kernel's k-block), 2-bit level-1 exponent codes + a ranked
 * escape stream, sign/mantissa verbatim; lossless, ~10.4 bits/weight on
 * uniform-init and ~10.9 on gaussian-like weights. h, h_i multiples of 128.
 * smo_tcode_max_bytes is the capacity (every segment raw); encode is
 * synchronous on `stream` and returns the bytes used; code blocks must be
 * 16-byte aligned.                                                          */
size_t smo_tcode_max_bytes(int32_t h, int32_t h_i);
smo_status smo_tcode_encode(const void* src, int32_t h, int32_t h_i, void* dst, uint64_t* bytes, smo_stream stream);
smo_status smo_tcode_decode(const void* src, int32_t h, int32_t h_i, void* dst, smo_stream stream);
/* K4-MoE on T2-coded experts: as smo_moe_experts, but expert e's weights are
 * the T2 block at w_code[e] (w_code: DEVICE array of E pointers), decoded
 * tile by tile into shared memory by the kernel itself (no bf16 copy in
 * HBM). Bit-identical to smo_moe_experts on the decoded weights.            */
smo_status smo_moe_experts_coded(const void* x_perm, int32_t rows, int32_t h, int32_t h_i, int32_t E,
                                 const int32_t* offsets, const void* const* w_code, void* h_out, float* y,
                                 int32_t splits, int32_t* splits_used, int32_t* scratch, smo_stream stream);
/* ---- K5 tile code T3 (tcode.cuh; format restated in tests/tcode3_ref.py) ----
 * The same tiles with every exponent a fixed 3-bit code (escapes, ~1/128 of
 * uniform-init values, as a per-segment (position, exponent) list): ~11.2
 * bits/weight, a decoder without per-lane loops — the code for a
 * device-bound step (every block resident in the coded hot cache). Capacity
 * smo_tcode_max_bytes; the expert kernel on T3 blocks is
 * smo_moe_experts_coded3 (same contract as smo_moe_experts_coded).         */
smo_status smo_tcode3_encode(const void* src, int32_t h, int32_t h_i, void* dst, uint64_t* bytes, smo_stream stream);
smo_status smo_tcode3_decode(const void* src, int32_t h, int32_t h_i, void* dst, smo_stream stream);
smo_status smo_moe_experts_coded3(const void* x_perm, int32_t rows, int32_t h, int32_t h_i, int32_t E,
                                  const int32_t* offsets, const void* const* w_code, void* h_out, float* y,
                                  int32_t splits, int32_t* splits_used, int32_t* scratch, smo_stream stream);

/* ---- K5 expert streamer as a standalone handle (streamer.cu) --------------
 * The reference's H2D_EXPERTS(l) stage and the GPU_MOE(l) dependency on it
 * (pipeline.hpp:147-206; transfer bytes roofline.hpp:56-77; LARGE_BATCH vs
 * BATCH_ONE roofline.hpp:155-162 -> `active`). Expert blocks (bf16, block_bytes
 * each, a multiple of 2048) live in caller-owned PINNED host memory, raw or in
 * a K5 code (host_codes 1 = unary, 3 / 4 = window codes; host_bytes = coded
 * size). Layer l streams into HBM slot l % hbm_slots on the streamer's own
 * copy-engine stream; the first cache_bytes / block_bytes blocks in (layer,
 * expert) order are copied to HBM once at create (the hot-expert cache,
 * MemoryPolicy.expert_cache_bytes) and never streamed. Per layer:
 *   enqueue_layer (async; waits for the slot's previous release)
 *   wait_layer(stream)   -- stream waits for the copies; coded blocks are
 *                           expanded into the slot on `stream`
 *   expert_ptr           -- device block [W1|W3|W2] of (layer, expert)
 *   release_layer(stream)-- the slot may be refilled once `stream` gets here
 * active (nullable, [n_experts]): 0 = not routed to, not streamed.          */
typedef struct smo_streamer smo_streamer;
typedef struct {
  int32_t n_layers, n_experts;
  uint64_t block_bytes;            /* bf16 bytes of one expert block in HBM */
  const void* const* host_blocks;  /* [n_layers * n_experts] pinned host pointers */
  const uint64_t* host_bytes;      /* nullable: link bytes of each coded block */
  const int32_t* host_codes;       /* nullable: 0 raw, 1 unary, 3 / 4 bits per block */
  int32_t hbm_slots;               /* >= 2 */
  int64_t cache_bytes;             /* hot-expert cache in HBM */
  int32_t device;
} smo_streamer_args;
smo_status smo_streamer_create(const smo_streamer_args* args, smo_streamer** out);
smo_status smo_streamer_destroy(smo_streamer* s);
smo_status smo_streamer_enqueue_layer(smo_streamer* s, int32_t layer, const uint8_t* active);
smo_status smo_streamer_expert_ready_event(smo_streamer* s, int32_t layer, void** cuda_event);
smo_status smo_streamer_wait_layer(smo_streamer* s, int32_t layer, smo_stream stream);
smo_status smo_streamer_expert_ptr(smo_streamer* s, int32_t layer, int32_t expert, const void** out);
smo_status smo_streamer_release_layer(smo_streamer* s, int32_t layer, smo_stream stream);

/* ---- support ops of the verify layer (standard Mixtral block, not in the
 *      reference: SURVEY.md §2.3 "support")                                 */
/* y bf16 [T,h] = x f32 [T,h] * rsqrt(mean(x^2)+eps) * gain bf16 [h] */
smo_status smo_rmsnorm(const float* x, const void* gain, int32_t T, int32_t h, float eps, void* y,
                       smo_stream stream);
/* x f32 [T,h] = embed bf16 [V,h] rows at tokens [T] */
smo_status smo_embed(const int32_t* tokens, const void* embed, int32_t T, int32_t h, float* x,
                     smo_stream stream);
/* qkv bf16 [b*n, (n_q+2 n_kv) d]: RoPE (rotate-half, theta) on q and k at
 * position prefix[r] + depth(r,i) (depth = i for chains, from parent[]
 * otherwise), q written to q_out [b*n, n_q, d]; k/v appended to the caches
 * at row prefix[r] + i.                                                     */
smo_status smo_rope_append(const void* qkv, const int32_t* prefix_len, const int32_t* parent,
                           int32_t b, int32_t n, int32_t n_q, int32_t n_kv, int32_t d, int32_t s_max,
                           float theta, void* q_out, void* k_cache, void* v_cache, smo_stream stream);
/* Synthetic prefix KV: cache[r,h,pos,c] for pos < prefix[r] =
 * uniform(seed, tensor_id, idx = ((r*n_kv+h) << 32) | (pos*d + c)).       */
smo_status smo_fill_kv_prefix(void* cache, const int32_t* prefix_len, int32_t b, int32_t n_kv,
                              int32_t d, int32_t s_max, uint64_t seed, uint64_t tensor_id,
                              smo_stream stream);

/* ---- K6: argmax + greedy accept + KV rollback ------------------------------
 * Greedy verification restating specdec.hpp:65-76 with the Bernoulli draw
 * replaced by argmax(logits of the parent row) == token. Chain when parent
 * is NULL; tree otherwise (parent[r*n+i] < i, -1 for the root row 0): the
 * longest matching root path, ties to the lower node id.
 * acc_len[b] accepted drafts (committed = acc_len + 1, config.hpp:69-70),
 * bonus[b] = argmax at the accepted tip, keep[b*n] accepted rows in path
 * order (root first, -1 padded).                                           */
smo_status smo_argmax_reduce(const float* part_val, const int32_t* part_idx, int32_t rows,
                             int32_t parts, int32_t* target, smo_stream stream);
smo_status smo_argmax_rows(const float* logits, int32_t rows, int32_t V, int32_t* target,
                           smo_stream stream);
smo_status smo_greedy_accept(const int32_t* tokens, const int32_t* target, const int32_t* parent,
                             int32_t b, int32_t n, int32_t* acc_len, int32_t* bonus, int32_t* keep,
                             smo_stream stream);
/* Tree rollback: move the accepted rows keep[r, 0..acc] of every layer's
 * K/V to prefix[r] + 0..acc (chains are already in place) and set
 * kv_len[r] = prefix[r] + acc_len[r] + 1. caches: n_layers pointers.       */
smo_status smo_kv_rollback(void* const* k_caches, void* const* v_caches, int32_t n_layers,
                           const int32_t* prefix_len, const int32_t* acc_len, const int32_t* keep,
                           int32_t b, int32_t n, int32_t n_kv, int32_t d, int32_t s_max,
                           int32_t* kv_len, smo_stream stream);

/* ---- K5 + engine: the measured verify step ---------------------------------
 * The engine owns the model (procedural weights; experts in pinned host
 * DRAM), the expert streamer (copy-engine stream, double-buffered HBM slots,
 * hot-expert cache) and the KV cache. One verify() = the reference's target
 * DAG (pipeline.hpp:147-206) realised on streams + events.                 */
typedef struct {
  int32_t hidden;      /* h        (ModelSpec.h, config.hpp:48) */
  int32_t inter;       /* h_i      (ModelSpec.h_i) */
  int32_t n_expert;    /* E        (ModelSpec.n_expert) */
  int32_t top_k;       /* n_activate */
  int32_t n_layers;
  int32_t n_q_heads;
  int32_t n_kv_heads;  /* h / g */
  int32_t head_dim;
  int32_t vocab;
  float rope_theta;
  float rms_eps;
  uint64_t seed;
  float lm_scale;      /* multiplier on the LM-head init scale (margin screening) */
  float router_scale;  /* multiplier on the router init scale */
  int32_t shared_inter; /* always-on shared expert width (0: none; DeepSeek/Qwen-style,
                           resident in HBM, SwiGLU over every token) */
  int32_t draft_layers; /* drafter depth, DraftModelSpec.n_layers (config.hpp:40-45); 0: no drafter.
                           Dense decoder layers with the target's attention shape, sharing
                           its embedding and LM head (EAGLE convention), resident in HBM */
  int32_t draft_inter;  /* drafter SwiGLU width: DraftModelSpec.ffn_ops_per_token = 6*h*draft_inter */
  int32_t expert_init;  /* routed-expert weight distribution: SMO_INIT_UNIFORM (default) or
                           SMO_INIT_GAUSSIAN (trained-like, smo_fill_normal_bf16); same variance */
} smo_model_config;
enum { SMO_INIT_UNIFORM = 0, SMO_INIT_GAUSSIAN = 1 };

enum { SMO_ENGINE_DEBUG = 1 /* keep per-layer intermediates for parity tests */ };

typedef struct {
  int32_t max_batch;          /* b */
  int32_t max_verify;         /* n = k+1 rows per request (chain or tree) */
  int32_t max_seq;            /* KV capacity per request (s_max) */
  int32_t hbm_slots;          /* expert-layer staging slots, >= 2 */
  int64_t expert_cache_bytes; /* hot-expert HBM cache (MemoryPolicy.expert_cache_bytes) */
  int32_t host_alias_layers;  /* 0: one pinned expert buffer per layer; A: layer l uses l % A */
  int32_t device;             /* smo_engine_create makes it current on the calling thread; drive the
                                 engine from one host thread with that device current */
  int32_t flags;
  int32_t ep_rank, ep_size;   /* expert parallelism: this rank owns experts e % ep_size == ep_rank */
  void* nccl_comm;            /* smo_ep_group* (NCCL or loopback) when ep_size > 1 */
  int32_t kv_pages;           /* K/V layout: 0 = contiguous [b][n_kv][max_seq][d];
                                 > 0 = paged pool of that many 128-token pages per layer, one block
                                 table shared by all layers, pages assigned as requests grow;
                                 -1 = paged, pool = max_batch * ceil(max_seq / 128) */
  int32_t attn_cpu;           /* AttentionPlacement::CPU (config.hpp:110): the
                                 target K/V live in pinned host DRAM (the GPU appends rows through
                                 mapped memory) and verification attention runs on a host thread
                                 pool; 0 = GPU_RESIDENT (K1 on HBM). Contiguous K/V only. */
  int32_t moe_batching;       /* ExecStrategy::moe_batching (config.hpp:110-116, optimizer.hpp:81-96):
                                 0 = LARGE_BATCH: stream whole layers ahead (layer l+S during l);
                                 1 = BATCH_ONE: after layer l's router, stream only the experts its
                                 tokens selected (host waits for the routing, then issues the copies).
                                 Prefill always streams whole layers. With expert parallelism each
                                 owner streams its local experts that received rows, once the
                                 dispatch exchange has landed (no link-gap prefetch). */
  int32_t compress_experts;   /* 1: experts sit in pinned host DRAM in the smallest lossless code of
                                 smo_expert_encode that holds the block (unary exponents: 1.56x fewer
                                 bytes on uniform-init weights; 3-bit window 1.41x; 4-bit 1.29x;
                                 else raw; env SMO_CODEC=fixed skips unary) and cross the link
                                 coded; the compute stream expands each layer's blocks into its HBM
                                 slot before the expert kernel. 2 (or env SMO_CODEC=tile): the T2
                                 tile code (smo_tcode_encode) for every block, streamed and hot-cached
                                 in that code and decoded by the expert kernel itself in shared memory
                                 (smo_moe_experts_coded): no expansion launch, no bf16 expert in HBM.
                                 3 (or SMO_CODEC=tile3): the T3 tile code (smo_tcode3_encode). With 1
                                 and no SMO_CODEC the engine probes the first block: T3 when the hot
                                 cache holds every block (device-bound step), else T2 when smaller
                                 than the unary code, else unary. */
  int32_t micro_batches;      /* Hyperparameters.m (config.hpp:118-125): the batch runs as m micro-
                                 batches of ~b/m requests, issued stage-major per layer like
                                 build_target_dag (pipeline.hpp:147-206): GPU_OTHER1 of every
                                 micro-batch, then their attention, GPU_OTHER2, GPU_MOE (all waiting
                                 on the layer's one expert transfer). With the CPU placement the host
                                 attends micro-batch j while the GPU runs j+1's stages. 0/1 = one;
                                 at most 8; LARGE_BATCH without expert parallelism. */
  int32_t draft_cpu_kv;       /* 1: also keep a pinned host copy slot for every request's drafter K/V,
                                 so smo_engine_set_draft_split can move requests' drafter attention
                                 to the host thread pool (the paper's draft CPU part, build_draft_dag
                                 pipeline.hpp:217-253; split from dynamic_split_ratio memory.hpp:93-106).
                                 Contiguous K/V only (kv_pages = 0). */
} smo_engine_options;

/* ---- expert parallelism ----------------------------------
 * Rank r of P owns experts e % P == r and streams only those; per layer the
 * engine dispatches token rows to the owners and combines the results
 * (fixed-capacity block all-to-all, owner-major order; results bit-identical
 * to one GPU). Every rank must use identical engine options. The transport is
 * an smo_ep_group: NCCL (one process per GPU; rank 0 makes the unique id and
 * the caller broadcasts it) or an in-process loopback group (P engines on one
 * device, one host thread per engine calling smo_engine_verify).          */
typedef struct smo_ep_group smo_ep_group;
smo_status smo_nccl_unique_id(uint8_t* id128);
smo_status smo_ep_nccl_create(const uint8_t* id128, int32_t nranks, int32_t rank, smo_ep_group** out);
smo_status smo_ep_loopback_create(int32_t ep_size, smo_ep_group** out);
smo_status smo_ep_group_destroy(smo_ep_group* g);
/* Peer-memory transport (CUDA IPC; NVLink between GPUs, or several processes
 * on one GPU): each rank owns a mailbox [2][nranks][slot_bytes] peers write
 * into directly, plus a flag area (per-peer round counters written with
 * release stores and polled with acquire loads by one-thread kernels: the
 * exchange is device-side only and CUDA-graph capturable). create returns
 * this rank's handle blob (smo_ep_ipc_handle_bytes() bytes); the caller
 * all-gathers the blobs (rank order) and connects with a host barrier
 * callback over the same ranks (called once, at the end of connect).
 * slot_bytes >= the largest exchange block: max(T*k*h*2 + 16 + 4*E/P,
 * T*k*h*4) for the engine's T = max_batch * max_verify.                    */
typedef void (*smo_barrier_fn)(void* ctx);
/* Standalone dispatch / combine around a caller-run expert shard (the engine
 * runs the same kernels internally). Rank `rank` of the group owns experts
 * e % P == rank (local index e / P). dispatch: x bf16 [T,h], ids int32 [T,k]
 * (global expert ids, router output) -> xl bf16 [P*C,h] rows grouped by local
 * expert (offsets_l [E/P+1]; src-major inside an expert), back int32 [P*C]
 * (where each row returns), pos_ep int32 [T*k] (for combine). combine: the
 * shard's fp32 outputs yl [P*C,h] travel back and x fp32 [T,h] +=
 * sum_j weights[t,j] * y(t,j) in slot order (the single-GPU combine). C =
 * rows per destination, the same on every rank, >= T*k. workspace: device,
 * smo_ep_workspace(P,T,k,h,E,C) bytes, shared by both calls. All ranks call
 * collectively (same order); async on `stream` (host-synchronising for the
 * loopback transport's barriers). */
size_t smo_ep_workspace(int32_t P, int32_t T, int32_t k, int32_t h, int32_t E, int32_t C);
smo_status smo_ep_dispatch(smo_ep_group* g, int32_t rank, const void* x, const int32_t* ids, int32_t T, int32_t k,
                           int32_t h, int32_t E, int32_t C, void* xl, int32_t* offsets_l, int32_t* back,
                           int32_t* pos_ep, void* workspace, smo_stream stream);
smo_status smo_ep_combine(smo_ep_group* g, int32_t rank, const float* yl, const int32_t* back,
                          const int32_t* offsets_l, const int32_t* pos_ep, const float* weights, int32_t T,
                          int32_t k, int32_t h, int32_t E, int32_t C, float* x, void* workspace, smo_stream stream);
size_t smo_ep_ipc_handle_bytes(void);
smo_status smo_ep_ipc_create(int32_t nranks, int32_t rank, uint64_t slot_bytes, smo_ep_group** out,
                             uint8_t* handles);
smo_status smo_ep_ipc_connect(smo_ep_group* g, const uint8_t* all_handles, smo_barrier_fn barrier, void* ctx);

typedef struct smo_engine smo_engine;

smo_status smo_engine_create(const smo_model_config* cfg, const smo_engine_options* opt,
                             smo_engine** out);
/* Change the micro-batch count for subsequent verify / decode steps (the m
 * that optimize() returns, optimizer.hpp:130-175). Same limits as above.     */
smo_status smo_engine_set_micro_batches(smo_engine* e, int32_t m);
smo_status smo_engine_destroy(smo_engine* e);
/* Fill the synthetic prefix KV of every layer for requests 0..b-1. */
smo_status smo_engine_fill_prefix(smo_engine* e, const int32_t* prefix_len_host, int32_t b);

typedef struct {
  int32_t b, n;
  const int32_t* tokens;     /* [b*n], row 0 of each request = root token */
  const int32_t* parent;     /* [b*n] or NULL (chain) */
  const int32_t* prefix_len; /* [b] */
  int32_t on_device;         /* 0: host pointers (copied in on the stream) */
} smo_verify_batch;

typedef struct {
  int32_t* acc_len; /* [b] */
  int32_t* bonus;   /* [b] */
  int32_t* keep;    /* [b*n] or NULL */
  int32_t* target;  /* [b*n] argmax per row, or NULL */
  int32_t on_device;
} smo_verify_output;

smo_status smo_engine_verify(smo_engine* e, const smo_verify_batch* in, smo_verify_output* out,
                             smo_stream stream);

/* Measured stage durations of the last verify (seconds, CUDA events), in the
 * reference's IterationBreakdown vocabulary (report.hpp:27-37).             */
typedef struct {
  double target_total;
  double attention;    /* K1 (the reference's CPU_ATTN slot) */
  double gpu_moe;      /* K4 + combine */
  double h2d_transfer; /* K5 copy-engine busy time */
  double others;       /* norms, QKV/O GEMMs, router, permute, LM head, accept */
  double h2d_bytes;    /* bytes streamed */
  double launches;     /* kernels launched */
  double draft;        /* drafter time of the last decode step (DRAFT_GPU_STEP total) */
  double h2d_raw_bytes; /* bf16 bytes the streamed blocks carry (= h2d_bytes unless coded) */
  double codec;        /* device time expanding coded expert blocks (compress_experts) */
  double codec_bytes;  /* their algorithmic bytes: code read + bf16 written (streamed + coded hot cache) */
  double link_code;    /* the engine's expert link code: 0 raw bf16, 1 unary / window codes expanded in HBM,
                          2 T2 tile code decoded inside the expert kernel */
  double host_numa;    /* NUMA node the pinned expert blocks were bound to (the GPU's own; -1: default
                          placement, e.g. a single-node host or SMO_HOST_NUMA=-1) */
  double code_bits;    /* mean bits per weight of the engine's expert blocks as stored in host memory
                          and the coded hot cache (16: raw bf16) — defined even when no block crossed
                          the link in the last step (everything cached) */
} smo_stage_times;
smo_status smo_engine_last_times(smo_engine* e, smo_stage_times* t);
/* Measured per-layer timeline of the last verify step with m micro-batches
 * (smo_engine_last_micro_batches), 4 + 6m doubles per layer, seconds from
 * the step start: H2D_EXPERTS start, end, the bytes streamed for the layer
 * (hot-cached experts excluded), their bf16 size; then per micro-batch j:
 * GPU_OTHER1 start, attention start, attention end (CPU placement: when the
 * GPU saw the host job finish), pre-MoE (GPU_OTHER2 end), GPU_MOE start
 * (after the slot wait), GPU_MOE end. n >= (4 + 6m) * L.                    */
smo_status smo_engine_layer_times(smo_engine* e, double* out, size_t n);
smo_status smo_engine_last_micro_batches(smo_engine* e, int32_t* m);

/* ---- prefill + decode loop ------------------------------
 * The KV lifecycle around the verify step, all on the engine's device state:
 *  smo_engine_prefill: runs the prompts through the target (and drafter) and
 *    writes their real K/V at positions 0..len_r-1. Layer-major: each layer's
 *    experts are streamed ONCE for the whole prompt batch; attention runs the
 *    prompt as causal verify-shaped chunks of C = min(64, 128*n_kv/n_q) rows
 *    (K1 with a chain mask and prefix = c*C). tokens: host [b, max_len]
 *    (row r valid up to len[r], 1 <= len[r] <= max_len); next_token: host [b]
 *    greedy token after each prompt. Sets the decode state: kv_len = len,
 *    root = next_token, empty history. Not available with expert parallelism.
 *  smo_engine_decode_begin: sets the decode state from host arrays instead
 *    (e.g. after smo_engine_fill_prefix).
 *  smo_engine_decode_step: one iteration = draft (k+1 drafter steps: chain,
 *    greedy; the last one only appends d_k's draft K/V) -> verify (n = k+1,
 *    prefix = kv_len) -> greedy accept -> commit (kv_len += acc+1, root =
 *    bonus, accepted drafts + bonus appended to the history). drafts: NULL
 *    (drafter proposes) or host [b*k] planted drafts (the drafter still runs
 *    teacher-forced to keep its K/V in step). k = 0 is plain decoding.
 *  smo_engine_decode_read: history [b, cap] (-1 padded), its lengths, kv_len
 *    and the next root, to host (synchronous).                             */
smo_status smo_engine_prefill(smo_engine* e, const int32_t* tokens, const int32_t* len, int32_t b,
                              int32_t max_len, int32_t* next_token, smo_stream stream);
smo_status smo_engine_decode_begin(smo_engine* e, const int32_t* root, const int32_t* kv_len, int32_t b);
smo_status smo_engine_decode_step(smo_engine* e, int32_t k, const int32_t* drafts, smo_stream stream);
/* One iteration with a planted draft TREE of n nodes per request: node 0 is
 * the root (the current root token), tokens host [b*(n-1)] for nodes 1..n-1,
 * parents host [b*n] (parents[r*n] = -1, 0 <= parents[r*n+i] < i). The
 * drafter runs over all nodes at once (tree positions and mask), verify uses
 * the ancestor-or-self mask, greedy accept takes the longest matching root
 * path (children in id order), and that path's K/V rows of every target and
 * drafter layer are compacted to kv_len + j (smo_kv_rollback) before the
 * commit — the tree K/V lifecycle of SURVEY.md §8 f2.                      */
smo_status smo_engine_decode_step_tree(smo_engine* e, int32_t n, const int32_t* tokens, const int32_t* parents,
                                       smo_stream stream);
/* `steps` decode iterations with k drafts from the drafter (asynchronous).
 * use_graph: the device part of an iteration is captured once into a CUDA
 * graph and replayed (one launch per iteration; needs a non-default stream,
 * GPU attention, LARGE_BATCH streaming, no expert parallelism). K/V pages
 * for the whole run are mapped before it starts.                           */
smo_status smo_engine_decode_run(smo_engine* e, int32_t k, int32_t steps, int32_t use_graph, smo_stream stream);
/* Measured duration (s) of each drafter step of the last decode step
 * (DRAFT_GPU_STEP events, pipeline.hpp:208-253); *steps = k+1 (0: no drafter). */
smo_status smo_engine_draft_times(smo_engine* e, double* out, size_t n, int32_t* steps);
/* Drafter GPU-part / CPU-part split (engine created with draft_cpu_kv):
 * requests [0, gpu_requests) keep their drafter K/V in HBM and attend with K1
 * (DRAFT_GPU_STEP); requests [gpu_requests, b) keep it in pinned host memory
 * and attend on the host thread pool (DRAFT_CPU_ATTN), whose output feeds the
 * drafter's GPU projections / FFN (DRAFT_GPU_FFN) — the two parts of a step
 * run concurrently. Moves the affected requests' drafter K/V rows (call after
 * prefill / decode_begin, between steps). -1: every request on the GPU. Chain
 * decode steps only (no tree steps or decode graphs while split).          */
smo_status smo_engine_set_draft_split(smo_engine* e, int32_t gpu_requests);
/* Per drafter step of the last decode step with a split: out[3t..3t+2] =
 * (GPU part up to the host join, host attention wall time summed over the
 * drafter layers, GPU work after the join) in seconds; *steps = k+1, or 0
 * when the last step ran without a split.                                   */
smo_status smo_engine_draft_split_times(smo_engine* e, double* out, size_t n, int32_t* steps);
smo_status smo_engine_decode_read(smo_engine* e, int32_t* committed, int32_t cap, int32_t* n_committed,
                                  int32_t* kv_len, int32_t* root);

/* Debug intermediates of the last verify (engine created with SMO_ENGINE_DEBUG).
 * name: "x_in" f32 [T,h] layer input, "xn1" bf16, "q" bf16 [T,n_q,d],
 * "attn" bf16 [T,n_q,d], "xn2" bf16 [T,h], "logits_r" f32 [T,E],
 * "ids" i32 [T,k], "weights" f32 [T,k], "offsets" i32 [E+1], "pos" i32 [T*k],
 * "x_out" f32 [T,h]; layer -1 with "xf" bf16 [T,h], "logits" f32 [T,V].
 * Copies into host dst (synchronous).                                      */
smo_status smo_engine_debug_tensor(smo_engine* e, const char* name, int32_t layer, void* dst,
                                   size_t bytes);
/* Device pointer of a weight tensor ("embed","lm_head","final_norm" with
 * layer -1; "wqkv","wo","attn_norm","ffn_norm","router" per layer) or of an
 * expert's pinned host block ("expert_host", layer, expert): [W1|W3|W2].  */
smo_status smo_engine_tensor_ptr(smo_engine* e, const char* name, int32_t layer, int32_t expert,
                                 void** ptr, size_t* bytes);

#ifdef __cplusplus
}
#endif
#endif /* SPECMOE_C_API_H */
