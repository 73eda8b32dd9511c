// decode.cu — Engine: dense building blocks shared by the drafter and the
// prefill, the on-device drafter and the decode loop.
#include "engine.cuh"

namespace smo {

void Engine::dense_gemm(const void* xin, int rows, int Kd, int N, const void* w, const void* w_up, int epi, void* out,
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
void Engine::attn_sublayer(const Scratch& sc, const uint16_t* wqkv, const uint16_t* wo, uint16_t* kc, uint16_t* vc, int b,
                   int n, int nch, const int32_t* prefix, const std::vector<int>& max_prefix, const uint64_t* mask,
                   cudaStream_t st, const int32_t* parent) {
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
void Engine::attn_sublayer_cpu(const Scratch& sc, const uint16_t* wqkv, const uint16_t* wo, uint16_t* kc, uint16_t* vc,
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
  copy_from_mapped(sc.attn, ah, size_t(rows) * nq * d * 2, st);  // not behind the expert stream's H2D copies
  dense_gemm(sc.attn, rows, nq * d, h, wo, nullptr, SMO_EPI_F32_ADD, sc.x, sc.split, st);
}

// x += W2 . (silu(W1 . rmsnorm(x)) * W3 . rmsnorm(x))  (dense SwiGLU)
void Engine::ffn_dense(const Scratch& sc, uint16_t* hb, int rows, const uint16_t* w1, const uint16_t* w3,
               const uint16_t* w2, int inter, cudaStream_t st) {
  rmsnorm(sc.x, ones, rows, h, cfg.rms_eps, sc.xn, st);
  dense_gemm(sc.xn, rows, h, inter, w1, w3, SMO_EPI_SWIGLU, hb, 0, st);
  dense_gemm(hb, rows, inter, h, w2, nullptr, SMO_EPI_F32_ADD, sc.x, sc.split, st);
}

// final RMSNorm -> LM head with fused argmax partials -> per-row argmax
void Engine::lm_argmax(const float* xr, int rows, int32_t* out, cudaStream_t st) {
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
// (its K/V appended there), greedy next token into out_tok[r]. With the
// draft split (draft_g = g < b) the projections, FFN and LM head still run
// batched over all b rows on the GPU, but the attention of rows [g, b) runs
// on the host pool over their host-resident drafter K/V (DRAFT_CPU_ATTN,
// started as soon as their q is written, joined before O-proj =
// DRAFT_GPU_FFN) while K1 attends rows [0, g) (DRAFT_GPU_STEP).
void Engine::draft_forward(int b, const int32_t* tok_in, const int32_t* pos, int max_pos, int32_t* out_tok,
                   cudaStream_t st, int step) {
  const Scratch sc{x, xn, qkv, q, attn, attn_ws, attn_ws_bytes, 0};
  embed(tok_in, embed_w, b, h, x, st);
  const std::vector<int> mp{max_pos};
  const int g = draft_g < 0 ? b : std::min(draft_g, b);
  if (g == b) {
    for (auto& dl : dlayers) {
      attn_sublayer(sc, dl.wqkv, dl.wo, dl.kc, dl.vc, b, 1, 1, pos, mp, d_mask1, st);
      ffn_dense(sc, dh, b, dl.w1, dl.w3, dl.w2, dI, st);
    }
    lm_argmax(x, b, out_tok, st);
    return;
  }
  const size_t kv_req = size_t(nkv) * s_max * d;
  for (int li = 0; li < dL; ++li) {
    DLayer& dl = dlayers[size_t(li)];
    rmsnorm(x, ones, b, h, cfg.rms_eps, xn, st);
    dense_gemm(xn, b, h, qkv_w, dl.wqkv, nullptr, SMO_EPI_BF16, qkv, 0, st);
    // CPU part first: its q / K / V rows to host memory, then the host starts
    rope_append(qkv + size_t(g) * qkv_w, pos + g, nullptr, b - g, 1, nq, nkv, d, s_max, cfg.rope_theta, dq_h,
                dkc_h[size_t(li)] + size_t(g) * kv_req, dvc_h[size_t(li)] + size_t(g) * kv_req, st);
    SMO_CUDA_CHECK(cudaMemcpyAsync(dpos_h, pos + g, size_t(b - g) * 4, cudaMemcpyDeviceToDevice, st));
    const uint32_t seq = ++host_seq;
    async_host.push({CpuAttnJob{dq_h, dkc_h[size_t(li)] + size_t(g) * kv_req, dvc_h[size_t(li)] + size_t(g) * kv_req,
                                dmask_h, dpos_h, da_h, b - g, 1, nq, nkv, d, s_max, 1},
                     cpu_pool.get(), seq});
    signal_host_ready(seq, st);
    if (step >= 0) step_seqs[size_t(step)].push_back(seq);
    if (g > 0) {  // GPU part: K1 over its HBM drafter K/V
      rope_append(qkv, pos, nullptr, g, 1, nq, nkv, d, s_max, cfg.rope_theta, q, dl.kc, dl.vc, st);
      smo_attn_args a{};
      a.q = q;
      a.k_cache = dl.kc;
      a.v_cache = dl.vc;
      a.mask = d_mask1;
      a.prefix_len = pos;
      a.out = attn;
      a.b = g;
      a.n = 1;
      a.n_q = nq;
      a.n_kv = nkv;
      a.d = d;
      a.s_max = s_max;
      a.max_prefix = max_pos;
      a.workspace = attn_ws;
      a.workspace_bytes = attn_ws_bytes;
      attention_launch(a, st);
    }
    if (step >= 0 && li == dL - 1) SMO_CUDA_CHECK(cudaEventRecord(join_ev[size_t(step)], st));
    wait_host_flag(seq, st);
    copy_from_mapped(attn + size_t(g) * nq * d, da_h, size_t(b - g) * nq * d * 2, st);
    dense_gemm(attn, b, nq * d, h, dl.wo, nullptr, SMO_EPI_F32_ADD, x, 0, st);
    ffn_dense(sc, dh, b, dl.w1, dl.w3, dl.w2, dI, st);
  }
  lm_argmax(x, b, out_tok, st);
}

// ------------------------------------------------------------------ decode
void Engine::decode_begin(const int32_t* root_h, const int32_t* kv_h, int b) {
  SMO_REQUIRE(b > 0 && b <= maxB, "decode_begin: batch exceeds engine capacity");
  int64_t mx = 0;
  for (int r = 0; r < b; ++r) {
    SMO_REQUIRE(kv_h[r] >= 0 && kv_h[r] < s_max, "decode_begin: kv_len out of range");
    SMO_REQUIRE(root_h[r] >= 0 && root_h[r] < V, "decode_begin: root token out of range");
    mx = std::max<int64_t>(mx, kv_h[r]);
  }
  if (draft_g >= 0 && dec_b > 0) set_draft_split(-1);  // the drafter K/V back in HBM
  draft_g = -1;
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
void Engine::decode_step(int k, const int32_t* drafts_h, cudaStream_t st, const int32_t* parents_h) {
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
void Engine::decode_device(int k, bool planted, int bound, cudaStream_t st, bool tree) {
  const int b = dec_b, n = k + 1;
  last_was_decode = true;
  begin_step(st, !batch_one);  // the first layers' experts stream while the drafter runs
  decode_prep(d_root, planted ? d_drafts : nullptr, b, n, d_dec_tok, st);
  if (tree) {
    SMO_REQUIRE(draft_g < 0 || draft_g >= b, "decode: tree steps need every request's drafter on the GPU");
    last_split = false;
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
  last_split = dL > 0 && draft_g >= 0 && draft_g < b;
  step_seqs.assign(size_t(k) + 1, {});
  for (int t = 0; dL > 0 && t <= k; ++t) {
    SMO_CUDA_CHECK(cudaEventRecord(draft_ev[size_t(t)], st));
    draft_io(d_dec_tok, d_kvlen, t, b, n, d_dtok, d_dpos, st);
    draft_forward(b, d_dtok, d_dpos, bound + t, d_dout, st, t);
    if (!planted && t < k) draft_scatter(d_dout, b, n, t, d_dec_tok, st);
  }
  SMO_CUDA_CHECK(cudaEventRecord(ev[3], st));
  if (last_draft_steps > 0) SMO_CUDA_CHECK(cudaEventRecord(draft_ev[size_t(last_draft_steps)], st));
  verify_core(b, n, d_dec_tok, nullptr, d_kvlen, bound, st);
  decode_commit(d_dec_tok, d_acc, d_bonus, b, n, hist_cap, d_hist, d_hist_n, d_kvlen, d_root, st);
}

void Engine::decode_run(int k, int steps, bool graph, cudaStream_t st) {
  if (!graph) {
    for (int i = 0; i < steps; ++i) decode_step(k, nullptr, st);
    return;
  }
  const int b = dec_b, n = k + 1;
  SMO_REQUIRE(b > 0, "decode: call smo_engine_prefill or smo_engine_decode_begin first");
  SMO_REQUIRE(k >= 0 && n <= maxN, "decode: k + 1 exceeds max_verify");
  SMO_REQUIRE(k == 0 || dL > 0, "decode: k > 0 needs a drafter (draft_layers)");
  SMO_REQUIRE(!batch_one && !attn_cpu && !ep_on && !debug && (draft_g < 0 || draft_g >= b),
              "decode graph: not with BATCH_ONE, CPU attention, expert parallelism, debug snapshots or a draft split");
  SMO_REQUIRE(st != nullptr, "decode graph: needs a non-default stream");
  if (next_pf) {  // a cross-step prefetch from an eager step: let it land (the graph streams its own)
    SMO_CUDA_CHECK(cudaStreamSynchronize(copy));
    next_pf = false;
  }
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
int Engine::draft_times(double* out, size_t n) {
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

void Engine::decode_read(int32_t* committed, int cap, int32_t* n_committed, int32_t* kv_len, int32_t* root) {
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
}  // namespace smo
