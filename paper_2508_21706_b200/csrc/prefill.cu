// prefill.cu — Engine: layer-major chunked prefill: each
// layer's experts cross the link once for the whole prompt batch.
#include "engine.cuh"

namespace smo {

void Engine::check_finite(const char* what, int layer, const void* p, size_t count, bool bf16, cudaStream_t st) {
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
void Engine::prefill(const int32_t* tok_h, const int32_t* len_h, int b, int Lmax, int32_t* next_h, cudaStream_t st) {
  SMO_REQUIRE(!ep_on, "prefill: not available with expert parallelism");
  SMO_REQUIRE(b > 0 && b <= maxB && Lmax > 0, "prefill: bad batch");
  SMO_REQUIRE(tok_h && len_h && next_h, "prefill: null argument");
  const int g = nq / nkv;
  const int C = std::max(1, std::min(64, 128 / g));
  const int nch = (Lmax + C - 1) / C;
  SMO_REQUIRE(int64_t(nch) * C + maxN <= s_max, "prefill: prompt exceeds max_seq");
  for (int r = 0; r < b; ++r) SMO_REQUIRE(len_h[r] >= 1 && len_h[r] <= Lmax, "prefill: len out of range");
  draft_g = -1;  // the prefill writes every request's drafter K/V in HBM
  next_pf = false;  // (a pending cross-step prefetch only duplicates the prefill's own copies)
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
      expert_block(l, p_xp, PT, E, p_off, d_w_index + size_t(l) * E, tmode ? d_w_code + size_t(l) * E : nullptr, p_hb,
                   p_y, pf_splits, pf_splits, st);
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
}  // namespace smo
