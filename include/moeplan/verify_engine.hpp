#pragma once
// moeplan/verify_engine.hpp — the measured verify step behind the planner API.
//
// Additive engine API of SURVEY.md §8(b): a C++ VerifyEngine constructed from
// the reference's own value types (HardwareSpec, ModelSpec, Hyperparameters,
// MemoryPlan). verify() runs one speculative verification step on the B200
// (libspecmoe.so: K1-K6 kernels + the K5 expert streamer) and returns the
// reference's IterationResult with MEASURED durations: the target DAG of
// pipeline.hpp:147-206 with one event per layer and stage, its measured
// Schedule, and the Table-3 breakdown (report.hpp:27-37). profile() returns
// ProfileSamples with the reference's driving variables (pipeline.hpp:256-264)
// so fit_latency_models() -> optimize() -> DraftLengthController run on real
// timings.
//
// Stage mapping: K1 attention -> CPU_ATTN (name kept),
// norms/QKV/RoPE -> GPU_OTHER1, O-proj/router/permute -> GPU_OTHER2,
// K4 experts + combine -> GPU_MOE, K5 copy-engine transfer -> H2D_EXPERTS.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "moeplan/config.hpp"
#include "moeplan/memory.hpp"
#include "moeplan/optimizer.hpp"
#include "moeplan/pipeline.hpp"
#include "moeplan/specdec.hpp"
#include "specmoe/c_api.h"

namespace moeplan {

struct EngineOptions {
  std::int64_t max_seq = 0;            // KV capacity per request (0: 2048)
  int hbm_slots = 2;                   // expert staging slots
  int host_alias_layers = 0;           // pinned host buffers shared by layers (0: one per layer)
  int device = 0;
  bool debug = false;
  std::uint64_t seed = 0x5EED;         // procedural weights
  float lm_scale = 1.0f;
  float router_scale = 1.0f;
  bool drafter = true;                 // build the drafter from ModelSpec.draft (f1) when it has FFN ops
  int kv_pages = 0;                    // K/V layout (f2): 0 contiguous, > 0 paged pool size, -1 paged auto
  bool compress_experts = true;        // experts cross the host link in the lossless K5 code (xfer.cu)
  // expert parallelism: this rank owns experts e % ep_size ==
  // ep_rank and streams only those; ep_group = an smo_ep_group (NCCL, CUDA-IPC
  // peer mailboxes or loopback) of ep_size ranks, owned by the caller
  int ep_rank = 0;
  int ep_size = 1;
  smo_ep_group* ep_group = nullptr;
  // drafter GPU-part / CPU-part split (build_draft_dag
  // pipeline.hpp:217-253): with draft_cpu_kv every decode step first sets how
  // many requests keep the drafter on the GPU — dynamic_split_ratio(hw, model,
  // *draft_split_policy, current length, b) (memory.hpp:93-106) when a policy
  // is given, else draft_gpu_requests (-1: all); the rest attend on the host
  bool draft_cpu_kv = false;
  std::optional<MemoryPolicy> draft_split_policy;
  std::int64_t draft_gpu_requests = -1;
};

struct VerifyBatch {
  std::int64_t b = 0;
  std::int64_t n = 0;                  // verify rows per request = k + 1 (root + drafts)
  std::vector<std::int32_t> tokens;    // b*n, row 0 of each request is the root
  std::vector<std::int32_t> parent;    // empty: chain; else b*n tree parents (-1 root)
  std::vector<std::int32_t> prefix_len;  // b
};

struct VerifyOutput {
  std::vector<std::int32_t> acc_len;   // accepted drafts per request (committed = acc + 1)
  std::vector<std::int32_t> bonus;     // greedy token at the accepted tip
  std::vector<std::int32_t> keep;      // accepted rows, root first, -1 padded
  std::vector<std::int32_t> target;    // argmax per verify row
};

namespace detail {
inline void smo_check(smo_status st) {
  if (st == SMO_OK) return;
  if (st == SMO_INVALID_ARG) throw std::invalid_argument(smo_last_error());
  if (st == SMO_CAPACITY) throw CapacityError(smo_last_error());
  throw std::runtime_error(std::string("specmoe: ") + smo_last_error());
}
}  // namespace detail

class VerifyEngine {
 public:
  VerifyEngine(const HardwareSpec& hw, const ModelSpec& model, const Hyperparameters& hyper, const MemoryPlan& plan,
               const EngineOptions& opt = {})
      : hw_(hw), model_(model), hyper_(hyper) {
    if (hyper.exec_strategy.attention_placement == AttentionPlacement::GPU_TRANSFER)
      throw std::invalid_argument(
          "VerifyEngine: AttentionPlacement::GPU_TRANSFER (target K/V streamed over the host link every step, "
          "roofline.hpp:94-103) is not implemented; use GPU_RESIDENT (K/V in HBM) or CPU (host attention)");
    if (!model.arch || model.arch->n_q_heads <= 0 || model.arch->head_dim <= 0 || model.arch->vocab <= 0)
      throw std::invalid_argument("VerifyEngine: ModelSpec.arch (n_q_heads, head_dim, vocab) is required");
    const ModelArch& a = *model.arch;
    const std::int64_t kv_width = model.h / model.g;  // K (or V) width per token, config.hpp:54
    if (kv_width % a.head_dim != 0) throw std::invalid_argument("VerifyEngine: h/g must be a multiple of head_dim");
    smo_model_config c{};
    c.hidden = std::int32_t(model.h);
    c.inter = std::int32_t(model.h_i);
    c.n_expert = std::int32_t(model.n_expert);
    c.top_k = std::int32_t(model.n_activate);
    c.n_layers = std::int32_t(model.n_layers);
    c.n_q_heads = std::int32_t(a.n_q_heads);
    c.n_kv_heads = std::int32_t(kv_width / a.head_dim);
    c.head_dim = std::int32_t(a.head_dim);
    c.vocab = std::int32_t(a.vocab);
    c.rope_theta = float(a.rope_theta);
    c.rms_eps = float(a.rms_eps);
    c.seed = opt.seed;
    c.lm_scale = opt.lm_scale;
    c.router_scale = opt.router_scale;
    c.shared_inter = std::int32_t(a.shared_expert_inter);
    // drafter: DraftModelSpec (config.hpp:40-45) -> dense
    // decoder layers; ffn_ops_per_token = 2*3*h*draft_inter
    if (opt.drafter && model.draft.n_layers > 0 && model.draft.ffn_ops_per_token > 0) {
      const double di = model.draft.ffn_ops_per_token / (6.0 * double(model.h));
      c.draft_layers = std::int32_t(model.draft.n_layers);
      c.draft_inter = std::int32_t(std::max(1.0, std::round(di / 128.0)) * 128.0);
    }
    smo_engine_options o{};
    o.max_batch = std::int32_t(hyper.b);
    o.max_verify = std::int32_t(std::max(1, hyper.k) + 1);
    o.max_seq = std::int32_t(opt.max_seq > 0 ? opt.max_seq : 2048);
    // capacity from the MemoryPlan: the hot cache, and (engine-placement
    // plan, memory.hpp overload) the streamer's staging slots
    if (hyper.b > plan.b_max) throw CapacityError("VerifyEngine: Hyperparameters.b exceeds MemoryPlan.b_max");
    const double layer_bytes = 3.0 * double(model.n_expert) * model.expert_size() * double(model.bytes_per_elem);
    o.hbm_slots = plan.slot_pool_bytes > 0 ? std::max(2, int(std::lround(plan.slot_pool_bytes / layer_bytes)))
                                           : opt.hbm_slots;
    o.expert_cache_bytes = std::int64_t(plan.expert_cache_bytes);
    o.host_alias_layers = opt.host_alias_layers;
    o.device = opt.device;
    o.flags = opt.debug ? SMO_ENGINE_DEBUG : 0;
    o.ep_rank = opt.ep_rank;
    o.ep_size = opt.ep_size;
    o.nccl_comm = opt.ep_group;
    if (opt.ep_size > 1 && !opt.ep_group)
      throw std::invalid_argument("VerifyEngine: ep_size > 1 needs EngineOptions.ep_group");
    // Hyperparameters.m (config.hpp:118-125): micro-batches, stage-major per
    // layer like build_target_dag (pipeline.hpp:147-206)
    o.micro_batches = std::int32_t(std::max<std::int64_t>(1, hyper.m));
    o.kv_pages = opt.kv_pages;
    o.compress_experts = opt.compress_experts ? 1 : 0;
    o.draft_cpu_kv = opt.draft_cpu_kv ? 1 : 0;
    // AttentionPlacement::CPU (the reference's default, config.hpp:110): target
    // K/V in pinned host DRAM, attention on the host pool (f4); GPU_RESIDENT
    // runs K1 on HBM-resident K/V (GPU_TRANSFER is rejected above)
    o.attn_cpu = hyper.exec_strategy.attention_placement == AttentionPlacement::CPU ? 1 : 0;
    // MoeBatching::BATCH_ONE (config.hpp:111): stream only router-selected experts
    o.moe_batching = hyper.exec_strategy.moe_batching == MoeBatching::BATCH_ONE ? 1 : 0;
    detail::smo_check(smo_engine_create(&c, &o, &h_));
    layers_ = model.n_layers;
    max_verify_ = o.max_verify;
    max_seq_ = o.max_seq;
    attn_cpu_ = o.attn_cpu != 0;
    draft_cpu_kv_ = opt.draft_cpu_kv;
    draft_split_policy_ = opt.draft_split_policy;
    draft_gpu_requests_ = opt.draft_gpu_requests;
  }
  VerifyEngine(const VerifyEngine&) = delete;
  VerifyEngine& operator=(const VerifyEngine&) = delete;
  ~VerifyEngine() {
    if (h_) smo_engine_destroy(h_);
  }

  // The m of a plan (optimize(), optimizer.hpp:130-175) for the next steps.
  void set_micro_batches(std::int64_t m) {
    detail::smo_check(smo_engine_set_micro_batches(h_, std::int32_t(std::max<std::int64_t>(1, m))));
  }

  void fill_prefix(const std::vector<std::int32_t>& prefix_len) {
    detail::smo_check(smo_engine_fill_prefix(h_, prefix_len.data(), std::int32_t(prefix_len.size())));
  }

  // One verify step from host buffers; returns the measured IterationResult.
  IterationResult verify(const VerifyBatch& in, VerifyOutput* out = nullptr) {
    const std::size_t T = std::size_t(in.b * in.n);
    if (in.tokens.size() != T || in.prefix_len.size() != std::size_t(in.b) ||
        (!in.parent.empty() && in.parent.size() != T))
      throw std::invalid_argument("VerifyEngine::verify: batch shape mismatch");
    VerifyOutput local;
    VerifyOutput& o = out ? *out : local;
    o.acc_len.assign(std::size_t(in.b), 0);
    o.bonus.assign(std::size_t(in.b), 0);
    o.keep.assign(T, -1);
    o.target.assign(T, 0);
    smo_verify_batch vb{std::int32_t(in.b), std::int32_t(in.n), in.tokens.data(),
                        in.parent.empty() ? nullptr : in.parent.data(), in.prefix_len.data(), 0};
    smo_verify_output vo{o.acc_len.data(), o.bonus.data(), o.keep.data(), o.target.data(), 0};
    detail::smo_check(smo_engine_verify(h_, &vb, &vo, nullptr));
    return measured(in);
  }

  // ---- KV lifecycle + decode loop ----------------------
  // Prefill (f2): the prompts' real K/V for the target and the drafter,
  // layer-major (each layer's experts streamed once). Returns the greedy next
  // token per request and starts the decode state (kv_len = prompt length).
  std::vector<std::int32_t> prefill(const std::vector<std::vector<std::int32_t>>& prompts) {
    if (prompts.empty()) throw std::invalid_argument("VerifyEngine::prefill: no prompts");
    std::size_t lmax = 0;
    for (const auto& p : prompts) lmax = std::max(lmax, p.size());
    std::vector<std::int32_t> tok(prompts.size() * lmax, 0), len, next(prompts.size(), 0);
    for (std::size_t r = 0; r < prompts.size(); ++r) {
      std::copy(prompts[r].begin(), prompts[r].end(), tok.begin() + std::ptrdiff_t(r * lmax));
      len.push_back(std::int32_t(prompts[r].size()));
    }
    detail::smo_check(smo_engine_prefill(h_, tok.data(), len.data(), std::int32_t(prompts.size()),
                                         std::int32_t(lmax), next.data(), nullptr));
    kv_len_ = len;
    return next;
  }

  void decode_begin(const std::vector<std::int32_t>& root, const std::vector<std::int32_t>& kv_len) {
    if (root.size() != kv_len.size()) throw std::invalid_argument("VerifyEngine::decode_begin: size mismatch");
    detail::smo_check(smo_engine_decode_begin(h_, root.data(), kv_len.data(), std::int32_t(root.size())));
    kv_len_ = kv_len;
  }

  // One decode iteration (f1): k drafts from the on-device drafter (or the
  // planted b*k tokens) -> verify -> greedy accept -> commit. Returns the
  // measured IterationResult with the draft DAG (pipeline.hpp:208-253) of
  // k+1 DRAFT_GPU_STEP events and breakdown.iteration = draft + target.
  IterationResult decode_step(int k, const std::vector<std::int32_t>* planted = nullptr) {
    if (kv_len_.empty()) throw std::invalid_argument("VerifyEngine::decode_step: call prefill or decode_begin first");
    if (planted && planted->size() != kv_len_.size() * std::size_t(std::max(k, 0)))
      throw std::invalid_argument("VerifyEngine::decode_step: planted drafts must be b*k tokens");
    VerifyBatch vb;  // driving variables of this step (pipeline.hpp:256-264)
    vb.b = std::int64_t(kv_len_.size());
    vb.n = k + 1;
    vb.prefix_len = kv_len_;
    double s = 0;
    for (auto p : kv_len_) s += double(p);
    s /= double(kv_len_.size());
    // the drafter split of this step (f1): GPU-part requests from the memory
    // policy at the current length (memory.hpp:93-106) or the fixed count
    std::int64_t g = vb.b;
    if (draft_cpu_kv_) {
      g = draft_split_policy_
              ? dynamic_split_ratio(hw_, model_, *draft_split_policy_, std::max<std::int64_t>(1, std::llround(s) + k + 1),
                                    vb.b)
              : (draft_gpu_requests_ < 0 ? vb.b : std::min(draft_gpu_requests_, vb.b));
      detail::smo_check(smo_engine_set_draft_split(h_, g >= vb.b ? -1 : std::int32_t(g)));
      split_gpu_.push_back(g);
    }
    detail::smo_check(smo_engine_decode_step(h_, k, planted ? planted->data() : nullptr, nullptr));
    IterationResult r = measured(vb);
    std::vector<double> dt(std::size_t(k) + 2, 0.0), sp(3 * (std::size_t(k) + 2), 0.0);
    std::int32_t steps = 0, ssteps = 0;
    detail::smo_check(smo_engine_draft_times(h_, dt.data(), dt.size(), &steps));
    if (g < vb.b) detail::smo_check(smo_engine_draft_split_times(h_, sp.data(), sp.size(), &ssteps));
    double t0 = 0;
    std::vector<int> prev;
    auto add = [&](EventKind kind, ExecResource res, double start, double dur, std::vector<int> deps,
                   const std::string& label) {
      EventNode ev;
      ev.id = int(r.draft_dag.size());
      ev.kind = kind;
      ev.resource = res;
      ev.duration = dur;
      ev.deps = std::move(deps);
      ev.label = label;
      r.draft_dag.push_back(ev);
      r.draft_schedule.start.push_back(start);
      r.draft_schedule.end.push_back(start + dur);
      r.draft_schedule.busy[std::size_t(res)] += dur;
      return ev.id;
    };
    for (int t = 0; t < steps; ++t) {
      const std::string tag = "draft/step" + std::to_string(t) + "/";
      std::vector<int> ends;
      if (ssteps > t) {  // build_draft_dag (pipeline.hpp:217-253): GPU_STEP || CPU_ATTN -> GPU_FFN
        const double a = sp[3 * std::size_t(t)], host = sp[3 * std::size_t(t) + 1], after = sp[3 * std::size_t(t) + 2];
        const double end = t0 + a + after, ffn0 = t0 + std::max(a, host);
        if (g > 0) {
          ends.push_back(add(EventKind::DRAFT_GPU_STEP, ExecResource::GPU, t0, a, prev, tag + "GPU_STEP"));
          samples_.push_back({EventKind::DRAFT_GPU_STEP, double(g) * s, a});
          r.breakdown.draft_gpu_part += a;
        }
        const int at = add(EventKind::DRAFT_CPU_ATTN, ExecResource::CPU, t0, host, prev, tag + "CPU_ATTN");
        samples_.push_back({EventKind::DRAFT_CPU_ATTN, double(vb.b - g) * s, host});
        const double ffn = std::max(0.0, end - ffn0);
        ends.push_back(add(EventKind::DRAFT_GPU_FFN, ExecResource::GPU, ffn0, ffn, {at}, tag + "GPU_FFN"));
        r.breakdown.draft_cpu_part += host + ffn;  // the breakdown's convention (pipeline.hpp:407-411)
        t0 = end;
      } else {
        ends.push_back(add(EventKind::DRAFT_GPU_STEP, ExecResource::GPU, t0, dt[std::size_t(t)], prev,
                           tag + "GPU_STEP"));
        samples_.push_back({EventKind::DRAFT_GPU_STEP, double(vb.b) * s, dt[std::size_t(t)]});
        r.breakdown.draft_gpu_part += dt[std::size_t(t)];
        t0 += dt[std::size_t(t)];
      }
      prev = std::move(ends);
    }
    r.draft_schedule.makespan = t0;
    r.breakdown.draft_total = t0;
    r.breakdown.iteration = r.breakdown.target_total + t0;
    std::vector<std::int32_t> kv(kv_len_.size());
    detail::smo_check(smo_engine_decode_read(h_, nullptr, 0, nullptr, kv.data(), nullptr));
    kv_len_ = kv;
    return r;
  }

  // Closed loop (f3): each iteration asks the controller for k at the current
  // mean prefix (DraftLengthController::update, specdec.hpp:97-124) — its
  // SweepFn typically runs optimize() on fit_latency_models(profile()) — and
  // runs one measured decode step with it (clamped to the engine's capacity).
  std::vector<IterationResult> decode(int iterations, DraftLengthController& ctl) {
    std::vector<IterationResult> out;
    for (int it = 0; it < iterations; ++it) {
      double s = 0;
      for (auto p : kv_len_) s += double(p);
      s /= double(std::max<std::size_t>(1, kv_len_.size()));
      const int k = std::clamp(ctl.update(std::int64_t(s), std::int64_t(kv_len_.size())), 0, max_verify_ - 1);
      ks_.push_back(k);
      out.push_back(decode_step(k));
    }
    return out;
  }

  // Committed tokens per request since prefill/decode_begin (accepted drafts
  // + bonus of every step; the prefill's next token is the first root).
  std::vector<std::vector<std::int32_t>> committed() {
    const std::int32_t b = std::int32_t(kv_len_.size()), cap = std::int32_t(max_seq_);  // history capacity
    std::vector<std::int32_t> buf(static_cast<std::size_t>(b) * std::size_t(cap)), n(static_cast<std::size_t>(b));
    detail::smo_check(smo_engine_decode_read(h_, buf.data(), cap, n.data(), nullptr, nullptr));
    std::vector<std::vector<std::int32_t>> out(static_cast<std::size_t>(b));
    for (std::int32_t r = 0; r < b; ++r)
      out[std::size_t(r)].assign(buf.begin() + std::ptrdiff_t(r) * cap,
                                 buf.begin() + std::ptrdiff_t(r) * cap + std::min<std::int32_t>(cap, n[std::size_t(r)]));
    return out;
  }
  const std::vector<std::int32_t>& kv_len() const { return kv_len_; }
  const std::vector<int>& chosen_k() const { return ks_; }
  // GPU-part request count the drafter split used at each decode step
  const std::vector<std::int64_t>& draft_split_history() const { return split_gpu_; }

  // Accumulated measured samples (one per stage kind and verify call).
  const std::vector<ProfileSample>& profile() const { return samples_; }
  void clear_profile() { samples_.clear(); }

 private:
  IterationResult measured(const VerifyBatch& in) {
    smo_stage_times st{};
    detail::smo_check(smo_engine_last_times(h_, &st));
    std::int32_t m = 1;
    detail::smo_check(smo_engine_last_micro_batches(h_, &m));
    const std::size_t stride = 4 + 6 * std::size_t(m);
    std::vector<double> lt(std::size_t(layers_) * stride);
    detail::smo_check(smo_engine_layer_times(h_, lt.data(), lt.size()));
    IterationResult r;
    EventDag& dag = r.target_dag;
    Schedule& sc = r.target_schedule;
    auto add = [&](EventKind k, ExecResource res, double t0, double t1, std::vector<int> deps, std::string lbl) {
      EventNode ev;
      ev.id = int(dag.size());
      ev.kind = k;
      ev.resource = res;
      ev.duration = std::max(0.0, t1 - t0);
      ev.deps = std::move(deps);
      ev.label = std::move(lbl);
      dag.push_back(ev);
      sc.start.push_back(t0);
      sc.end.push_back(t0 + dag.back().duration);
      sc.busy[std::size_t(res)] += dag.back().duration;
      sc.makespan = std::max(sc.makespan, sc.end.back());
      return ev.id;
    };
    // the measured DAG has build_target_dag's structure and id order
    // (pipeline.hpp:147-206): per layer the transfer, then each stage for
    // every micro-batch (stage-major); GPU_MOE(l, j) <- {GPU_OTHER2(l, j),
    // H2D(l)}, GPU_OTHER1(l, j) <- GPU_MOE(l-1, j)
    const ExecResource attn_res = attn_cpu_ ? ExecResource::CPU : ExecResource::GPU;
    int prev_h2d = -1;
    const std::size_t nm = std::size_t(m);
    std::vector<int> prev_moe(nm, -1), v_o1(nm, -1), v_at(nm, -1), v_o2(nm, -1);
    double attn = 0, moe = 0, h2d = 0, o1t = 0, o2t = 0;
    for (std::int64_t l = 0; l < layers_; ++l) {
      const double* t = lt.data() + std::size_t(l) * stride;  // h2d0 h2d1 bytes raw | per mb: o1 a0 a1 pre m0 m1
      const std::string L = "L" + std::to_string(l);
      std::vector<int> hd;
      if (prev_h2d >= 0) hd.push_back(prev_h2d);
      const int eh = add(EventKind::H2D_EXPERTS, ExecResource::H2D, t[0], t[1], hd, L + "/H2D_EXPERTS");
      prev_h2d = eh;
      h2d += t[1] - t[0];
      auto mbt = [&](int j) { return t + 4 + 6 * j; };
      auto tag = [&](int j, const char* stage) { return L + "/mb" + std::to_string(j) + "/" + stage; };
      for (int j = 0; j < m; ++j) {
        std::vector<int> od;
        if (prev_moe[std::size_t(j)] >= 0) od.push_back(prev_moe[std::size_t(j)]);
        v_o1[std::size_t(j)] = add(EventKind::GPU_OTHER1, ExecResource::GPU, mbt(j)[0], mbt(j)[1], od,
                                 tag(j, "GPU_OTHER1"));
        o1t += mbt(j)[1] - mbt(j)[0];
      }
      for (int j = 0; j < m; ++j) {
        v_at[std::size_t(j)] = add(EventKind::CPU_ATTN, attn_res, mbt(j)[1], mbt(j)[2], {v_o1[std::size_t(j)]},
                                 tag(j, "CPU_ATTN"));
        attn += mbt(j)[2] - mbt(j)[1];
      }
      for (int j = 0; j < m; ++j) {
        v_o2[std::size_t(j)] = add(EventKind::GPU_OTHER2, ExecResource::GPU, mbt(j)[2], mbt(j)[3],
                                 {v_at[std::size_t(j)]}, tag(j, "GPU_OTHER2"));
        o2t += mbt(j)[3] - mbt(j)[2];
      }
      for (int j = 0; j < m; ++j) {
        prev_moe[std::size_t(j)] = add(EventKind::GPU_MOE, ExecResource::GPU, mbt(j)[4], mbt(j)[5],
                                       {v_o2[std::size_t(j)], eh}, tag(j, "GPU_MOE"));
        moe += mbt(j)[5] - mbt(j)[4];
      }
    }
    IterationBreakdown& bd = r.breakdown;
    bd.target_total = st.target_total;
    bd.cpu_attention = attn;
    bd.gpu_moe = moe;
    bd.h2d_transfer = h2d;
    bd.others = std::max(0.0, st.target_total - attn - moe - o1t - o2t);
    bd.iteration = st.target_total;
    // driving variables as the reference defines them (pipeline.hpp:256-264);
    // the engine verifies n = k+1 rows, the reference charges k (App. C.2).
    // Per-micro-batch stages are charged per layer for the whole batch, as
    // iteration_time looks them up before dividing by m (pipeline.hpp:358-372).
    const double b = double(in.b);
    const double k = double(std::max<std::int64_t>(1, in.n - 1));
    double s = 0;
    for (auto p : in.prefix_len) s += double(p);
    s /= std::max(1.0, double(in.prefix_len.size()));
    const double nl = double(layers_);
    samples_.push_back({EventKind::CPU_ATTN, b * (s + k) * k, attn / nl});
    samples_.push_back({EventKind::GPU_MOE, b * k, moe / nl});
    // one transfer sample per layer. Driving variable: the bf16 bytes of the
    // experts the layer streamed — the unit iteration_time looks H2D_EXPERTS
    // up with (3 * n_expert * expert_size * bytes_per_elem, pipeline.hpp:
    // 361-364) — so the fitted slope absorbs the link code (and a hot cache
    // shows up as layers with fewer bytes): seconds per bf16 byte carried
    for (std::int64_t l = 0; l < layers_; ++l) {
      const double* t = lt.data() + std::size_t(l) * stride;
      if (t[3] > 0) samples_.push_back({EventKind::H2D_EXPERTS, t[3], t[1] - t[0]});
    }
    samples_.push_back({EventKind::GPU_OTHER1, b * k, o1t / nl});
    samples_.push_back({EventKind::GPU_OTHER2, b * k, o2t / nl});
    samples_.push_back({EventKind::OVERHEAD, b * (k + 1), bd.others});
    return r;
  }

  HardwareSpec hw_;
  ModelSpec model_;
  Hyperparameters hyper_;
  smo_engine* h_ = nullptr;
  std::int64_t layers_ = 0;
  int max_verify_ = 1;
  std::int64_t max_seq_ = 2048;
  bool attn_cpu_ = false;
  bool draft_cpu_kv_ = false;
  std::optional<MemoryPolicy> draft_split_policy_;
  std::int64_t draft_gpu_requests_ = -1;
  std::vector<std::int64_t> split_gpu_;
  std::vector<std::int32_t> kv_len_;  // decode state mirror (host)
  std::vector<int> ks_;
  std::vector<ProfileSample> samples_;
};

}  // namespace moeplan
