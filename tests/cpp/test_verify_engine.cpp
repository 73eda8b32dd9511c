// GPU test: the C++ VerifyEngine behind the reference's planner API.
// Measured IterationResult / Schedule / ProfileSamples -> fit_latency_models
// -> optimize -> DraftLengthController, on the tiny config (BASELINE config 1).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <sstream>

#include "moeplan/optimizer.hpp"
#include "moeplan/report.hpp"
#include "moeplan/verify_engine.hpp"

using namespace moeplan;

namespace {

HardwareSpec b200() {
  HardwareSpec hw;
  hw.p_gpu = 1384.5e12;  // MEASURED_PEAKS.json bf16 sustained
  hw.b_gpu = 6555.5e9;   // MEASURED_PEAKS.json HBM
  hw.b_h2d = 55.5e9;     // pinned PCIe Gen5 x16, tools/probe_box.py
  hw.p_cpu = 2.0e12;
  hw.b_cpu = 200e9;
  hw.gpu_mem = 180e9;
  hw.cpu_mem = 196e9;
  return hw;
}

ModelSpec tiny() {
  ModelSpec m;
  m.h = 512;
  m.h_i = 1792;
  m.n_expert = 8;
  m.n_activate = 2;
  m.n_layers = 2;
  m.g = 4;  // 2 KV heads of 64
  m.draft.param_bytes = 1e8;
  m.draft.kv_bytes_per_token = 16;  // keeps the planner clear of the draft-KV DRAM spill quirk
  m.draft.ffn_ops_per_token = 1e7;
  ModelArch a;
  a.n_q_heads = 8;
  a.head_dim = 64;
  a.vocab = 32000;
  m.arch = a;
  return m;
}

WorkloadSpec apps() {
  WorkloadSpec w;
  w.mean_input_len = 512;
  w.std_input_len = 0;
  w.output_len = 128;
  w.acceptance = AcceptanceCurve::geometric(0.8, 8);
  return w;
}

VerifyBatch chain_batch(std::int64_t b, std::int64_t n, std::int32_t prefix) {
  VerifyBatch vb;
  vb.b = b;
  vb.n = n;
  for (std::int64_t i = 0; i < b * n; ++i) vb.tokens.push_back(std::int32_t((i * 7919) % 32000));
  vb.prefix_len.assign(std::size_t(b), prefix);
  return vb;
}

}  // namespace

TEST_CASE("VerifyEngine measures the reference's target DAG") {
  HardwareSpec hw = b200();
  ModelSpec m = tiny();
  WorkloadSpec w = apps();
  Hyperparameters hp;
  hp.b = 4;
  hp.k = 8;
  hp.exec_strategy.attention_placement = AttentionPlacement::GPU_RESIDENT;
  MemoryPlan plan = plan_memory(hw, m, w, hp.b, hp.mem_policy);
  EngineOptions opt;
  opt.max_seq = 1024;
  VerifyEngine eng(hw, m, hp, plan, opt);
  eng.fill_prefix(std::vector<std::int32_t>(4, 600));

  VerifyOutput out;
  IterationResult r = eng.verify(chain_batch(4, 5, 600), &out);
  CHECK(out.acc_len.size() == 4);
  CHECK(r.target_dag.size() == std::size_t(5 * m.n_layers));
  CHECK(r.breakdown.target_total > 0);
  CHECK(r.breakdown.h2d_transfer > 0);
  CHECK(r.breakdown.gpu_moe > 0);
  CHECK(r.breakdown.cpu_attention > 0);
  // measured schedule is consistent: every event starts after its deps end
  for (const auto& ev : r.target_dag)
    for (int d : ev.deps) CHECK(r.target_schedule.start[std::size_t(ev.id)] >= r.target_schedule.end[std::size_t(d)] - 1e-6);
  // Table-3 report labels and a Chrome trace of the measured timeline
  json rep = to_json(r.breakdown);
  CHECK(rep.contains("HtoD Transfer"));
  std::ostringstream tr;
  emit_trace(r.target_dag, r.target_schedule, tr);
  json trace = json::parse(tr.str());
  CHECK(trace["traceEvents"].size() == r.target_dag.size() + 3);
}

TEST_CASE("micro-batches: the measured DAG has build_target_dag(d, L, m)'s structure") {
  HardwareSpec hw = b200();
  ModelSpec m = tiny();
  WorkloadSpec w = apps();
  for (AttentionPlacement pl : {AttentionPlacement::GPU_RESIDENT, AttentionPlacement::CPU}) {
    Hyperparameters hp;
    hp.b = 4;
    hp.k = 4;
    hp.m = 2;
    hp.exec_strategy.attention_placement = pl;
    MemoryPlan plan = plan_memory(hw, m, w, hp.b, hp.mem_policy);
    EngineOptions opt;
    opt.max_seq = 1024;
    opt.lm_scale = 8.0f;  // decisive greedy margins: m = 1 and m = 2 round differently in K1 / split-K
    opt.router_scale = 4.0f;
    VerifyEngine eng(hw, m, hp, plan, opt);
    eng.fill_prefix(std::vector<std::int32_t>(4, 600));
    VerifyOutput o2, o1;
    IterationResult r = eng.verify(chain_batch(4, 5, 600), &o2);
    TargetStageDurations d;
    d.attn_resource = pl == AttentionPlacement::CPU ? ExecResource::CPU : ExecResource::GPU;
    const EventDag want = build_target_dag(d, m.n_layers, 2);
    REQUIRE(r.target_dag.size() == want.size());
    for (std::size_t i = 0; i < want.size(); ++i) {
      CHECK(r.target_dag[i].kind == want[i].kind);
      CHECK(r.target_dag[i].resource == want[i].resource);
      CHECK(r.target_dag[i].deps == want[i].deps);
      CHECK(r.target_dag[i].label == want[i].label);
    }
    // every measured event starts after its dependencies end
    for (const auto& ev : r.target_dag)
      for (int dd : ev.deps) CHECK(r.target_schedule.start[std::size_t(ev.id)] >= r.target_schedule.end[std::size_t(dd)] - 1e-6);
    // the same requests with m = 1: identical greedy results (tiny model: margins are wide)
    eng.set_micro_batches(1);
    IterationResult r1 = eng.verify(chain_batch(4, 5, 600), &o1);
    CHECK(r1.target_dag.size() == std::size_t(5 * m.n_layers));
    CHECK(o1.acc_len == o2.acc_len);
    CHECK(o1.bonus == o2.bonus);
  }
}

TEST_CASE("H2D_EXPERTS samples use the estimator's driving unit (bf16 layer bytes)") {
  HardwareSpec hw = b200();
  ModelSpec m = tiny();
  WorkloadSpec w = apps();
  Hyperparameters hp;
  hp.b = 4;
  hp.k = 4;
  hp.mem_policy.expert_cache_bytes = 3.0 * 3.0 * m.expert_size() * 2.0;  // layers stream 5 and 8 blocks
  MemoryPlan plan = plan_memory(hw, m, w, hp.b, hp.mem_policy);
  EngineOptions opt;
  opt.max_seq = 1024;
  VerifyEngine eng(hw, m, hp, plan, opt);
  eng.fill_prefix(std::vector<std::int32_t>(4, 600));
  for (int rep = 0; rep < 4; ++rep) {  // two batch shapes: every stage kind gets two driving values
    eng.verify(chain_batch(4, 5, 600));
    eng.verify(chain_batch(2, 3, 600));
  }
  const double blk = 3.0 * m.expert_size() * 2.0;
  double t8 = 0;
  int n8 = 0;
  for (const auto& smp : eng.profile())
    if (smp.kind == EventKind::H2D_EXPERTS) {
      const double blocks = smp.driving / blk;
      CHECK(std::abs(blocks - std::round(blocks)) < 1e-9);  // whole bf16 blocks, coded or not
      if (std::round(blocks) == 8) {
        t8 += smp.seconds;
        ++n8;
      }
    }
  REQUIRE(n8 > 0);
  LatencyModel lm = fit_latency_models(eng.profile());
  // at the driving value iteration_time uses (the full bf16 layer,
  // pipeline.hpp:361-364) the fit predicts the measured full-layer transfer
  const double pred = lm.at(EventKind::H2D_EXPERTS).at(3.0 * double(m.n_expert) * m.expert_size() * 2.0);
  CHECK(pred == doctest::Approx(t8 / n8).epsilon(0.25));
}

TEST_CASE("measured profiles drive fit_latency_models, optimize and the controller") {
  HardwareSpec hw = b200();
  ModelSpec m = tiny();
  WorkloadSpec w = apps();
  Hyperparameters hp;
  hp.b = 4;
  hp.k = 8;
  // three hot-cached experts: layer 0 streams 5 blocks, layer 1 streams 8
  hp.mem_policy.expert_cache_bytes = 3.0 * 3.0 * m.expert_size() * 2.0;
  MemoryPlan plan = plan_memory(hw, m, w, hp.b, hp.mem_policy);
  EngineOptions opt;
  opt.max_seq = 2048;
  VerifyEngine eng(hw, m, hp, plan, opt);
  eng.fill_prefix(std::vector<std::int32_t>(4, 1024));
  for (int rep = 0; rep < 2; ++rep)
    for (std::int64_t n : {2, 3, 5, 9}) {
      eng.verify(chain_batch(4, n, 1024));
      eng.verify(chain_batch(2, n, 512));
    }
  REQUIRE(eng.profile().size() == 2 * 8 * (5 + 2));
  std::vector<std::string> warnings;
  LatencyModel lm = fit_latency_models(eng.profile(), &warnings);
  CHECK(lm.count(EventKind::CPU_ATTN) == 1);
  CHECK(lm.count(EventKind::H2D_EXPERTS) == 1);
  CHECK(lm.at(EventKind::H2D_EXPERTS).slope > 1.0 / 100e9);  // slower than 100 GB/s: it is the PCIe link
  CHECK(lm.at(EventKind::GPU_MOE).intercept >= 0);
  // the reference tuner on measured latencies
  Plan p = optimize(hw, m, w, &lm, 8);
  CHECK(p.k >= 0);
  CHECK(p.expected_throughput > 0);
  DraftLengthController ctl([&](std::int64_t prefix, std::int64_t active) {
    Hyperparameters base;
    (void)active;
    return optimize(hw, m, w, &lm, 8, base, prefix).k;
  });
  const int k1 = ctl.update(600, 4);
  const int k2 = ctl.update(700, 4);
  CHECK(k2 <= k1);
}

TEST_CASE("closed loop: prefill -> measured fit -> controller picks k -> decode commits the greedy sequence") {
  HardwareSpec hw = b200();
  ModelSpec m = tiny();
  WorkloadSpec w = apps();
  Hyperparameters hp;
  hp.b = 3;
  hp.k = 4;
  // two hot-cached experts: the layers stream different byte counts, so the
  // H2D_EXPERTS fit has two driving values
  hp.mem_policy.expert_cache_bytes = 2.0 * 3.0 * m.expert_size() * 2.0;
  MemoryPlan plan = plan_memory(hw, m, w, hp.b, hp.mem_policy);
  EngineOptions opt;
  opt.max_seq = 512;
  opt.seed = 0x5EED + 7;
  opt.lm_scale = 8.0f;  // decisive greedy margins (SURVEY.md §7.5 screening)
  opt.router_scale = 4.0f;
  std::vector<std::vector<std::int32_t>> prompts(3);
  std::uint64_t lcg = 12345;
  const int lens[3] = {40, 17, 9};
  for (int r = 0; r < 3; ++r)
    for (int i = 0; i < lens[r]; ++i) {
      lcg = lcg * 6364136223846793005ull + 1442695040888963407ull;
      prompts[std::size_t(r)].push_back(std::int32_t((lcg >> 33) % 32000));
    }

  VerifyEngine eng(hw, m, hp, plan, opt);
  const std::vector<std::int32_t> next = eng.prefill(prompts);
  CHECK(eng.kv_len() == std::vector<std::int32_t>({40, 17, 9}));
  for (int k : {1, 2, 4}) {  // measured warm-up across draft lengths
    IterationResult r = eng.decode_step(k);
    CHECK(r.draft_dag.size() == std::size_t(k + 1));
    CHECK(r.breakdown.draft_total > 0);
    CHECK(r.breakdown.iteration >= r.breakdown.target_total);
  }
  LatencyModel lm = fit_latency_models(eng.profile());
  CHECK(lm.count(EventKind::DRAFT_GPU_STEP) == 1);
  DraftLengthController ctl([&](std::int64_t prefix, std::int64_t active) {
    Hyperparameters base;
    base.b = active;
    return optimize(hw, m, w, &lm, 4, base, prefix).k;
  });
  const std::vector<IterationResult> rs = eng.decode(6, ctl);
  CHECK(rs.size() == 6);
  CHECK(eng.chosen_k().size() == 6);
  for (std::size_t i = 1; i < eng.chosen_k().size(); ++i) CHECK(eng.chosen_k()[i] <= eng.chosen_k()[i - 1]);
  const auto spec = eng.committed();

  // greedy invariance: plain decoding (k = 0) on a second engine commits the
  // same tokens (acceptance only changes how many per step)
  VerifyEngine plain(hw, m, hp, plan, opt);
  CHECK(plain.prefill(prompts) == next);
  std::size_t need = 0;
  for (const auto& c : spec) need = std::max(need, c.size());
  for (std::size_t i = 0; i < need; ++i) plain.decode_step(0);
  const auto ref = plain.committed();
  for (std::size_t r = 0; r < spec.size(); ++r) {
    REQUIRE(ref[r].size() >= spec[r].size());
    CHECK(std::vector<std::int32_t>(ref[r].begin(), ref[r].begin() + std::ptrdiff_t(spec[r].size())) == spec[r]);
  }
}

TEST_CASE("drafter split: dynamic_split_ratio moves requests to the host part, build_draft_dag structure, greedy") {
  HardwareSpec hw = b200();
  ModelSpec m = tiny();
  WorkloadSpec w = apps();
  Hyperparameters hp;
  hp.b = 3;
  hp.k = 4;
  MemoryPlan plan = plan_memory(hw, m, w, hp.b, hp.mem_policy);
  EngineOptions opt;
  opt.max_seq = 512;
  opt.seed = 0x5EED + 7;
  opt.lm_scale = 8.0f;
  opt.router_scale = 4.0f;
  std::vector<std::vector<std::int32_t>> prompts(3);
  std::uint64_t lcg = 777;
  const int lens[3] = {40, 17, 9};
  for (int r = 0; r < 3; ++r)
    for (int i = 0; i < lens[r]; ++i) {
      lcg = lcg * 6364136223846793005ull + 1442695040888963407ull;
      prompts[std::size_t(r)].push_back(std::int32_t((lcg >> 33) % 32000));
    }
  // an HBM budget that holds the draft K/V of ~500 / (16 B x current length)
  // requests: 1 of 3 at the start, none once the mean length passes 31
  HardwareSpec tight = hw;
  tight.gpu_mem = m.draft.param_bytes + 500.0;
  EngineOptions so = opt;
  so.draft_cpu_kv = true;
  MemoryPolicy pol;
  pol.activation_bytes = 0;
  so.draft_split_policy = pol;
  VerifyEngine eng(tight, m, hp, plan, so);
  eng.prefill(prompts);
  bool partial = false, all_cpu = false;
  for (int it = 0; it < 8; ++it) {
    const int k = 2 + it % 2;  // two driving values per stage for the fit below
    IterationResult r = eng.decode_step(k);
    const std::int64_t g = eng.draft_split_history().back();
    if (g >= 3) {
      CHECK(r.draft_dag.size() == std::size_t(k + 1));
      continue;
    }
    partial = partial || g > 0;
    all_cpu = all_cpu || g == 0;
    std::size_t n_gpu = 0, n_cpu = 0, n_ffn = 0;
    for (const auto& ev : r.draft_dag) {
      if (ev.kind == EventKind::DRAFT_GPU_STEP) ++n_gpu;
      if (ev.kind == EventKind::DRAFT_CPU_ATTN) {
        ++n_cpu;
        CHECK(ev.resource == ExecResource::CPU);
        CHECK(ev.duration > 0);
      }
      if (ev.kind == EventKind::DRAFT_GPU_FFN) {
        ++n_ffn;
        REQUIRE(ev.deps.size() == 1);
        CHECK(r.draft_dag[std::size_t(ev.deps[0])].kind == EventKind::DRAFT_CPU_ATTN);
      }
    }
    CHECK(n_cpu == std::size_t(k + 1));
    CHECK(n_ffn == std::size_t(k + 1));
    CHECK(n_gpu == (g > 0 ? std::size_t(k + 1) : 0u));
    CHECK(r.breakdown.draft_cpu_part > 0);
    // the same structure as the reference's DAG for these splits
    CHECK(build_draft_dag(DraftStepDurations{}, k + 1, g, 3 - g).size() == r.draft_dag.size());
  }
  const auto& hist = eng.draft_split_history();
  for (std::size_t i = 1; i < hist.size(); ++i) CHECK(hist[i] <= hist[i - 1]);  // nonincreasing in length
  CHECK(partial);
  CHECK(all_cpu);
  // DRAFT_CPU_ATTN samples on the reference's driving variable (cpu requests x
  // prefix, pipeline.hpp:262) for fit_latency_models
  std::vector<double> xs;
  for (const auto& sm : eng.profile())
    if (sm.kind == EventKind::DRAFT_CPU_ATTN) xs.push_back(sm.driving);
  CHECK(xs.size() >= 8);
  CHECK(*std::max_element(xs.begin(), xs.end()) > *std::min_element(xs.begin(), xs.end()));
  const auto split = eng.committed();
  // greedy invariance: the split only moves where the drafter attends
  VerifyEngine plain(hw, m, hp, plan, opt);
  plain.prefill(prompts);
  for (int it = 0; it < 8; ++it) plain.decode_step(2 + it % 2);
  const auto ref = plain.committed();
  for (std::size_t r = 0; r < split.size(); ++r) {
    const std::size_t nn = std::min(ref[r].size(), split[r].size());
    CHECK(nn >= 8);
    CHECK(std::vector<std::int32_t>(ref[r].begin(), ref[r].begin() + std::ptrdiff_t(nn)) ==
          std::vector<std::int32_t>(split[r].begin(), split[r].begin() + std::ptrdiff_t(nn)));
  }
}
