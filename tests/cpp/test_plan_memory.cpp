// CPU test: the additive plan_memory overload for the B200 engine placement
// (SURVEY.md App. C.5): resident target K/V and the streamer's HBM slots are
// charged to HBM; the reference's own plan_memory is unchanged.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include "moeplan/memory.hpp"

using namespace moeplan;

namespace {
HardwareSpec b200() {
  HardwareSpec hw;
  hw.p_gpu = 1384.5e12;
  hw.b_gpu = 6555.5e9;
  hw.b_h2d = 55.5e9;
  hw.p_cpu = 2.0e12;
  hw.b_cpu = 200e9;
  hw.gpu_mem = 180e9;
  hw.cpu_mem = 196e9;
  return hw;
}
ModelSpec mixtral() {
  ModelSpec m;
  m.h = 4096;
  m.h_i = 14336;
  m.n_expert = 8;
  m.n_activate = 2;
  m.n_layers = 32;
  m.g = 4;
  m.bytes_per_elem = 2;
  m.param_bytes = 87e9;
  m.draft.param_bytes = 1e9;
  m.draft.kv_bytes_per_token = 16384;
  return m;
}
WorkloadSpec w1024() {
  WorkloadSpec w;
  w.mean_input_len = 1024;
  w.std_input_len = 0;
  w.output_len = 64;
  w.acceptance = AcceptanceCurve::geometric(0.8, 8);
  return w;
}
}  // namespace

TEST_CASE("resident target K/V and expert slots are charged to HBM") {
  const HardwareSpec hw = b200();
  const ModelSpec m = mixtral();
  const WorkloadSpec w = w1024();
  MemoryPolicy pol;
  pol.expert_cache_bytes = 5.25e9;
  ExecStrategy es;
  es.attention_placement = AttentionPlacement::GPU_RESIDENT;
  const MemoryPlan ref = plan_memory(hw, m, w, 32, pol);
  const MemoryPlan eng = plan_memory(hw, m, w, 32, pol, es, 2);
  const double kv = 32.0 * kv_bytes_per_request(m, w.total_len());
  CHECK(eng.target_kv_gpu_bytes == doctest::Approx(kv));
  CHECK(eng.target_kv_cpu_bytes == 0.0);
  CHECK(ref.target_kv_cpu_bytes == doctest::Approx(kv));
  CHECK(ref.target_kv_gpu_bytes == 0.0);
  CHECK(eng.slot_pool_bytes == doctest::Approx(2.0 * 3.0 * 8.0 * 4096.0 * 14336.0 * 2.0));  // 2 x 2.82 GB
  // the draft-KV HBM split shrinks by exactly the two new terms
  const double each = double(w.total_len()) * m.draft.kv_bytes_per_token;
  CHECK(eng.gpu_split_requests <= ref.gpu_split_requests);
  CHECK(eng.draft_kv_total_bytes == ref.draft_kv_total_bytes);
  (void)each;
  // CPU placement: K/V stay in DRAM as in the reference; slots still in HBM
  es.attention_placement = AttentionPlacement::CPU;
  const MemoryPlan cpu = plan_memory(hw, m, w, 32, pol, es, 2);
  CHECK(cpu.target_kv_cpu_bytes == doctest::Approx(ref.target_kv_cpu_bytes));
  CHECK(cpu.target_kv_gpu_bytes == 0.0);
}

TEST_CASE("resident K/V beyond HBM raises CapacityError") {
  const HardwareSpec hw = b200();
  const ModelSpec m = mixtral();
  WorkloadSpec w = w1024();
  w.mean_input_len = 32768;
  MemoryPolicy pol;
  ExecStrategy es;
  es.attention_placement = AttentionPlacement::GPU_RESIDENT;
  // 64 requests x 32k tokens x 128 KiB per token = 275 GB of K/V > 180 GB of HBM
  CHECK_THROWS_AS(plan_memory(hw, m, w, 64, pol, es, 2), CapacityError);
  es.attention_placement = AttentionPlacement::CPU;  // in DRAM: the reference's (DRAM) check decides
  CHECK_THROWS_AS(plan_memory(hw, m, w, 64, pol, es, 2), CapacityError);
  const MemoryPlan ok = plan_memory(hw, m, w, 4, pol, es, 2);
  CHECK(ok.b_max == 4);
}
