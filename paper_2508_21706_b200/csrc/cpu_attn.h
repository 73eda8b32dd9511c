// cpu_attn.h — host-side verification attention for the CPU placement
// (the paper's CPU attention, roofline.hpp:82-91,
// AttentionPlacement::CPU in config.hpp:110): target K/V live in pinned host
// DRAM and a pool of host threads computes the chunked verification attention
// of attention.hpp:117-156 for every (request, KV head) pair.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace smo {

struct CpuAttnJob {
  const uint16_t* q;        // bf16 [b*n, n_q, d]
  const uint16_t* k_cache;  // bf16 [b, n_kv, s_max, d]
  const uint16_t* v_cache;
  const uint64_t* mask;     // [b*n] compact draft mask (bit j = draft j visible)
  const int32_t* prefix;    // [b]
  uint16_t* out;            // bf16 [b*n, n_q, d]
  int b, n, n_q, n_kv, d, s_max;
  // chunked prefill: `chunks` consecutive verify batches of b*n rows, chunk c
  // reading prefix[c*b + r] (q/out advance by b*n rows per chunk; the [b*n]
  // mask is shared by every chunk)
  int chunks = 1;
};

// Fixed-size pool; run() blocks until every item is done. Not reentrant.
class CpuPool {
 public:
  explicit CpuPool(int threads);
  ~CpuPool();
  int threads() const { return int(workers_.size()); }
  void run(int items, const std::function<void(int)>& fn);

 private:
  void loop();
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int items_ = 0, next_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// fp32 arithmetic on bf16 inputs, output rounded to bf16: for each query row
// the visible scores (prefix keys + masked drafts) are scaled by 1/sqrt(d),
// exponentiated against the row maximum, normalised and applied to V.
void cpu_verify_attention(const CpuAttnJob& job, CpuPool& pool);

}  // namespace smo
