// streamer.cu — the expert weight streamer as a standalone handle
// (smo_streamer_*, SURVEY.md §8(b) "C-ABI to export"; north_star subsystem 2).
//
// The same mechanism the engine runs internally (engine.cu enqueue_h2d /
// decode_slot), for a caller that drives its own layers: expert blocks sit in
// caller-owned pinned host memory, raw bf16 or in a K5 link code; layer l
// streams into HBM slot l % slots on the streamer's copy-engine stream
// (after the slot's previous layer was released), hot-cached blocks are
// copied once at create and never streamed. The consumer makes its stream
// wait for the layer (coded blocks are expanded on that stream then), uses
// the block pointers, and releases the slot. This is the reference's
// H2D_EXPERTS(l) stage and its GPU_MOE(l) dependency (pipeline.hpp:147-206)
// with LARGE_BATCH / BATCH_ONE (roofline.hpp:155-162) choosing `active`.
#include <vector>

#include "engine.cuh"

namespace smo {

smo_status run_guarded(const std::function<void()>& f);

// makes the streamer's device current for the duration of a call, then
// restores the caller's (the C-ABI must not change the thread's device)
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    SMO_CUDA_CHECK(cudaGetDevice(&prev));
    if (prev != dev) SMO_CUDA_CHECK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

struct Streamer {
  int device = 0;
  int L = 0, E = 0, slots = 2;
  size_t blk = 0;                    // bf16 bytes of one block
  std::vector<const uint8_t*> host;  // [L*E]
  std::vector<uint64_t> hbytes;      // [L*E] bytes on the link
  std::vector<int32_t> code;         // [L*E] 0 raw, 1 unary, 3 / 4 bits
  std::vector<int> cache;            // [L*E] pool block of a cached expert, -1
  uint8_t* pool = nullptr;           // [slots*E + cached] blocks
  uint8_t* cstage = nullptr;         // [slots*E] coded staging (max coded bytes each)
  size_t cstride = 0;
  cudaStream_t copy = nullptr;
  std::vector<cudaEvent_t> ready, freed;  // per slot
  std::vector<int> slot_layer;            // layer last enqueued into each slot
  std::vector<std::vector<int>> pending;  // per slot: coded experts to expand at wait

  ~Streamer() {
    if (copy) cudaStreamSynchronize(copy);
    for (auto e : ready) cudaEventDestroy(e);
    for (auto e : freed) cudaEventDestroy(e);
    if (copy) cudaStreamDestroy(copy);
    cudaFree(pool);
    cudaFree(cstage);
  }
  size_t idx(int l, int e) const { return size_t(l) * E + size_t(e); }
  int slot_of(int l) const { return l % slots; }
  uint8_t* slot_block(int l, int e) const { return pool + (size_t(slot_of(l)) * E + e) * blk; }
};

}  // namespace smo

struct smo_streamer {
  smo::Streamer s;
};

extern "C" {

smo_status smo_streamer_create(const smo_streamer_args* a, smo_streamer** out) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(a && out && a->n_layers > 0 && a->n_experts > 0 && a->block_bytes > 0 && a->host_blocks,
                "streamer: bad arguments");
    SMO_REQUIRE(a->hbm_slots >= 2 && a->block_bytes % 2048 == 0, "streamer: >= 2 slots, block of 1024-value segments");
    smo::DeviceGuard dg(a->device);
    auto* h = new smo_streamer();
    smo::Streamer& s = h->s;
    s.device = a->device;
    try {
      s.L = a->n_layers;
      s.E = a->n_experts;
      s.slots = a->hbm_slots;
      s.blk = size_t(a->block_bytes);
      const size_t n = size_t(s.L) * s.E;
      s.host.resize(n);
      s.hbytes.resize(n);
      s.code.assign(n, 0);
      for (size_t i = 0; i < n; ++i) {
        s.host[i] = reinterpret_cast<const uint8_t*>(a->host_blocks[i]);
        SMO_REQUIRE(s.host[i], "streamer: null host block");
        s.code[i] = a->host_codes ? a->host_codes[i] : 0;
        SMO_REQUIRE(s.code[i] == 0 || s.code[i] == 1 || s.code[i] == 3 || s.code[i] == 4,
                    "streamer: host code must be 0 (raw), 1 (unary), 3 or 4");
        s.hbytes[i] = s.code[i] ? (a->host_bytes ? a->host_bytes[i] : 0) : s.blk;
        SMO_REQUIRE(s.hbytes[i] > 0 && s.hbytes[i] <= s.blk, "streamer: coded block needs 0 < host_bytes <= block_bytes");
        if (s.code[i]) s.cstride = std::max(s.cstride, size_t((s.hbytes[i] + 255) & ~uint64_t(255)));
      }
      // hot cache: the first blocks in (layer, expert) order, as the engine
      const int64_t cache_blocks = a->cache_bytes > 0 ? a->cache_bytes / int64_t(s.blk) : 0;
      s.cache.assign(n, -1);
      int placed = 0;
      for (size_t i = 0; i < n && placed < cache_blocks; ++i) s.cache[i] = s.slots * s.E + placed++;
      SMO_CUDA_CHECK(cudaMalloc(&s.pool, (size_t(s.slots) * s.E + placed) * s.blk));
      if (s.cstride) SMO_CUDA_CHECK(cudaMalloc(&s.cstage, size_t(s.slots) * s.E * s.cstride));
      SMO_CUDA_CHECK(cudaStreamCreateWithFlags(&s.copy, cudaStreamNonBlocking));
      s.ready.resize(size_t(s.slots));
      s.freed.resize(size_t(s.slots));
      for (int k = 0; k < s.slots; ++k) {
        SMO_CUDA_CHECK(cudaEventCreateWithFlags(&s.ready[size_t(k)], cudaEventDisableTiming));
        SMO_CUDA_CHECK(cudaEventCreateWithFlags(&s.freed[size_t(k)], cudaEventDisableTiming));
      }
      s.slot_layer.assign(size_t(s.slots), -1);
      s.pending.assign(size_t(s.slots), {});
      // cached blocks: staged once (coded ones expanded through the staging area)
      for (size_t i = 0; i < n; ++i) {
        if (s.cache[i] < 0) continue;
        uint8_t* dst = s.pool + size_t(s.cache[i]) * s.blk;
        if (s.code[i]) {
          SMO_CUDA_CHECK(cudaMemcpyAsync(s.cstage, s.host[i], s.hbytes[i], cudaMemcpyHostToDevice, s.copy));
          smo::expert_decode(s.cstage, s.blk / 2, s.code[i], dst, s.copy);
        } else {
          SMO_CUDA_CHECK(cudaMemcpyAsync(dst, s.host[i], s.blk, cudaMemcpyHostToDevice, s.copy));
        }
        SMO_CUDA_CHECK(cudaStreamSynchronize(s.copy));
      }
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

smo_status smo_streamer_destroy(smo_streamer* h) {
  return smo::run_guarded([&] {
    if (!h) return;
    smo::DeviceGuard dg(h->s.device);
    delete h;
  });
}

smo_status smo_streamer_enqueue_layer(smo_streamer* h, int32_t layer, const uint8_t* active) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(h && layer >= 0 && layer < h->s.L, "streamer: bad layer");
    smo::Streamer& s = h->s;
    smo::DeviceGuard dg(s.device);
    const int k = s.slot_of(layer);
    // the slot's previous layer must have been released by its consumer
    SMO_CUDA_CHECK(cudaStreamWaitEvent(s.copy, s.freed[size_t(k)], 0));
    s.pending[size_t(k)].clear();
    for (int e = 0; e < s.E; ++e) {
      const size_t i = s.idx(layer, e);
      if (s.cache[i] >= 0 || (active && !active[e])) continue;
      if (s.code[i]) {
        SMO_CUDA_CHECK(cudaMemcpyAsync(s.cstage + (size_t(k) * s.E + e) * s.cstride, s.host[i], s.hbytes[i],
                                       cudaMemcpyHostToDevice, s.copy));
        s.pending[size_t(k)].push_back(e);
      } else {
        SMO_CUDA_CHECK(cudaMemcpyAsync(s.slot_block(layer, e), s.host[i], s.blk, cudaMemcpyHostToDevice, s.copy));
      }
    }
    SMO_CUDA_CHECK(cudaEventRecord(s.ready[size_t(k)], s.copy));
    s.slot_layer[size_t(k)] = layer;
  });
}

smo_status smo_streamer_expert_ready_event(smo_streamer* h, int32_t layer, void** event) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(h && event && layer >= 0 && layer < h->s.L, "streamer: bad arguments");
    const int k = h->s.slot_of(layer);
    SMO_REQUIRE(h->s.slot_layer[size_t(k)] == layer, "streamer: layer not enqueued");
    *event = h->s.ready[size_t(k)];
  });
}

smo_status smo_streamer_wait_layer(smo_streamer* h, int32_t layer, smo_stream stream) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(h && layer >= 0 && layer < h->s.L, "streamer: bad layer");
    smo::Streamer& s = h->s;
    smo::DeviceGuard dg(s.device);
    const int k = s.slot_of(layer);
    SMO_REQUIRE(s.slot_layer[size_t(k)] == layer, "streamer: layer not enqueued");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    SMO_CUDA_CHECK(cudaStreamWaitEvent(st, s.ready[size_t(k)], 0));
    for (int code : {1, 3, 4}) {  // one expansion launch per code
      const void* src[64];
      void* dst[64];
      int n = 0;
      for (int e : s.pending[size_t(k)]) {
        if (s.code[s.idx(layer, e)] != code) continue;
        if (n == 64) {
          smo::expert_decode_blocks(src, dst, n, s.blk / 2, code, st);
          n = 0;
        }
        src[n] = s.cstage + (size_t(k) * s.E + e) * s.cstride;
        dst[n] = s.slot_block(layer, e);
        ++n;
      }
      smo::expert_decode_blocks(src, dst, n, s.blk / 2, code, st);
    }
    s.pending[size_t(k)].clear();
  });
}

smo_status smo_streamer_expert_ptr(smo_streamer* h, int32_t layer, int32_t expert, const void** out) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(h && out && layer >= 0 && layer < h->s.L && expert >= 0 && expert < h->s.E,
                "streamer: bad arguments");
    const smo::Streamer& s = h->s;
    const int cb = s.cache[s.idx(layer, expert)];
    *out = cb >= 0 ? s.pool + size_t(cb) * s.blk : s.slot_block(layer, expert);
  });
}

smo_status smo_streamer_release_layer(smo_streamer* h, int32_t layer, smo_stream stream) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(h && layer >= 0 && layer < h->s.L, "streamer: bad layer");
    smo::DeviceGuard dg(h->s.device);
    SMO_CUDA_CHECK(cudaEventRecord(h->s.freed[size_t(h->s.slot_of(layer))], reinterpret_cast<cudaStream_t>(stream)));
  });
}

}  // extern "C"
