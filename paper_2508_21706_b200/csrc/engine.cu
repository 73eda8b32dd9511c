#include <cstring>
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
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cctype>
#include <cstdio>

#include "engine.cuh"

namespace smo {

// every page back to the free list (lowest ids handed out first)
void Engine::bt_reset() {
  if (!paged) return;
  for (size_t i = 0; i < size_t(maxB) * max_pages; ++i) h_bt[i] = -1;
  free_pages.clear();
  for (int pg = num_pages - 1; pg >= 0; --pg) free_pages.push_back(pg);
  req_pages.assign(size_t(maxB), 0);
  bt_dirty = true;
}

// map pages for positions [0, len) of request r
void Engine::bt_ensure(int r, int64_t len) {
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

void Engine::bt_sync(cudaStream_t st) {
  if (!paged || !bt_dirty) return;
  SMO_CUDA_CHECK(cudaMemcpyAsync(d_bt, h_bt, size_t(maxB) * max_pages * 4, cudaMemcpyHostToDevice, st));
  bt_dirty = false;
}

int device_numa_node(int device) {
  if (const char* f = std::getenv("SMO_HOST_NUMA")) return std::atoi(f);  // -1: no placement
  struct stat sb {};
  if (stat("/sys/devices/system/node/node1", &sb) != 0) return -1;  // single-node host
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof(bus), device) != cudaSuccess) return -1;
  for (char* c = bus; *c; ++c) *c = char(std::tolower(*c));
  std::string path = std::string("/sys/bus/pci/devices/") + bus + "/numa_node";
  FILE* f = std::fopen(path.c_str(), "r");
  if (!f) {  // sysfs uses a 4-hex-digit domain; CUDA prints 8
    if (std::strlen(bus) > 12) f = std::fopen((std::string("/sys/bus/pci/devices/") + (bus + 4) + "/numa_node").c_str(), "r");
    if (!f) return -1;
  }
  int node = -1;
  if (std::fscanf(f, "%d", &node) != 1) node = -1;
  std::fclose(f);
  return node;
}

void* pinned_alloc(size_t bytes, int node, size_t* bytes_out) {
  *bytes_out = 0;
  if (node >= 0 && node < 64) {
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
    if (p != MAP_FAILED) {
      unsigned long mask = 1ul << node;
      const long rc = syscall(SYS_mbind, p, bytes, 2 /* MPOL_BIND */, &mask, 64ul, 0u);
      if (rc == 0 && cudaHostRegister(p, bytes, cudaHostRegisterPortable) == cudaSuccess) {
        *bytes_out = bytes;
        return p;
      }
      cudaGetLastError();
      munmap(p, bytes);
    }
  }
  void* hp = nullptr;
  if (cudaHostAlloc(&hp, bytes, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return hp;
}

void pinned_free(void* p, size_t numa_bytes) {
  if (!p) return;
  if (numa_bytes) {
    cudaHostUnregister(p);
    munmap(p, numa_bytes);
  } else {
    cudaFreeHost(p);
  }
}

// expand layer l's coded blocks (streamed into cstage) into its pool slot,
// on the compute stream after slot_ready(l)
void Engine::decode_slot(int l, cudaStream_t st) {
  if (tmode) return;  // tile-coded blocks are decoded inside K4-MoE
  const int s = l % slots;
  if (coded_streamed[size_t(l)].empty() && coded_cached[size_t(l)].empty()) return;
  SMO_CUDA_CHECK(cudaEventRecord(dec_ev[size_t(2 * l)], st));
  for (int bits : {1, 3, 4}) {  // one launch per code (blocks of a layer share it in practice)
    const void* src[64];
    void* dst[64];
    int n = 0;
    for (int le : coded_streamed[size_t(l)]) {
      if (code_bits(l, le) != bits) continue;
      if (n == 64) {
        expert_decode_blocks(src, dst, n, blk_elems, bits, st);
        n = 0;
      }
      src[n] = cstage + (size_t(s) * E_loc + le) * cblk_bytes;
      dst[n] = pool + (size_t(s) * E_loc + le) * blk_elems;
      step_codec_bytes += double(blk_csize[size_t(host_layer(l)) * E_loc + size_t(le)] + blk_bytes);
      ++n;
    }
    for (int le : coded_cached[size_t(l)]) {  // hot-cached in their code: source already in HBM
      if (code_bits(l, le) != bits) continue;
      if (n == 64) {
        expert_decode_blocks(src, dst, n, blk_elems, bits, st);
        n = 0;
      }
      src[n] = ccache + ccache_off[size_t(l) * E + size_t(owned[size_t(le)])];
      dst[n] = pool + (size_t(s) * E_loc + le) * blk_elems;
      step_codec_bytes += double(blk_csize[size_t(host_layer(l)) * E_loc + size_t(le)] + blk_bytes);
      ++n;
    }
    expert_decode_blocks(src, dst, n, blk_elems, bits, st);
  }
  SMO_CUDA_CHECK(cudaEventRecord(dec_ev[size_t(2 * l + 1)], st));
  step_dec_ev.push_back({dec_ev[size_t(2 * l)], dec_ev[size_t(2 * l + 1)]});
}

int Engine::expert_block(int l, const void* x_perm, int rows, int nexp, const int32_t* offsets, const int32_t* w_index,
                         const void* const* w_code, void* hb, float* y, int splits, int max_splits, cudaStream_t st) {
  (void)l;
  if (tmode)
    return moe_coded_launch(x_perm, rows, h, hi, nexp, offsets, w_code, hb, y, splits, max_splits, d_done, st, tfmt);
  return moe_launch(x_perm, rows, h, hi, nexp, offsets, pool, blk_bytes, pool_blocks, w_index, hb, y, splits,
                    max_splits, d_done, st);
}

void Engine::create() {
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
  SMO_REQUIRE(cfg.expert_init == SMO_INIT_UNIFORM || cfg.expert_init == SMO_INIT_GAUSSIAN, "engine: bad expert_init");
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
    batch_one = true;
    SMO_CUDA_CHECK(cudaEventCreateWithFlags(&route_ev, cudaEventDisableTiming));
    const char* f = std::getenv("SMO_B1_PREFETCH");
    b1_prefetch = !(f && f[0] == '0') && !(opt.ep_size > 1 || opt.nccl_comm);  // (1 GPU: global routing on host)
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
  host_numa = device_numa_node(opt.device);
  uint16_t* stage = dalloc<uint16_t>(blk_elems);
  xcomp = opt.compress_experts != 0;
  uint8_t* cenc = nullptr;
  int* d_ovf = nullptr;
  bool unary = false;
  if (xcomp) {
    cblk_bytes = expert_code_bytes(blk_elems, 4);  // staging stride: no block is kept coded above it
    const char* f = std::getenv("SMO_CODEC");
    unary = !(f && std::strcmp(f, "fixed") == 0);
    tmode = opt.compress_experts == 2 || opt.compress_experts == 3 || (f && std::strncmp(f, "tile", 4) == 0);
    tfmt = (opt.compress_experts == 3 || (f && std::strcmp(f, "tile3") == 0)) ? 3 : 2;
    const bool tile_ok = h % 128 == 0 && hi % 128 == 0;
    if (tmode) SMO_REQUIRE(tile_ok, "engine: the tile code needs h and h_i multiples of 128");
    cenc = dalloc<uint8_t>(std::max(tile_ok ? tcode_max_bytes(h, hi) : size_t(0),
                                    unary ? expert_code_bytes(blk_elems, 1) : cblk_bytes));
    // compress_experts = 1 without SMO_CODEC: the link code with fewer bytes on
    // this model's weights, probed on the first expert block — unary (the
    // geometric exponents of uniform-init blocks: 10.25 vs 10.42 bits/weight)
    // or the tile code (gaussian-like blocks: 11.0 vs 11.46)
    if (opt.compress_experts == 1 && !f && tile_ok && !owned.empty()) {
      const uint64_t base = tid::layer(0) + tid::kExpert + 3ull * owned[0];
      auto fill = cfg.expert_init == SMO_INIT_GAUSSIAN ? fill_normal : fill_uniform;
      fill(stage, size_t(hi) * h, cfg.seed, base + 0, 0, std::sqrt(3.0f / h), st);
      fill(stage + size_t(hi) * h, size_t(hi) * h, cfg.seed, base + 1, 0, std::sqrt(3.0f / h), st);
      fill(stage + 2 * size_t(hi) * h, size_t(h) * hi, cfg.seed, base + 2, 0, std::sqrt(3.0f / hi), st);
      SMO_CUDA_CHECK(cudaStreamSynchronize(st));
      const size_t tb = tcode_encode(stage, h, hi, cenc, st);
      const size_t t3b = tcode_encode(stage, h, hi, cenc, st, 3);
      expert_encode(stage, blk_elems, 1, cenc, d_ovf ? d_ovf : (d_ovf = dalloc<int>(1)), st);
      const size_t ub = expert_coded_size(cenc, blk_elems, 1);
      // When the hot cache holds every block, no block crosses the link and
      // the step is device-bound: a tile code decoded inside the expert
      // kernel, T3 (fixed 3-bit exponents, the fastest decode) if every block
      // fits in it, else T2 (profiles/r02h_t3.md). Otherwise the link binds:
      // the smaller code (unary for uniform-init, T2 for gaussian-like).
      auto all = [&](size_t per) {
        return 1.005 * double(L) * double(owned.size()) * double((per + 255) & ~size_t(255));
      };
      const double cache = double(opt.expert_cache_bytes);
      tmode = true;
      if (cache >= all(t3b)) {
        tfmt = 3;
      } else if (cache >= all(tb)) {
        tfmt = 2;
      } else {
        tmode = double(tb) < 0.99 * double(ub);
        tfmt = 2;
      }
    }
    if (!d_ovf) d_ovf = dalloc<int>(1);
    blk_coded.assign(size_t(host_alias) * E_loc, 0);
    blk_csize.assign(size_t(host_alias) * E_loc, 0);
  }
  for (int a = 0; a < host_alias; ++a) {
    size_t nb = 0;
    void* hp = pinned_alloc(blk_bytes * E_loc, host_numa, &nb);
    if (!hp)
      throw Error(SMO_CAPACITY, "engine: pinned host allocation of " + std::to_string(blk_bytes * E_loc) +
                                    " bytes failed; set host_alias_layers");
    host_bufs[a] = reinterpret_cast<uint16_t*>(hp);
    host_numa_bytes.push_back(nb);
    for (int e : owned) {
      const uint64_t base = tid::layer(a) + tid::kExpert + 3ull * e;
      auto fill = cfg.expert_init == SMO_INIT_GAUSSIAN ? fill_normal : fill_uniform;
      fill(stage, size_t(hi) * h, cfg.seed, base + 0, 0, std::sqrt(3.0f / h), st);
      fill(stage + size_t(hi) * h, size_t(hi) * h, cfg.seed, base + 1, 0, std::sqrt(3.0f / h), st);
      fill(stage + 2 * size_t(hi) * h, size_t(h) * hi, cfg.seed, base + 2, 0, std::sqrt(3.0f / hi), st);
      uint16_t* hdst = host_bufs[a] + size_t(local(e)) * blk_elems;
      bool coded = false;
      // the smallest code that holds the block: unary (variable length) when
      // it beats the 3-bit window, else 3 or 4 bits, else unary if still
      // within the staging stride, else raw bf16 — lossless in every case
      size_t ubytes = 0;
      if (tmode) {  // T2: always (lossless for any bits; raw tiles inside the code)
        SMO_CUDA_CHECK(cudaStreamSynchronize(st));
        const size_t tb = tcode_encode(stage, h, hi, cenc, st, tfmt);
        SMO_REQUIRE(tb <= blk_bytes, "engine: tile code of an expert block larger than its bf16 size");
        SMO_CUDA_CHECK(cudaMemcpy(hdst, cenc, tb, cudaMemcpyDeviceToHost));
        blk_coded[size_t(a) * E_loc + local(e)] = 2;
        blk_csize[size_t(a) * E_loc + local(e)] = tb;
        continue;
      }
      if (xcomp && unary) {
        SMO_CUDA_CHECK(cudaStreamSynchronize(st));
        expert_encode(stage, blk_elems, 1, cenc, d_ovf, st);
        ubytes = expert_coded_size(cenc, blk_elems, 1);
      }
      auto keep = [&](int bits, size_t cb) {
        SMO_CUDA_CHECK(cudaMemcpy(hdst, cenc, cb, cudaMemcpyDeviceToHost));
        blk_coded[size_t(a) * E_loc + local(e)] = uint8_t(bits);
        blk_csize[size_t(a) * E_loc + local(e)] = cb;
        coded = true;
      };
      // a fixed window code only where it is smaller than unary (and holds the block)
      for (int bits = 3; xcomp && !coded && bits <= 4; ++bits) {
        if (ubytes && expert_code_bytes(blk_elems, bits) >= ubytes) continue;
        SMO_CUDA_CHECK(cudaMemset(d_ovf, 0, sizeof(int)));
        expert_encode(stage, blk_elems, bits, cenc, d_ovf, st);
        int ovf = 0;
        SMO_CUDA_CHECK(cudaMemcpy(&ovf, d_ovf, sizeof(int), cudaMemcpyDeviceToHost));
        if (!ovf) keep(bits, expert_code_bytes(blk_elems, bits));
      }
      if (xcomp && !coded && ubytes && ubytes <= cblk_bytes) {
        expert_encode(stage, blk_elems, 1, cenc, d_ovf, st);
        keep(1, ubytes);
      }
      if (!coded) SMO_CUDA_CHECK(cudaMemcpy(hdst, stage, blk_bytes, cudaMemcpyDeviceToHost));
    }
  }

  // HBM pool: slots x E staging blocks + hot-expert cache. With the coded
  // transfer the cache keeps blocks in their link code (~1.56x more experts
  // per cache byte) and expands them into the layer's slot each step, like
  // a streamed block whose bytes are already in HBM (SMO_CODED_CACHE=0: bf16).
  cache_blk.assign(size_t(L) * E, -1);
  int placed = 0;
  {
    const char* f = std::getenv("SMO_CODED_CACHE");
    const bool coded_cache = xcomp && (tmode || !(f && f[0] == '0'));
    int64_t budget = std::max<int64_t>(opt.expert_cache_bytes, 0);
    size_t cc_bytes = 0;
    std::vector<std::pair<size_t, size_t>> cc_src;  // (l*E+e, offset)
    bool full = false;
    for (int l = 0; l < L && !full; ++l)
      for (int e : owned) {
        const size_t i = size_t(host_layer(l)) * E_loc + size_t(local(e));
        const bool coded = coded_cache && code_bits(l, local(e)) != 0;
        const int64_t cost = coded ? int64_t((blk_csize[i] + 255) & ~size_t(255)) : int64_t(blk_bytes);
        if (cost > budget) {
          full = true;
          break;
        }
        budget -= cost;
        if (coded) {
          cache_blk[size_t(l) * E + e] = kCachedCoded;
          cc_src.push_back({size_t(l) * E + e, cc_bytes});
          cc_bytes += size_t(cost);
        } else {
          cache_blk[size_t(l) * E + e] = slots * E_loc + placed;
          ++placed;
        }
      }
    coded_cached.assign(size_t(L), {});
    ccache_off.assign(size_t(L) * E, 0);
    if (cc_bytes) {
      ccache = dalloc<uint8_t>(cc_bytes);
      for (auto [le_idx, off] : cc_src) {
        const int l = int(le_idx / E), e = int(le_idx % E);
        const size_t i = size_t(host_layer(l)) * E_loc + size_t(local(e));
        SMO_CUDA_CHECK(cudaMemcpy(ccache + off, host_bufs[host_layer(l)] + size_t(local(e)) * blk_elems, blk_csize[i],
                                  cudaMemcpyHostToDevice));
        ccache_off[le_idx] = off;
        coded_cached[size_t(l)].push_back(local(e));
      }
    }
  }
  if (tmode) {  // staging stride: the largest tile code (16-B multiples), no bf16 slots
    cblk_bytes = 256;
    for (size_t b : blk_csize) cblk_bytes = std::max(cblk_bytes, (b + 255) & ~size_t(255));
  }
  pool_blocks = (tmode ? 0 : slots * E_loc) + placed;
  pool = dalloc<uint16_t>(size_t(pool_blocks) * blk_elems);
  coded_streamed.assign(size_t(L), {});
  if (xcomp) cstage = dalloc<uint8_t>(size_t(slots) * E_loc * cblk_bytes);
  for (int l = 0; l < L; ++l)
    for (int e : owned) {
      const int cb = cache_blk[size_t(l) * E + e];
      if (cb < 0) continue;  // streamed, or cached in its code (expanded per step)
      const uint16_t* hsrc = host_bufs[host_layer(l)] + size_t(local(e)) * blk_elems;
      if (const int bits = code_bits(l, local(e))) {
        SMO_CUDA_CHECK(cudaMemcpy(cenc, hsrc, blk_csize[size_t(host_layer(l)) * E_loc + size_t(local(e))],
                                  cudaMemcpyHostToDevice));
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
  if (tmode) {  // code block of (layer, expert): its staging slot, or the coded hot cache
    std::vector<const void*> wc(size_t(L) * E, nullptr);
    for (int l = 0; l < L; ++l)
      for (int e : owned) {
        const size_t i = size_t(l) * E + size_t(e);
        wc[i] = cache_blk[i] == kCachedCoded ? static_cast<const void*>(ccache + ccache_off[i])
                                             : static_cast<const void*>(cstage + (size_t(l % slots) * E_loc + local(e)) *
                                                                                     cblk_bytes);
      }
    d_w_code = dalloc<const void*>(wc.size());
    SMO_CUDA_CHECK(cudaMemcpy(d_w_code, wc.data(), wc.size() * sizeof(void*), cudaMemcpyHostToDevice));
    if (ep_on) {
      std::vector<const void*> wl(size_t(L) * E_loc);
      for (int l = 0; l < L; ++l)
        for (int le = 0; le < E_loc; ++le) wl[size_t(l) * E_loc + le] = wc[size_t(l) * E + le * P + opt.ep_rank];
      d_w_code_loc = dalloc<const void*>(wl.size());
      SMO_CUDA_CHECK(cudaMemcpy(d_w_code_loc, wl.data(), wl.size() * sizeof(void*), cudaMemcpyHostToDevice));
    }
  }
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
  offsets = dalloc<int32_t>(size_t(E + 1) * kMaxMb);  // one [E+1] region per micro-batch
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
    {
      const size_t ds = ept->direct_slot();
      const char* f = std::getenv("SMO_EP_STAGED");
      ep_direct = !(f && f[0] == '1') && ds >= std::max(blk_d, size_t(C) * h * 4) && ds % (size_t(h) * 4) == 0;
      ep_rows = ep_direct ? int(ds / (size_t(h) * 4)) : C;
    }
    if (!ep_direct) {
      ep_send = dalloc<uint8_t>(size_t(PR) * blk_d);
      ep_recv = dalloc<uint8_t>(size_t(PR) * blk_d);
      ep_sendback = dalloc<float>(size_t(PR) * C * h);
      ep_recvback = dalloc<float>(size_t(PR) * C * h);
    }
    xl = dalloc<uint16_t>(size_t(PR) * C * h);
    yl = dalloc<float>(size_t(4) * PR * C * h);  // room for the fused kernel's down slices
    hbuf = dalloc<uint16_t>(size_t(PR) * C * hi);
  } else {
    hbuf = dalloc<uint16_t>(size_t(P) * hi);
  }
  {
    const char* sp = std::getenv("SMO_STEP_PREFETCH");
    step_pf = !(sp && sp[0] == '0');
    const char* f = std::getenv("SMO_MOE_FUSED");
    moe_fused = tmode || !(f && f[0] == '0');  // the tile-coded expert kernel is the fused one
  }
  // fused MoE down splits from the GLOBAL shapes (every EP rank uses the
  // same S, so expert parallelism reproduces one GPU bit for bit)
  moe_splits = moe_fused ? pick_moe_splits(maxT * K, h, hi, E, 4) : 1;
  ybuf = dalloc<float>(size_t(moe_splits) * P * h);
  d_done = dalloc<int>(128);
  SMO_CUDA_CHECK(cudaMemset(d_done, 0, 128 * sizeof(int)));  // the expert kernel leaves its counters zero
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
    host_jobs.resize(size_t(L) * kMaxMb);
    ensure_async_host();
  }
  if (opt.draft_cpu_kv) {  // drafter CPU part (f1): host drafter K/V, q / attention staging
    SMO_REQUIRE(dL > 0, "engine: draft_cpu_kv needs a drafter (draft_layers)");
    SMO_REQUIRE(!paged, "engine: draft_cpu_kv needs contiguous K/V (kv_pages = 0)");
    draft_cpu = true;
    for (int l = 0; l < dL; ++l) {
      dkc_h.push_back(halloc_mapped<uint16_t>(kv_elems()));
      dvc_h.push_back(halloc_mapped<uint16_t>(kv_elems()));
    }
    dq_h = halloc_mapped<uint16_t>(size_t(maxB) * nq * d);
    da_h = halloc_mapped<uint16_t>(size_t(maxB) * nq * d);
    dpos_h = halloc_mapped<int32_t>(maxB);
    dmask_h = halloc_mapped<uint64_t>(maxB);
    for (int r = 0; r < maxB; ++r) dmask_h[r] = 1;
    if (!cpu_pool) cpu_pool.reset(new CpuPool(int(std::max(1u, std::thread::hardware_concurrency()))));
    ensure_async_host();
  }
  set_micro_batches(opt.micro_batches);
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
  ev.resize(8 + size_t(L) * 8 * kMaxMb);  // per layer: 8 events of micro-batch 0, then 8 per further one
  for (auto& e : ev) SMO_CUDA_CHECK(cudaEventCreate(&e));
  draft_ev.resize(size_t(maxN) + 1);
  for (auto& e : draft_ev) SMO_CUDA_CHECK(cudaEventCreate(&e));
  join_ev.resize(size_t(maxN));
  for (auto& e : join_ev) SMO_CUDA_CHECK(cudaEventCreate(&e));
  dec_ev.resize(size_t(2) * L);
  for (auto& e : dec_ev) SMO_CUDA_CHECK(cudaEventCreate(&e));
  SMO_CUDA_CHECK(cudaDeviceSynchronize());
}

void Engine::fill_prefix(const int32_t* prefix_host, int b) {
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

// Stream layer l's non-cached owned experts into slot l % slots. Host and
// slot blocks are in local order, so runs of consecutive local experts go
// out as one copy (a whole layer when nothing is cached: 2.8 GB for 8x7B).
// active (optional, BATCH_ONE): per local expert, 0 = not routed to -> not streamed
double Engine::enqueue_h2d(int l, cudaEvent_t t0, cudaEvent_t t1, const uint8_t* active) {
  const int s = l % slots;
  // while capturing a graph the first `slots` layers' release events belong
  // to the previous iteration (outside the graph; replays are serialised)
  if (!(capturing && l < slots)) SMO_CUDA_CHECK(cudaStreamWaitEvent(copy, slot_free[s], 0));
  if (t0) SMO_CUDA_CHECK(cudaEventRecord(t0, copy));
  double bytes = 0;
  const uint16_t* hb = host_bufs[host_layer(l)];
  auto streamed = [&](int le) {
    return cache_blk[size_t(l) * E + owned[size_t(le)]] == -1 && (!active || active[le]);
  };
  coded_streamed[size_t(l)].clear();
  // BATCH_ONE link-gap prefetch of this layer: only the remainders are left
  const bool spec = spec_layer == l;
  auto staged = [&](int q) { return spec ? spec_done[size_t(q)] : size_t(0); };
  if (xcomp || spec) {
    // coded blocks into cstage (expanded by decode_slot), raw ones straight into the slot
    for (int q = 0; q < E_loc; ++q) {
      if (!streamed(q) || (!xcomp && staged(q) == 0)) continue;
      const bool coded = code_bits(l, q) != 0;
      const size_t full = coded ? blk_csize[size_t(host_layer(l)) * E_loc + size_t(q)] : blk_bytes;
      const size_t done = staged(q);
      uint8_t* dstp = coded ? cstage + (size_t(s) * E_loc + q) * cblk_bytes
                            : reinterpret_cast<uint8_t*>(pool + (size_t(s) * E_loc + q) * blk_elems);
      if (full > done)
        SMO_CUDA_CHECK(cudaMemcpyAsync(dstp + done, reinterpret_cast<const uint8_t*>(hb + size_t(q) * blk_elems) + done,
                                       full - done, cudaMemcpyHostToDevice, copy));
      bytes += double(full - done);
      if (coded) coded_streamed[size_t(l)].push_back(q);
    }
  }
  spec_layer = spec ? -1 : spec_layer;
  int le = xcomp ? E_loc : 0;
  while (le < E_loc) {
    if (!streamed(le) || staged(le) > 0) {  // (partly prefetched raw blocks were completed above)
      ++le;
      continue;
    }
    int le2 = le;
    while (le2 + 1 < E_loc && streamed(le2 + 1) && staged(le2 + 1) == 0) ++le2;
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

void Engine::snap(const char* name, int layer, const void* src, size_t bytes, cudaStream_t st) {
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
double Engine::moe_ep(int l, int T, cudaStream_t st, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* h2d_ev) {
  double streamed = 0;
  const int PT = T * K;
  const int rank = opt.ep_rank;
  ep_pos(oid, pos, offsets, PT, E_loc, ep_rows, pos_ep, st);
  if (ep_direct) {  // dispatch kernel stores each block into its owner's mailbox
    const uint8_t* recv = nullptr;
    uint8_t* const* dests = ept->direct_begin(st, &recv);
    ep_pack(xp, offsets, P, E_loc, C, h, blk_d, nullptr, st, dests);
    ept->direct_exchange(st);
    ep_unpack(recv, P, E_loc, C, h, ept->direct_slot(), xl, offsets_l, back, st);
    ept->direct_done(st);
  } else {
    ep_pack(xp, offsets, P, E_loc, C, h, blk_d, ep_send, st);
    ept->alltoall(rank, ep_send, ep_recv, blk_d, st);
    ep_unpack(ep_recv, P, E_loc, C, h, blk_d, xl, offsets_l, back, st);
  }
  if (batch_one) {
    // BATCH_ONE with expert parallelism: the rows every rank routed to this
    // rank's experts are known once the dispatch exchange landed; stream
    // only the local experts that received any (optimizer.hpp:81-96)
    SMO_CUDA_CHECK(cudaMemcpyAsync(h_offsets, offsets_l, size_t(E_loc + 1) * 4, cudaMemcpyDeviceToHost, st));
    SMO_CUDA_CHECK(cudaEventRecord(route_ev, st));
    SMO_CUDA_CHECK(cudaEventSynchronize(route_ev));
    std::vector<uint8_t> act(size_t(E_loc), 0);
    for (int le = 0; le < E_loc; ++le) act[size_t(le)] = h_offsets[le + 1] > h_offsets[le] ? 1 : 0;
    streamed += enqueue_h2d(l, tev(l * 8 + 0), tev(l * 8 + 1), act.data());
    if (h2d_ev) h2d_ev->push_back({tev(l * 8 + 0), tev(l * 8 + 1)});
  }
  SMO_CUDA_CHECK(cudaEventRecord(tev(l * 8 + 7), st));
  SMO_CUDA_CHECK(cudaStreamWaitEvent(st, slot_ready[l % slots], 0));
  decode_slot(l, st);
  SMO_CUDA_CHECK(cudaEventRecord(tev(l * 8 + 4), st));
  int splits = 1;
  if (moe_fused) {
    expert_block(l, xl, P * C, E_loc, offsets_l, d_w_index_loc + size_t(l) * E_loc,
                 tmode ? d_w_code_loc + size_t(l) * E_loc : nullptr, hbuf, yl, moe_splits, 4, st);
    splits = moe_splits;
  } else {
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
  }
  SMO_CUDA_CHECK(cudaEventRecord(slot_free[l % slots], st));
  if (ep_direct) {  // combine rows stored straight into the source ranks' mailboxes
    const uint8_t* recv = nullptr;
    uint8_t* const* dests = ept->direct_begin(st, &recv);
    ep_pack_back(yl, back, offsets_l, E_loc, h, nullptr, st, splits, size_t(P) * C * h, dests, C);
    ept->direct_exchange(st);
    unpermute_combine(reinterpret_cast<const float*>(recv), pos_ep, rw, T, K, h, x, st);
    ept->direct_done(st);
  } else {
    ep_pack_back(yl, back, offsets_l, E_loc, h, ep_sendback, st, splits, size_t(P) * C * h);
    ept->alltoall(rank, ep_sendback, ep_recvback, size_t(C) * h * sizeof(float), st);
    unpermute_combine(ep_recvback, pos_ep, rw, T, K, h, x, st);
  }
  return streamed;
}

void Engine::verify(const smo_verify_batch& in, smo_verify_output& out, cudaStream_t st) {
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

// BATCH_ONE: from the previous step's per-layer copy events, the link idle
// time between layer l's copies and layer l+1's becomes the prefetch budget
// after layer l (90 % of the gap). A prefetch longer than the true gap
// delays layer l+1's copies, so the measured gap is then the prefetch
// itself and the budget shrinks; a shorter one leaves the true gap visible.
void Engine::b1_update_budget() {
  b1_budget.assign(size_t(L), 0.0);
  if (!b1_prefetch || !b1_measured) return;
  b1_measured = false;
  // the previous step's last copies: this step's copies queue behind them on
  // the same stream anyway, and BATCH_ONE synchronises the host per layer
  if (cudaEventSynchronize(tev((L - 1) * 8 + 1)) != cudaSuccess) return;
  double busy = 0, bytes = 0;
  for (int l = 0; l < L; ++l) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, tev(l * 8 + 0), tev(l * 8 + 1)) != cudaSuccess) return;
    busy += ms * 1e-3;
    bytes += layer_bytes[size_t(l)];
  }
  if (busy <= 0 || bytes <= 0) return;
  const double bw = bytes / busy;
  for (int l = 0; l + 1 < L; ++l) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, tev(l * 8 + 1), tev((l + 1) * 8 + 0)) != cudaSuccess) continue;
    b1_budget[size_t(l)] = std::max(0.0, 0.9 * ms * 1e-3 * bw);
  }
}

// After layer l's copies (BATCH_ONE): stage prefixes of layer l+1's blocks,
// the experts most routed at layer l first, up to the budget.
double Engine::b1_prefetch_step(int l, cudaStream_t copy_st) {
  spec_layer = -1;
  if (!b1_prefetch || l + 1 >= L || b1_budget.empty() || b1_budget[size_t(l)] <= 0) return 0;
  const int ln = l + 1, s = ln % slots;
  // a guessed expert is routed at layer l+1 with probability ~ the fraction
  // of experts layer l routed to; below one half the wasted prefixes cost
  // more than the gap buys (measured: DeepSeek-V2-Lite shape at b = 1)
  int used = 0;
  for (int q = 0; q < E_loc; ++q) used += h_offsets[owned[size_t(q)] + 1] > h_offsets[owned[size_t(q)]] ? 1 : 0;
  if (2 * used < E_loc) return 0;
  std::vector<int> order;
  for (int q = 0; q < E_loc; ++q)
    if (cache_blk[size_t(ln) * E + owned[size_t(q)]] == -1) order.push_back(q);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    const int ea = owned[size_t(a)], eb = owned[size_t(b)];
    return h_offsets[ea + 1] - h_offsets[ea] > h_offsets[eb + 1] - h_offsets[eb];
  });
  SMO_CUDA_CHECK(cudaStreamWaitEvent(copy_st, slot_free[s], 0));
  spec_done.assign(size_t(E_loc), 0);
  double left = b1_budget[size_t(l)], bytes = 0;
  const uint8_t* hb = reinterpret_cast<const uint8_t*>(host_bufs[host_layer(ln)]);
  for (int q : order) {
    if (left < 4096) break;
    const bool coded = code_bits(ln, q) != 0;
    const size_t full = coded ? blk_csize[size_t(host_layer(ln)) * E_loc + size_t(q)] : blk_bytes;
    const size_t nb = std::min(full, size_t(left) & ~size_t(4095));
    uint8_t* dstp = coded ? cstage + (size_t(s) * E_loc + q) * cblk_bytes
                          : reinterpret_cast<uint8_t*>(pool + (size_t(s) * E_loc + q) * blk_elems);
    SMO_CUDA_CHECK(cudaMemcpyAsync(dstp, hb + size_t(q) * blk_bytes, nb, cudaMemcpyHostToDevice, copy_st));
    spec_done[size_t(q)] = nb;
    left -= double(nb);
    bytes += double(nb);
  }
  spec_layer = ln;
  return bytes;
}

void Engine::begin_step(cudaStream_t st, bool prefetch) {
  if (!prefetch && batch_one) b1_update_budget();
  spec_layer = -1;
  SMO_CUDA_CHECK(cudaEventRecord(ev[0], st));
  // order the copy stream after the step start (so H2D timing is step-relative)
  SMO_CUDA_CHECK(cudaStreamWaitEvent(copy, ev[0], 0));
  step_h2d_bytes = 0;
  step_h2d_ev.clear();
  step_dec_ev.clear();
  step_codec_bytes = 0;
  std::fill(layer_bytes.begin(), layer_bytes.end(), 0.0);
  std::fill(layer_raw_bytes.begin(), layer_raw_bytes.end(), 0.0);
  const bool have_pf = next_pf && !capturing;  // (a graph must contain its own copies)
  next_pf = false;
  for (int l = 0; prefetch && l < std::min(slots, L); ++l) {
    if (have_pf) {  // already streaming since the previous step's end
      step_h2d_bytes += pf_bytes[size_t(l)];
      layer_bytes[size_t(l)] = pf_bytes[size_t(l)];
      layer_raw_bytes[size_t(l)] = pf_raw[size_t(l)];
      step_h2d_ev.push_back({pf_ev[size_t(2 * l)], pf_ev[size_t(2 * l + 1)]});
      continue;
    }
    step_h2d_bytes += enqueue_h2d(l, tev(l * 8 + 0), tev(l * 8 + 1));
    step_h2d_ev.push_back({tev(l * 8 + 0), tev(l * 8 + 1)});
  }
}

void Engine::prefetch_next_step() {
  if (!step_pf || batch_one || capturing || L <= slots) return;
  const int n = std::min(slots, L);
  if (pf_ev.empty()) {
    pf_ev.resize(size_t(2 * slots));
    for (auto& e : pf_ev) SMO_CUDA_CHECK(cudaEventCreate(&e));
    pf_bytes.assign(size_t(slots), 0.0);
    pf_raw.assign(size_t(slots), 0.0);
  }
  // this step's per-layer byte accounting of layers [0, n) stays as measured
  std::vector<double> lb(layer_bytes.begin(), layer_bytes.begin() + n), lr(layer_raw_bytes.begin(),
                                                                            layer_raw_bytes.begin() + n);
  for (int l = 0; l < n; ++l) {
    pf_bytes[size_t(l)] = enqueue_h2d(l, pf_ev[size_t(2 * l)], pf_ev[size_t(2 * l + 1)]);
    pf_raw[size_t(l)] = layer_raw_bytes[size_t(l)];
  }
  std::copy(lb.begin(), lb.end(), layer_bytes.begin());
  std::copy(lr.begin(), lr.end(), layer_raw_bytes.begin());
  next_pf = true;
}

// The target verification DAG on device inputs: tokens [b*n], parent
// [b*n] or null, prefix [b]; results in d_acc / d_bonus / d_keep / target.
// With m micro-batches (requests [j*b/m, (j+1)*b/m)) every stage of a layer
// is issued for all micro-batches before the next stage — the stage-major
// order of build_target_dag (pipeline.hpp:167-170) — and every micro-batch's
// GPU_MOE waits on the layer's single expert transfer.
void Engine::verify_core(int b, int n, const int32_t* tokens, const int32_t* parent, const int32_t* prefix, int max_prefix,
                 cudaStream_t st) {
  const int T = b * n;
  const int M = std::max(1, std::min(mb, b));
  last_mb = M;
  cudaEvent_t e_end = ev[1];
  double h2d_bytes = step_h2d_bytes;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> h2d_ev = step_h2d_ev, attn_ev, moe_ev;
  build_mask(parent, b, n, d_mask, st);
  embed(tokens, embed_w, T, h, x, st);
  const bool async_cpu = attn_cpu && !capturing;
  if (attn_cpu) {  // prefix lengths and the mask to the host once per step
    SMO_CUDA_CHECK(cudaMemcpyAsync(prefix_host, prefix, size_t(b) * 4, cudaMemcpyDeviceToHost, st));
    SMO_CUDA_CHECK(cudaMemcpyAsync(mask_host, d_mask, size_t(T) * 8, cudaMemcpyDeviceToHost, st));
  }
  // micro-batch j: requests [r0, r0 + bj), rows [R0, R0 + Tj)
  struct Mb {
    int r0, bj, R0, Tj;
  };
  std::vector<Mb> mbs;
  for (int j = 0; j < M; ++j) {
    const int r0 = j * b / M, r1 = (j + 1) * b / M;
    mbs.push_back({r0, r1 - r0, r0 * n, (r1 - r0) * n});
  }
  const size_t kv_req = paged ? 0 : size_t(nkv) * s_max * d;  // cache elements per request (contiguous)
  const int PT = T * K;  // (token, slot) pairs
  std::vector<uint32_t> seq(size_t(M), 0);
  for (int l = 0; l < L; ++l) {
    Layer& ly = layers[l];
    const int32_t* btl = bt();
    // ---- GPU_OTHER1: RMSNorm -> QKV -> RoPE + K/V append
    for (int j = 0; j < M; ++j) {
      const Mb& m = mbs[size_t(j)];
      SMO_CUDA_CHECK(cudaEventRecord(mev(l, j, 6), st));
      if (j == 0) snap("x_in", l, x, size_t(T) * h * 4, st);
      rmsnorm(x + size_t(m.R0) * h, ones, m.Tj, h, cfg.rms_eps, xn + size_t(m.R0) * h, st);
      if (j == M - 1) snap("xn1", l, xn, size_t(T) * h * 2, st);
      smo_gemm_args g{};
      g.x = xn + size_t(m.R0) * h;
      g.rows = m.Tj;
      g.K = h;
      g.N = qkv_w;
      g.groups = 1;
      g.max_rows_per_group = m.Tj;
      g.w = ly.wqkv;
      g.w_pool_blocks = 1;
      g.epilogue = SMO_EPI_BF16;
      g.out = qkv + size_t(m.R0) * qkv_w;
      g.ldo = qkv_w;
      g.workspace = gemm_ws;
      g.workspace_bytes = gemm_ws_bytes;
      gemm_launch(g, st);
      uint16_t* q_dst = (attn_cpu ? q_host : q) + size_t(m.R0) * nq * d;
      rope_append(qkv + size_t(m.R0) * qkv_w, prefix + m.r0, parent ? parent + m.R0 : nullptr, m.bj, n, nq, nkv, d,
                  s_max, cfg.rope_theta, q_dst, ly.kc + size_t(m.r0) * kv_req, ly.vc + size_t(m.r0) * kv_req, st,
                  btl ? btl + size_t(m.r0) * max_pages : nullptr, max_pages);
      if (j == M - 1) snap("q", l, attn_cpu ? q_host : q, size_t(T) * nq * d * 2, st);
      SMO_CUDA_CHECK(cudaEventRecord(mev(l, j, 2), st));
      if (attn_cpu) {
        HostAttn& hj = host_jobs[size_t(l) * kMaxMb + size_t(j)];
        hj.pool = cpu_pool.get();
        hj.job = CpuAttnJob{q_host + size_t(m.R0) * nq * d, ly.kc + size_t(m.r0) * kv_req,
                            ly.vc + size_t(m.r0) * kv_req, mask_host + m.R0, prefix_host + m.r0,
                            attn_host + size_t(m.R0) * nq * d, m.bj, n, nq, nkv, d, s_max, 1};
        if (async_cpu) {  // the host starts as soon as this micro-batch's q is written
          seq[size_t(j)] = ++host_seq;
          async_host.push({hj.job, hj.pool, seq[size_t(j)]});
          signal_host_ready(seq[size_t(j)], st);
        }
      }
    }
    // ---- attention (K1 on HBM, or the host job)
    for (int j = 0; j < M; ++j) {
      const Mb& m = mbs[size_t(j)];
      if (attn_cpu) {
        HostAttn& hj = host_jobs[size_t(l) * kMaxMb + size_t(j)];
        if (async_cpu) wait_host_flag(seq[size_t(j)], st);
        else SMO_CUDA_CHECK(cudaLaunchHostFunc(st, host_attn_cb, &hj));
        // SM loads of the mapped host output, not a copy-engine H2D copy: the
        // H2D engine is busy with the expert stream (a 1.8 GB layer copy)
        // and would queue this behind it
        copy_from_mapped(attn + size_t(m.R0) * nq * d, attn_host + size_t(m.R0) * nq * d, size_t(m.Tj) * nq * d * 2,
                         st);
      } else {
        smo_attn_args a{};
        a.q = q + size_t(m.R0) * nq * d;
        a.k_cache = ly.kc + size_t(m.r0) * kv_req;
        a.v_cache = ly.vc + size_t(m.r0) * kv_req;
        a.block_table = btl ? btl + size_t(m.r0) * max_pages : nullptr;
        a.max_pages = max_pages;
        a.num_pages = num_pages;
        a.mask = d_mask + m.R0;
        a.prefix_len = prefix + m.r0;
        a.out = attn + size_t(m.R0) * nq * d;
        a.b = m.bj;
        a.n = n;
        a.n_q = nq;
        a.n_kv = nkv;
        a.d = d;
        a.s_max = s_max;
        a.max_prefix = max_prefix;
        a.workspace = attn_ws;
        a.workspace_bytes = attn_ws_bytes;
        attention_launch(a, st);
      }
      SMO_CUDA_CHECK(cudaEventRecord(mev(l, j, 3), st));
      attn_ev.push_back({mev(l, j, 2), mev(l, j, 3)});
    }
    snap("attn", l, attn, size_t(T) * nq * d * 2, st);
    // ---- GPU_OTHER2: O-proj (+residual) -> RMSNorm -> router -> permute (-> shared expert)
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
    for (int j = 0; j < M; ++j) {
      const Mb& m = mbs[size_t(j)];
      float* xj = x + size_t(m.R0) * h;
      uint16_t* xnj = xn + size_t(m.R0) * h;
      smo_gemm_args g{};
      g.x = attn + size_t(m.R0) * nq * d;
      g.rows = m.Tj;
      g.K = nq * d;
      g.N = h;
      g.groups = 1;
      g.max_rows_per_group = m.Tj;
      g.w = ly.wo;
      g.w_pool_blocks = 1;
      g.epilogue = SMO_EPI_F32_ADD;
      g.out = xj;
      g.ldo = h;
      g.workspace = gemm_ws;
      g.workspace_bytes = gemm_ws_bytes;
      gemm_launch(g, st);
      rmsnorm(xj, ones, m.Tj, h, cfg.rms_eps, xnj, st);
      if (j == M - 1) snap("xn2", l, xn, size_t(T) * h * 2, st);
      const size_t p0 = size_t(m.R0) * K;  // first (token, slot) pair of the micro-batch
      int32_t* offj = offsets + size_t(j) * (E + 1);
      router_topk(xnj, ly.router, m.Tj, h, E, K, rlog ? rlog + size_t(m.R0) * E : nullptr, ids + p0, rw + p0, st);
      if (ep_on) {  // owner-major order: rows bound for one rank are contiguous
        ep_remap(ids, T * K, P, E_loc, oid, st);
        permute(oid, T, K, E, xn, h, offsets, perm, pos, xp, st);
      } else {
        permute(ids + p0, m.Tj, K, E, xnj, h, offj, perm + p0, pos + p0, xp + p0 * h, st);
      }
      if (j == M - 1) {
        snap("ids", l, ids, size_t(PT) * 4, st);
        snap("weights", l, rw, size_t(PT) * 4, st);
        snap("offsets", l, offsets, size_t(E + 1) * 4, st);
        snap("pos", l, pos, size_t(PT) * 4, st);
      }
      if (batch_one && !ep_on) {
        // BATCH_ONE (optimizer.hpp:81-96): wait for this layer's routing, then
        // stream only the experts its tokens selected
        SMO_CUDA_CHECK(cudaMemcpyAsync(h_offsets, offsets, size_t(E + 1) * 4, cudaMemcpyDeviceToHost, st));
        SMO_CUDA_CHECK(cudaEventRecord(route_ev, st));
        SMO_CUDA_CHECK(cudaEventSynchronize(route_ev));
        std::vector<uint8_t> act(size_t(E_loc), 0);
        for (int e = 0; e < E; ++e) act[size_t(local(e))] = h_offsets[e + 1] > h_offsets[e] ? 1 : 0;
        h2d_bytes += enqueue_h2d(l, tev(l * 8 + 0), tev(l * 8 + 1), act.data());
        h2d_ev.push_back({tev(l * 8 + 0), tev(l * 8 + 1)});
        const double pf = b1_prefetch_step(l, copy);  // fills the link while layer l+1 is routed
        h2d_bytes += pf;  // counted in the step's link bytes (wasted when the expert goes unrouted)
      }
      if (cfg.shared_inter > 0) {
        // always-on shared expert (config 4): x += SwiGLU_shared(xn2); its
        // weights are resident, so it runs before the wait for streamed experts
        smo_gemm_args gs{};
        gs.x = xnj;
        gs.rows = m.Tj;
        gs.K = h;
        gs.N = cfg.shared_inter;
        gs.groups = 1;
        gs.max_rows_per_group = m.Tj;
        gs.w = ly.ws1;
        gs.w_up = ly.ws3;
        gs.w_pool_blocks = 1;
        gs.epilogue = SMO_EPI_SWIGLU;
        gs.out = hs + size_t(m.R0) * cfg.shared_inter;
        gs.ldo = cfg.shared_inter;
        gemm_launch(gs, st);
        gs = smo_gemm_args{};
        gs.x = hs + size_t(m.R0) * cfg.shared_inter;
        gs.rows = m.Tj;
        gs.K = cfg.shared_inter;
        gs.N = h;
        gs.groups = 1;
        gs.max_rows_per_group = m.Tj;
        gs.w = ly.ws2;
        gs.w_pool_blocks = 1;
        gs.epilogue = SMO_EPI_F32_ADD;
        gs.out = xj;
        gs.ldo = h;
        gs.workspace = gemm_ws;
        gs.workspace_bytes = gemm_ws_bytes;
        gemm_launch(gs, st);
      }
      SMO_CUDA_CHECK(cudaEventRecord(mev(l, j, 7), st));
    }
    // ---- GPU_MOE: every micro-batch waits on this layer's expert transfer
    for (int j = 0; j < M; ++j) {
      const Mb& m = mbs[size_t(j)];
      if (ep_on) {
        h2d_bytes += moe_ep(l, T, st, &h2d_ev);
        SMO_CUDA_CHECK(cudaEventRecord(tev(l * 8 + 5), st));
      } else {
        if (j == 0) {
          SMO_CUDA_CHECK(cudaStreamWaitEvent(st, slot_ready[l % slots], 0));
          decode_slot(l, st);  // coded expert blocks -> bf16 slot (compress_experts)
        }
        SMO_CUDA_CHECK(cudaEventRecord(mev(l, j, 4), st));
        const size_t p0 = size_t(m.R0) * K;
        const int PTj = m.Tj * K;
        const int32_t* offj = offsets + size_t(j) * (E + 1);
        float* yj = ybuf + size_t(moe_splits) * p0 * h;  // this micro-batch's [splits][PTj][h] region
        if (moe_fused) {
          expert_block(l, xp + p0 * h, PTj, E, offj, d_w_index + size_t(l) * E,
                       tmode ? d_w_code + size_t(l) * E : nullptr, hbuf + p0 * hi, yj, moe_splits, moe_splits, st);
          // GPU_MOE = the expert kernel itself (the bench's kernel roofline)
          SMO_CUDA_CHECK(cudaEventRecord(mev(l, j, 5), st));
          if (j == M - 1) SMO_CUDA_CHECK(cudaEventRecord(slot_free[l % slots], st));
          unpermute_combine(yj, pos + p0, rw + p0, m.Tj, K, h, x + size_t(m.R0) * h, st, moe_splits,
                            size_t(PTj) * h);
        } else {
          smo_gemm_args g{};
          g.x = xp + p0 * h;
          g.rows = PTj;
          g.K = h;
          g.N = hi;
          g.groups = E;
          g.row_offsets = offj;
          g.max_rows_per_group = m.Tj;  // a token selects an expert at most once
          g.w = pool;
          g.w_up = pool + size_t(hi) * h;
          g.w_block_stride = blk_bytes;
          g.w_pool_blocks = pool_blocks;
          g.w_index = d_w_index + size_t(l) * E;
          g.epilogue = SMO_EPI_SWIGLU;
          g.out = hbuf + p0 * hi;
          g.ldo = hi;
          gemm_launch(g, st);
          g = smo_gemm_args{};
          g.x = hbuf + p0 * hi;
          g.rows = PTj;
          g.K = hi;
          g.N = h;
          g.groups = E;
          g.row_offsets = offj;
          g.max_rows_per_group = m.Tj;
          g.w = pool + 2 * size_t(hi) * h;
          g.w_block_stride = blk_bytes;
          g.w_pool_blocks = pool_blocks;
          g.w_index = d_w_index + size_t(l) * E;
          g.epilogue = SMO_EPI_F32;
          g.out = yj;
          g.ldo = h;
          gemm_launch(g, st);
          if (j == M - 1) SMO_CUDA_CHECK(cudaEventRecord(slot_free[l % slots], st));
          unpermute_combine(yj, pos + p0, rw + p0, m.Tj, K, h, x + size_t(m.R0) * h, st);
          SMO_CUDA_CHECK(cudaEventRecord(mev(l, j, 5), st));
        }
      }
      moe_ev.push_back({mev(l, j, 4), mev(l, j, 5)});
    }
    snap("x_out", l, x, size_t(T) * h * 4, st);
    if (!batch_one && l + slots < L) {
      const int ln = l + slots;
      h2d_bytes += enqueue_h2d(ln, tev(ln * 8 + 0), tev(ln * 8 + 1));
      h2d_ev.push_back({tev(ln * 8 + 0), tev(ln * 8 + 1)});
    }
  }
  prefetch_next_step();  // the next step's first layers, into the slots this step just freed
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
  b1_measured = batch_one;
}

// Per layer (c_api.h smo_engine_layer_times): [h2d_start, h2d_end, bytes,
// raw bytes] + per micro-batch [o1_start, attn_start, attn_end, pre_moe,
// moe_start, moe_end], seconds from the step's start event.
void Engine::layer_times(double* out, size_t n) {
  const int M = last_mb;
  const size_t stride = 4 + 6 * size_t(M);
  SMO_REQUIRE(n >= size_t(L) * stride, "layer_times: output too small");
  SMO_CUDA_CHECK(cudaDeviceSynchronize());
  auto at = [&](cudaEvent_t e) {
    float ms = 0;
    SMO_CUDA_CHECK(cudaEventElapsedTime(&ms, ev[0], e));
    return double(ms) * 1e-3;
  };
  for (int l = 0; l < L; ++l) {
    double* o = out + size_t(l) * stride;
    o[0] = at(tev(l * 8 + 0));
    o[1] = at(tev(l * 8 + 1));
    o[2] = layer_bytes[size_t(l)];
    o[3] = layer_raw_bytes[size_t(l)];
    for (int j = 0; j < M; ++j) {
      const int ks[6] = {6, 2, 3, 7, 4, 5};
      for (int q = 0; q < 6; ++q) o[4 + 6 * j + q] = at(mev(l, j, ks[q]));
    }
  }
}

namespace {
// the compute stream waits here until the host dispatcher has published
// job `seq` done (the host attention of one micro-batch)
__global__ void host_flag_wait_kernel(const uint32_t* flag, uint32_t seq) {
  uint32_t v;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (int32_t(v - seq) >= 0) break;
    __nanosleep(2000);
  }
}
// job `seq`'s inputs (written by the preceding kernels) are complete
__global__ void host_flag_set_kernel(uint32_t* flag, uint32_t seq) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(seq) : "memory");
}
}  // namespace

// zero-copy read of pinned mapped host memory by the SMs (16-byte loads)
__global__ void copy_from_mapped_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n16) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

void Engine::copy_from_mapped(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  SMO_REQUIRE(bytes % 16 == 0 && (uintptr_t(dst) & 15) == 0 && (uintptr_t(src) & 15) == 0,
              "copy_from_mapped: 16-byte aligned sizes");
  const size_t n16 = bytes / 16;
  const unsigned grid = unsigned(std::min<size_t>((n16 + 255) / 256, 296));
  copy_from_mapped_kernel<<<std::max(1u, grid), 256, 0, st>>>(reinterpret_cast<uint4*>(dst),
                                                               reinterpret_cast<const uint4*>(src), n16);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void Engine::ensure_async_host() {
  if (host_flags) return;
  host_flags = halloc_mapped<uint32_t>(2);
  async_host.start(host_flags, host_flags + 1);
}

// Move requests between the drafter's GPU part (HBM K/V, K1) and CPU part
// (pinned host K/V, host pool): their drafter K/V rows follow them.
void Engine::set_draft_split(int g) {
  SMO_REQUIRE(draft_cpu, "engine: the draft split needs draft_cpu_kv");
  SMO_REQUIRE(dec_b > 0, "engine: set the draft split after prefill / decode_begin");
  SMO_REQUIRE(g >= -1 && g <= dec_b, "engine: draft split out of range");
  const int old_g = draft_g < 0 ? dec_b : draft_g;
  const int new_g = g < 0 ? dec_b : g;
  if (new_g == old_g) {
    draft_g = g;
    return;
  }
  SMO_CUDA_CHECK(cudaDeviceSynchronize());
  const size_t kv_req = size_t(nkv) * s_max * d;  // elements per request (contiguous)
  const int lo = std::min(old_g, new_g), hi_r = std::max(old_g, new_g);
  const bool to_host = new_g < old_g;
  for (int l = 0; l < dL; ++l) {
    const size_t off = size_t(lo) * kv_req, bytes = size_t(hi_r - lo) * kv_req * 2;
    if (to_host) {
      SMO_CUDA_CHECK(cudaMemcpy(dkc_h[size_t(l)] + off, dlayers[size_t(l)].kc + off, bytes, cudaMemcpyDeviceToHost));
      SMO_CUDA_CHECK(cudaMemcpy(dvc_h[size_t(l)] + off, dlayers[size_t(l)].vc + off, bytes, cudaMemcpyDeviceToHost));
    } else {
      SMO_CUDA_CHECK(cudaMemcpy(dlayers[size_t(l)].kc + off, dkc_h[size_t(l)] + off, bytes, cudaMemcpyHostToDevice));
      SMO_CUDA_CHECK(cudaMemcpy(dlayers[size_t(l)].vc + off, dvc_h[size_t(l)] + off, bytes, cudaMemcpyHostToDevice));
    }
  }
  draft_g = g;
}

int Engine::draft_split_times(double* out, size_t n) {
  SMO_CUDA_CHECK(cudaDeviceSynchronize());
  if (!last_was_decode || !last_split) return 0;
  const int m = last_draft_steps;
  SMO_REQUIRE(n >= size_t(3) * m, "draft_split_times: output too small");
  for (int t = 0; t < m; ++t) {
    float a = 0, b = 0;
    SMO_CUDA_CHECK(cudaEventElapsedTime(&a, draft_ev[size_t(t)], join_ev[size_t(t)]));
    SMO_CUDA_CHECK(cudaEventElapsedTime(&b, join_ev[size_t(t)], draft_ev[size_t(t) + 1]));
    double host = 0;
    for (uint32_t sq : step_seqs[size_t(t)]) host += double(async_host.dur_ns[sq & 255u].load(std::memory_order_acquire)) * 1e-9;
    out[3 * t] = a * 1e-3;
    out[3 * t + 1] = host;
    out[3 * t + 2] = b * 1e-3;
  }
  return m;
}

void Engine::wait_host_flag(uint32_t seq, cudaStream_t st) {
  host_flag_wait_kernel<<<1, 1, 0, st>>>(host_flags + 1, seq);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void Engine::signal_host_ready(uint32_t seq, cudaStream_t st) {
  host_flag_set_kernel<<<1, 1, 0, st>>>(host_flags, seq);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

void Engine::set_micro_batches(int m) {
  SMO_REQUIRE(m >= 0 && m <= kMaxMb, "engine: micro_batches must be in [0, 8]");
  if (m > 1) {
    SMO_REQUIRE(!batch_one, "engine: micro-batching needs MoeBatching::LARGE_BATCH");
    SMO_REQUIRE(!ep_on, "engine: micro-batching is not available with expert parallelism");
  }
  mb = std::max(1, m);
}

void Engine::AsyncHost::start(volatile uint32_t* ready, volatile uint32_t* done) {
  ready_flag = ready;
  done_flag = done;
  th = std::thread([this] {
    for (;;) {
      Item it{};
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return stop || head < q.size(); });
        if (head >= q.size()) return;  // stopping with nothing queued
        it = q[head++];
        if (head == q.size()) {
          q.clear();
          head = 0;
        }
      }
      // wait until the GPU has written this job's inputs (queued jobs are
      // finished even when stopping: the stream waits on their results; only
      // a stream that stopped making progress is abandoned, after 30 s)
      const auto t0 = std::chrono::steady_clock::now();
      for (int spins = 0; int32_t(*ready_flag - it.seq) < 0; ++spins) {
        if (spins > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
        if ((spins & 1023) == 1023) {
          std::lock_guard<std::mutex> lk(mu);
          if (stop && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30)) return;
        }
      }
      std::atomic_thread_fence(std::memory_order_acquire);
      const auto ts = std::chrono::steady_clock::now();
      cpu_verify_attention(it.job, *it.pool);
      dur_ns[it.seq & 255u].store(
          uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - ts).count()),
          std::memory_order_release);
      std::atomic_thread_fence(std::memory_order_seq_cst);
      *done_flag = it.seq;  // publish (mapped pinned memory; the GPU polls it)
    }
  });
}

void Engine::AsyncHost::push(const Item& it) {
  {
    std::lock_guard<std::mutex> lk(mu);
    q.push_back(it);
  }
  cv.notify_one();
}

void Engine::AsyncHost::shutdown() {
  if (!th.joinable()) return;
  {
    std::lock_guard<std::mutex> lk(mu);
    stop = true;
  }
  cv.notify_one();
  th.join();
}

void Engine::times(smo_stage_times* t) {
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
  r.codec = span(step_dec_ev);
  r.codec_bytes = step_codec_bytes;
  r.link_code = tmode ? double(tfmt) : xcomp ? 1.0 : 0.0;
  bool bound = !host_numa_bytes.empty();
  for (size_t b : host_numa_bytes) bound = bound && b > 0;
  r.host_numa = bound ? double(host_numa) : -1.0;
  {
    double cb = 0.0, rb = 0.0;
    for (size_t i = 0; i < blk_csize.size(); ++i) {
      cb += blk_coded[i] ? double(blk_csize[i]) : double(blk_bytes);
      rb += double(blk_bytes);
    }
    r.code_bits = rb > 0.0 ? 16.0 * cb / rb : 16.0;
  }
  for (double v : layer_raw_bytes) r.h2d_raw_bytes += v;
  r.others = std::max(0.0, r.target_total - r.attention - r.gpu_moe);
  *t = r;
}
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

smo_status smo_engine_set_draft_split(smo_engine* e, int32_t gpu_requests) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(e, "engine: null argument");
    e->impl.set_draft_split(gpu_requests);
  });
}

smo_status smo_engine_draft_split_times(smo_engine* e, double* out, size_t n, int32_t* steps) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(e && out && steps, "engine: null argument");
    *steps = e->impl.draft_split_times(out, n);
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

smo_status smo_engine_set_micro_batches(smo_engine* e, int32_t m) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(e, "engine: null argument");
    e->impl.set_micro_batches(m);
  });
}

smo_status smo_engine_last_micro_batches(smo_engine* e, int32_t* m) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(e && m, "engine: null argument");
    *m = e->impl.last_mb;
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
