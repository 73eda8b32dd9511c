#include <algorithm>
// ep.cu — expert parallelism: token dispatch / combine
// around the grouped SwiGLU experts, and the transports that move the blocks.
//
// Rank r of P owns the experts e with e % P == r and streams only those
// (K5 per-rank shard). Per layer, on each rank:
//   router -> owner-major permutation -> ep_pack (fixed-capacity block per
//   destination: C rows + per-local-expert counts) -> all-to-all ->
//   ep_unpack (rows grouped by local expert, src-major inside an expert) ->
//   grouped SwiGLU/down on the local shard -> ep_pack_back -> all-to-all ->
//   combine at owner-major positions (fixed slot order, no atomics).
// Every expert row is computed by the same kernel with the same K order as on
// one GPU, so EP results are bit-identical to the single-GPU engine.
//
// Transports: NCCL grouped send/recv (libnccl.so.2 resolved with dlopen, so the
// library has no link-time NCCL dependency) and an in-process loopback group
// (P engines on one GPU, one host thread each) that makes dispatch/combine
// testable on a single B200.
#include <dlfcn.h>

#include <atomic>
#include <functional>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace smo {

// ---------------------------------------------------------------- kernels
namespace {

// owner-major expert id: experts of rank 0 first (in local order), then rank 1...
__global__ void ep_remap_kernel(const int32_t* ids, int n, int P, int E_loc, int32_t* oid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const int e = ids[i];
    oid[i] = (e % P) * E_loc + e / P;
  }
}

// send block d: rows [0, C) bf16 x h, then E_loc int32 counts. With `dests`
// (direct exchange) block d is stored straight into rank d's receive buffer.
__global__ void ep_pack_kernel(const uint16_t* __restrict__ xp, const int32_t* __restrict__ offsets, int P,
                               int E_loc, int C, int h, size_t block_bytes, uint8_t* __restrict__ send,
                               uint8_t* const* __restrict__ dests) {
  const int d = blockIdx.y;
  const int seg0 = offsets[d * E_loc], seg1 = offsets[(d + 1) * E_loc];
  uint8_t* blk = dests ? dests[d] : send + size_t(d) * block_bytes;
  if (blockIdx.x == 0 && threadIdx.x < E_loc) {
    int32_t* cnt = reinterpret_cast<int32_t*>(blk + size_t(C) * h * 2);
    cnt[threadIdx.x] = offsets[d * E_loc + threadIdx.x + 1] - offsets[d * E_loc + threadIdx.x];
  }
  const int rows = seg1 - seg0;
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const uint4* src = reinterpret_cast<const uint4*>(xp + size_t(seg0 + r) * h);
    uint4* dst = reinterpret_cast<uint4*>(blk + size_t(r) * h * 2);
    for (int c = threadIdx.x; c < h / 8; c += blockDim.x) dst[c] = src[c];
  }
}

// position of each local (token, slot) pair's returned row: d*C + rank in d
// (C = rows per returned block: the capacity, or the direct receive stride).
__global__ void ep_pos_kernel(const int32_t* __restrict__ oid, const int32_t* __restrict__ pos,
                              const int32_t* __restrict__ offsets, int n, int E_loc, int C, int32_t* pos_ep) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int d = oid[i] / E_loc;
  pos_ep[i] = d * C + (pos[i] - offsets[d * E_loc]);
}

// recv block s -> rows grouped by local expert (src-major within an expert);
// offsets_l [E_loc+1]; back[q] = s*C + i (where row q came from).
__global__ void ep_unpack_kernel(const uint8_t* __restrict__ recv, int P, int E_loc, int C, int h,
                                 size_t block_bytes, uint16_t* __restrict__ xl, int32_t* __restrict__ offsets_l,
                                 int32_t* __restrict__ back) {
  extern __shared__ int sh[];
  int* cnt = sh;                // [P][E_loc]
  int* dst0 = sh + P * E_loc;   // start row of (s, le) block in xl
  int* src0 = dst0 + P * E_loc; // start row of (s, le) block in the recv block s
  for (int i = threadIdx.x; i < P * E_loc; i += blockDim.x) {
    const int s = i / E_loc, le = i % E_loc;
    cnt[i] = reinterpret_cast<const int32_t*>(recv + size_t(s) * block_bytes + size_t(C) * h * 2)[le];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int le = 0; le < E_loc; ++le) {
      offsets_l[le] = run;
      for (int s = 0; s < P; ++s) {
        dst0[s * E_loc + le] = run;
        run += cnt[s * E_loc + le];
      }
    }
    offsets_l[E_loc] = run;
    for (int s = 0; s < P; ++s) {
      int r = 0;
      for (int le = 0; le < E_loc; ++le) {
        src0[s * E_loc + le] = r;
        r += cnt[s * E_loc + le];
      }
    }
  }
  __syncthreads();
  for (int blk = blockIdx.x; blk < P * E_loc; blk += gridDim.x) {
    const int s = blk / E_loc;
    const int n = cnt[blk];
    for (int i = 0; i < n; ++i) {
      const int src_row = src0[blk] + i, dst_row = dst0[blk] + i;
      const uint4* src = reinterpret_cast<const uint4*>(recv + size_t(s) * block_bytes + size_t(src_row) * h * 2);
      uint4* dst = reinterpret_cast<uint4*>(xl + size_t(dst_row) * h);
      for (int c = threadIdx.x; c < h / 8; c += blockDim.x) dst[c] = src[c];
      if (threadIdx.x == 0) back[dst_row] = s * C + src_row;
    }
  }
}

// expert outputs back to their source ranks' slots (fp32 rows).
// splits > 1: down-projection K slices (split_stride elements apart) summed
// in slice order — the same fixed order as the single-GPU combine
__global__ void ep_pack_back_kernel(const float* __restrict__ yl, const int32_t* __restrict__ back,
                                    const int32_t* __restrict__ offsets_l, int E_loc, int h,
                                    float* __restrict__ sendback, int splits, size_t split_stride,
                                    uint8_t* const* __restrict__ dests, int C) {
  const int rows = offsets_l[E_loc];
  for (int q = blockIdx.x; q < rows; q += gridDim.x) {
    const float4* src = reinterpret_cast<const float4*>(yl + size_t(q) * h);
    const int bq = back[q];
    float4* dst = dests ? reinterpret_cast<float4*>(dests[bq / C]) + size_t(bq % C) * (h / 4)
                        : reinterpret_cast<float4*>(sendback + size_t(bq) * h);
    for (int c = threadIdx.x; c < h / 4; c += blockDim.x) {
      float4 v = src[c];
      for (int s = 1; s < splits; ++s) {
        const float4 v2 = reinterpret_cast<const float4*>(yl + size_t(s) * split_stride + size_t(q) * h)[c];
        v.x += v2.x;
        v.y += v2.y;
        v.z += v2.z;
        v.w += v2.w;
      }
      dst[c] = v;
    }
  }
}

}  // namespace

void ep_remap(const int32_t* ids, int n, int P, int E_loc, int32_t* oid, cudaStream_t st) {
  ep_remap_kernel<<<(n + 255) / 256, 256, 0, st>>>(ids, n, P, E_loc, oid);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}
void ep_pack(const void* xp, const int32_t* offsets, int P, int E_loc, int C, int h, size_t block_bytes, void* send,
             cudaStream_t st, uint8_t* const* dests) {
  dim3 grid(64, P);
  ep_pack_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint16_t*>(xp), offsets, P, E_loc, C, h, block_bytes,
                                       reinterpret_cast<uint8_t*>(send), dests);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}
void ep_pos(const int32_t* oid, const int32_t* pos, const int32_t* offsets, int n, int E_loc, int C, int32_t* pos_ep,
            cudaStream_t st) {
  ep_pos_kernel<<<(n + 255) / 256, 256, 0, st>>>(oid, pos, offsets, n, E_loc, C, pos_ep);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}
void ep_unpack(const void* recv, int P, int E_loc, int C, int h, size_t block_bytes, void* xl, int32_t* offsets_l,
               int32_t* back, cudaStream_t st) {
  const size_t smem = size_t(3) * P * E_loc * sizeof(int);
  ep_unpack_kernel<<<128, 256, smem, st>>>(reinterpret_cast<const uint8_t*>(recv), P, E_loc, C, h, block_bytes,
                                           reinterpret_cast<uint16_t*>(xl), offsets_l, back);
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}
void ep_pack_back(const float* yl, const int32_t* back, const int32_t* offsets_l, int E_loc, int h, float* sendback,
                  cudaStream_t st, int splits, size_t split_stride, uint8_t* const* dests, int C) {
  ep_pack_back_kernel<<<256, 256, 0, st>>>(yl, back, offsets_l, E_loc, h, sendback, std::max(1, splits),
                                           split_stride, dests, std::max(1, C));
  count_launch();
  SMO_CUDA_CHECK(cudaGetLastError());
}

// ---------------------------------------------------------------- transports
// In-process loopback: P engines (one host thread each) on one device.
struct LoopbackTransport : EpTransport {
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  std::vector<const void*> sends;
  std::vector<cudaEvent_t> sent, copied;

  explicit LoopbackTransport(int p) {
    P = p;
    sends.assign(size_t(p), nullptr);
    sent.resize(size_t(p));
    copied.resize(size_t(p));
    for (int i = 0; i < p; ++i) {
      SMO_CUDA_CHECK(cudaEventCreateWithFlags(&sent[size_t(i)], cudaEventDisableTiming));
      SMO_CUDA_CHECK(cudaEventCreateWithFlags(&copied[size_t(i)], cudaEventDisableTiming));
    }
  }
  ~LoopbackTransport() override {
    for (auto e : sent) cudaEventDestroy(e);
    for (auto e : copied) cudaEventDestroy(e);
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t gen = generation;
    if (++arrived == P) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
  void alltoall(int rank, const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    SMO_CUDA_CHECK(cudaEventRecord(sent[size_t(rank)], st));
    {
      std::lock_guard<std::mutex> lk(mu);
      sends[size_t(rank)] = send;
    }
    barrier();  // every rank's send buffer and event are published
    for (int s = 0; s < P; ++s) {
      SMO_CUDA_CHECK(cudaStreamWaitEvent(st, sent[size_t(s)], 0));
      SMO_CUDA_CHECK(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(recv) + size_t(s) * bytes,
                                     reinterpret_cast<const uint8_t*>(sends[size_t(s)]) + size_t(rank) * bytes, bytes,
                                     cudaMemcpyDeviceToDevice, st));
    }
    SMO_CUDA_CHECK(cudaEventRecord(copied[size_t(rank)], st));
    barrier();  // every rank has enqueued its reads
    for (int s = 0; s < P; ++s) SMO_CUDA_CHECK(cudaStreamWaitEvent(st, copied[size_t(s)], 0));
    barrier();  // events consumed before they can be re-recorded
  }
};

// NCCL grouped send/recv through a dlopen'd libnccl.so.2.
struct NcclApi {
  void* so = nullptr;
  int (*getUniqueId)(void*) = nullptr;
  void* commInitRank = nullptr;  // int(ncclComm_t*, int, ncclUniqueId /*by value*/, int)
  int (*commDestroy)(void*) = nullptr;
  int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*groupStart)() = nullptr;
  int (*groupEnd)() = nullptr;
  const char* (*errStr)(int) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* cands[] = {"libnccl.so.2", "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2"};
    for (const char* c : cands) {
      api.so = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
      if (api.so) break;
    }
    if (!api.so) return;
    api.getUniqueId = reinterpret_cast<int (*)(void*)>(dlsym(api.so, "ncclGetUniqueId"));
    api.commInitRank = dlsym(api.so, "ncclCommInitRank");
    api.commDestroy = reinterpret_cast<int (*)(void*)>(dlsym(api.so, "ncclCommDestroy"));
    api.send = reinterpret_cast<int (*)(const void*, size_t, int, int, void*, cudaStream_t)>(dlsym(api.so, "ncclSend"));
    api.recv = reinterpret_cast<int (*)(void*, size_t, int, int, void*, cudaStream_t)>(dlsym(api.so, "ncclRecv"));
    api.groupStart = reinterpret_cast<int (*)()>(dlsym(api.so, "ncclGroupStart"));
    api.groupEnd = reinterpret_cast<int (*)()>(dlsym(api.so, "ncclGroupEnd"));
    api.errStr = reinterpret_cast<const char* (*)(int)>(dlsym(api.so, "ncclGetErrorString"));
  });
  if (!api.so || !api.send || !api.recv || !api.commInitRank)
    throw Error(SMO_NCCL, "libnccl.so.2 not found (expert parallelism needs NCCL)");
  return api;
}

static void nccl_check(int r, const char* what) {
  if (r != 0) throw Error(SMO_NCCL, std::string(what) + ": " + (nccl().errStr ? nccl().errStr(r) : "nccl error"));
}

// ncclCommInitRank takes the 128-byte ncclUniqueId by value; passing a struct
// of that size by value matches the x86-64 ABI of the real signature.
struct UniqueId {
  char b[128];
};

struct NcclTransport : EpTransport {
  void* comm = nullptr;
  NcclTransport(const uint8_t* id, int nranks, int rank) {
    P = nranks;
    UniqueId uid;
    std::memcpy(uid.b, id, 128);
    auto init = reinterpret_cast<int (*)(void**, int, UniqueId, int)>(nccl().commInitRank);
    nccl_check(init(&comm, nranks, uid, rank), "ncclCommInitRank");
  }
  ~NcclTransport() override {
    if (comm) nccl().commDestroy(comm);
  }
  void alltoall(int rank, const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    (void)rank;
    NcclApi& a = nccl();
    constexpr int kUint8 = 1;  // ncclUint8
    nccl_check(a.groupStart(), "ncclGroupStart");
    for (int peer = 0; peer < P; ++peer) {
      nccl_check(a.send(reinterpret_cast<const uint8_t*>(send) + size_t(peer) * bytes, bytes, kUint8, peer, comm, st),
                 "ncclSend");
      nccl_check(a.recv(reinterpret_cast<uint8_t*>(recv) + size_t(peer) * bytes, bytes, kUint8, peer, comm, st),
                 "ncclRecv");
    }
    nccl_check(a.groupEnd(), "ncclGroupEnd");
  }
};

// Peer-memory transport (CUDA IPC): every rank owns a mailbox [2][P][slot]
// that the other ranks write into directly — over NVLink between GPUs, or
// within one GPU between processes — followed by a flag area. Round R uses
// half R % 2: rank r stores its block for p into p's mailbox slot [R%2][r]
// (after p has consumed round R-2, which used that half), then a one-thread
// kernel publishes R into p's arrived[r] (release, system scope) and spins
// until its own arrived[q] >= R for every peer q (acquire); the consumer
// kernels then read the local mailbox, and a last one-thread kernel
// publishes "consumed R" into every peer's consumed_by[r]. The round
// counter lives in device memory, so the whole exchange is kernels only: no
// host barrier per exchange, no events, capturable in a CUDA graph (an
// iteration has an even number of exchanges, so replayed halves repeat).
// Direct mode: the dispatch / combine kernels store into the peers'
// mailboxes themselves (dests[half][p] = p's slot [half][r]); the staged
// alltoall is the same protocol with copies on both sides.
namespace {
struct EpFlags {
  uint32_t* arrived;      // local [P]: round whose block from rank q has landed here
  uint32_t* consumed_by;  // local [P]: round rank q has finished reading (the blocks this rank wrote)
  uint32_t* const* peer_arrived;      // device [P]: peer q's arrived array
  uint32_t* const* peer_consumed_by;  // device [P]: peer q's consumed_by array
  uint32_t* round;        // local: last completed round
  int P, rank;
};
__device__ __forceinline__ uint32_t ld_acq_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void spin_geq(const uint32_t* p, uint32_t want) {
  while (int32_t(ld_acq_sys(p) - want) < 0) __nanosleep(256);
}
// before writing round R = round + 1: every peer has consumed round R - 2
__global__ void ep_flag_begin_kernel(EpFlags f) {
  const uint32_t R = *f.round + 1;
  if (R <= 2) return;
  for (int q = 0; q < f.P; ++q)
    if (q != f.rank) spin_geq(f.consumed_by + q, R - 2);
}
// this rank's blocks for round R are stored: tell every peer, wait for theirs
__global__ void ep_flag_arrive_kernel(EpFlags f) {
  const uint32_t R = *f.round + 1;
  __threadfence_system();
  for (int q = 0; q < f.P; ++q)
    if (q != f.rank) st_rel_sys(f.peer_arrived[q] + f.rank, R);
  for (int q = 0; q < f.P; ++q)
    if (q != f.rank) spin_geq(f.arrived + q, R);
  *f.round = R;
}
// round R's mailbox half has been read here: peers may overwrite it at R + 2
__global__ void ep_flag_done_kernel(EpFlags f) {
  const uint32_t R = *f.round;
  __threadfence_system();
  for (int q = 0; q < f.P; ++q)
    if (q != f.rank) st_rel_sys(f.peer_consumed_by[q] + f.rank, R);
}
}  // namespace

struct IpcTransport : EpTransport {
  int rank = 0;
  size_t slot = 0, data_bytes = 0;
  uint8_t* mailbox = nullptr;   // [2][P][slot] + flags: arrived[P], consumed_by[P]
  uint8_t** d_dests = nullptr;  // device [2][P]
  uint32_t** d_peer_flags = nullptr;  // device [2][P]: peers' arrived, then consumed_by arrays
  uint32_t* d_round = nullptr;
  std::vector<uint8_t*> peer_mb;
  int parity = 0;
  EpFlags flags{};

  IpcTransport(int nranks, int r, size_t slot_bytes) {
    P = nranks;
    rank = r;
    slot = (slot_bytes + 255) & ~size_t(255);
    data_bytes = 2 * size_t(P) * slot;
    const size_t fb = (2 * size_t(P) * sizeof(uint32_t) + 255) & ~size_t(255);
    SMO_CUDA_CHECK(cudaMalloc(&mailbox, data_bytes + fb));
    SMO_CUDA_CHECK(cudaMemset(mailbox + data_bytes, 0, fb));
    SMO_CUDA_CHECK(cudaMalloc(&d_dests, 2 * size_t(P) * sizeof(uint8_t*)));
    SMO_CUDA_CHECK(cudaMalloc(&d_peer_flags, 2 * size_t(P) * sizeof(uint32_t*)));
    SMO_CUDA_CHECK(cudaMalloc(&d_round, sizeof(uint32_t)));
    SMO_CUDA_CHECK(cudaMemset(d_round, 0, sizeof(uint32_t)));
    SMO_CUDA_CHECK(cudaDeviceSynchronize());
  }
  ~IpcTransport() override {
    for (int p = 0; p < int(peer_mb.size()); ++p)
      if (p != rank && peer_mb[size_t(p)]) cudaIpcCloseMemHandle(peer_mb[size_t(p)]);
    if (d_round) cudaFree(d_round);
    if (d_peer_flags) cudaFree(d_peer_flags);
    if (d_dests) cudaFree(d_dests);
    if (mailbox) cudaFree(mailbox);
  }
  uint32_t* flags_of(uint8_t* mb) const { return reinterpret_cast<uint32_t*>(mb + data_bytes); }
  // handle blob: the mailbox memory handle
  static constexpr size_t kBlob = sizeof(cudaIpcMemHandle_t);
  void export_handles(uint8_t* out) const {
    cudaIpcMemHandle_t mh;
    SMO_CUDA_CHECK(cudaIpcGetMemHandle(&mh, mailbox));
    std::memcpy(out, &mh, sizeof(mh));
  }
  // `barrier` runs once, after every rank has mapped its peers (the flag
  // areas were zeroed at creation, before the handles were exchanged)
  void connect(const uint8_t* all, smo_barrier_fn barrier, void* ctx) {
    peer_mb.assign(size_t(P), nullptr);
    for (int p = 0; p < P; ++p) {
      if (p == rank) {
        peer_mb[size_t(p)] = mailbox;
        continue;
      }
      cudaIpcMemHandle_t mh;
      std::memcpy(&mh, all + size_t(p) * kBlob, sizeof(mh));
      void* ptr = nullptr;
      SMO_CUDA_CHECK(cudaIpcOpenMemHandle(&ptr, mh, cudaIpcMemLazyEnablePeerAccess));
      peer_mb[size_t(p)] = reinterpret_cast<uint8_t*>(ptr);
    }
    std::vector<uint8_t*> dests(2 * size_t(P));
    std::vector<uint32_t*> pf(2 * size_t(P));
    for (int half = 0; half < 2; ++half)
      for (int p = 0; p < P; ++p)
        dests[size_t(half) * P + p] = peer_mb[size_t(p)] + (size_t(half) * P + rank) * slot;
    for (int p = 0; p < P; ++p) {
      pf[size_t(p)] = flags_of(peer_mb[size_t(p)]);          // peer p's arrived[]
      pf[size_t(P + p)] = flags_of(peer_mb[size_t(p)]) + P;  // peer p's consumed_by[]
    }
    SMO_CUDA_CHECK(cudaMemcpy(d_dests, dests.data(), dests.size() * sizeof(uint8_t*), cudaMemcpyHostToDevice));
    SMO_CUDA_CHECK(cudaMemcpy(d_peer_flags, pf.data(), pf.size() * sizeof(uint32_t*), cudaMemcpyHostToDevice));
    flags = EpFlags{flags_of(mailbox), flags_of(mailbox) + P, d_peer_flags, d_peer_flags + P, d_round, P, rank};
    if (barrier) barrier(ctx);
  }
  size_t direct_slot() const override { return slot; }
  uint8_t* const* direct_begin(cudaStream_t st, const uint8_t** recv) override {
    SMO_REQUIRE(!peer_mb.empty(), "ep ipc: transport not connected");
    const int half = parity;
    parity ^= 1;
    ep_flag_begin_kernel<<<1, 1, 0, st>>>(flags);
    count_launch();
    SMO_CUDA_CHECK(cudaGetLastError());
    *recv = mailbox + size_t(half) * P * slot;
    return d_dests + size_t(half) * P;
  }
  void direct_exchange(cudaStream_t st) override {
    ep_flag_arrive_kernel<<<1, 1, 0, st>>>(flags);
    count_launch();
    SMO_CUDA_CHECK(cudaGetLastError());
  }
  void direct_done(cudaStream_t st) override {
    ep_flag_done_kernel<<<1, 1, 0, st>>>(flags);
    count_launch();
    SMO_CUDA_CHECK(cudaGetLastError());
  }
  void alltoall(int r, const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    SMO_REQUIRE(r == rank && bytes <= slot, "ep ipc: block larger than the mailbox slot");
    const int half = parity;
    const uint8_t* mine = nullptr;
    direct_begin(st, &mine);
    for (int p = 0; p < P; ++p)
      SMO_CUDA_CHECK(cudaMemcpyAsync(peer_mb[size_t(p)] + (size_t(half) * P + rank) * slot,
                                     reinterpret_cast<const uint8_t*>(send) + size_t(p) * bytes, bytes,
                                     cudaMemcpyDeviceToDevice, st));
    direct_exchange(st);
    for (int p = 0; p < P; ++p)
      SMO_CUDA_CHECK(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(recv) + size_t(p) * bytes, mine + size_t(p) * slot,
                                     bytes, cudaMemcpyDeviceToDevice, st));
    direct_done(st);
  }
};

}  // namespace smo

struct smo_ep_group {
  smo::EpTransport* t = nullptr;
  ~smo_ep_group() { delete t; }
};

namespace smo {
smo_status run_guarded(const std::function<void()>& f);
void permute(const int32_t* ids, int T, int k, int E, const void* x, int h, int32_t* offsets, int32_t* perm,
             int32_t* pos, void* xp, cudaStream_t st);
void unpermute_combine(const float* y, const int32_t* pos, const float* w, int T, int k, int h, float* res,
                       cudaStream_t st, int splits = 1, size_t split_stride = 0);
EpTransport* ep_transport(void* group) { return group ? reinterpret_cast<smo_ep_group*>(group)->t : nullptr; }
}  // namespace smo

extern "C" {

smo_status smo_ep_loopback_create(int32_t ep_size, smo_ep_group** out) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(out && ep_size >= 1, "ep: bad arguments");
    auto* g = new smo_ep_group();
    g->t = new smo::LoopbackTransport(ep_size);
    *out = g;
  });
}

smo_status smo_nccl_unique_id(uint8_t* id128) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(id128, "ep: null id buffer");
    smo::nccl_check(smo::nccl().getUniqueId(id128), "ncclGetUniqueId");
  });
}

smo_status smo_ep_nccl_create(const uint8_t* id128, int32_t nranks, int32_t rank, smo_ep_group** out) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(id128 && out && nranks >= 1 && rank >= 0 && rank < nranks, "ep: bad arguments");
    auto* g = new smo_ep_group();
    try {
      g->t = new smo::NcclTransport(id128, nranks, rank);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

size_t smo_ep_ipc_handle_bytes(void) { return smo::IpcTransport::kBlob; }

smo_status smo_ep_ipc_create(int32_t nranks, int32_t rank, uint64_t slot_bytes, smo_ep_group** out, uint8_t* handles) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(out && handles && nranks >= 1 && rank >= 0 && rank < nranks && slot_bytes > 0, "ep: bad arguments");
    auto* g = new smo_ep_group();
    try {
      auto* t = new smo::IpcTransport(nranks, rank, size_t(slot_bytes));
      g->t = t;
      t->export_handles(handles);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

smo_status smo_ep_ipc_connect(smo_ep_group* g, const uint8_t* all_handles, smo_barrier_fn barrier, void* ctx) {
  return smo::run_guarded([&] {
    SMO_REQUIRE(g && all_handles && barrier, "ep: bad arguments");
    auto* t = dynamic_cast<smo::IpcTransport*>(g->t);
    SMO_REQUIRE(t, "ep: not an IPC group");
    t->connect(all_handles, barrier, ctx);
  });
}

// ---- standalone dispatch / combine (SURVEY.md §8(b) smo_ep_dispatch/combine)
namespace {
struct EpWs {  // workspace carve-up, identical for dispatch and combine
  int32_t *oid, *offsets, *perm, *pos;
  uint16_t* xp;
  uint8_t *send, *recv;
  float *sendback, *recvback;
  size_t blk_d, bytes;
};
EpWs ep_ws(void* base, int P, int T, int k, int h, int E, int C) {
  const int E_loc = E / P;
  EpWs w{};
  w.blk_d = (size_t(C) * h * 2 + size_t(E_loc) * 4 + 15) & ~size_t(15);
  size_t off = 0;
  auto take = [&](size_t n) {
    const size_t at = off;
    off = (off + n + 255) & ~size_t(255);
    return reinterpret_cast<uint8_t*>(base) + at;
  };
  const size_t PT = size_t(T) * k;
  w.oid = reinterpret_cast<int32_t*>(take(PT * 4));
  w.offsets = reinterpret_cast<int32_t*>(take(size_t(E + 1) * 4));
  w.perm = reinterpret_cast<int32_t*>(take(PT * 4));
  w.pos = reinterpret_cast<int32_t*>(take(PT * 4));
  w.xp = reinterpret_cast<uint16_t*>(take(PT * h * 2));
  w.send = take(size_t(P) * w.blk_d);
  w.recv = take(size_t(P) * w.blk_d);
  w.sendback = reinterpret_cast<float*>(take(size_t(P) * C * h * 4));
  w.recvback = reinterpret_cast<float*>(take(size_t(P) * C * h * 4));
  w.bytes = off;
  return w;
}
void ep_check(smo_ep_group* g, int rank, int T, int k, int h, int E, int C) {
  SMO_REQUIRE(g && g->t, "ep: null group");
  const int P = g->t->P;
  SMO_REQUIRE(rank >= 0 && rank < P && T >= 0 && k >= 1 && h % 8 == 0 && E % P == 0 && C >= T * k,
              "ep: bad arguments (E % P == 0, h % 8 == 0, capacity C >= T*k on every rank)");
}
}  // namespace

size_t smo_ep_workspace(int32_t P, int32_t T, int32_t k, int32_t h, int32_t E, int32_t C) {
  if (P < 1 || T < 0 || k < 1 || h < 8 || E < P || C < 1) return 0;
  return ep_ws(nullptr, P, T, k, h, E, C).bytes;
}

smo_status smo_ep_dispatch(smo_ep_group* g, int32_t rank, const void* x, const int32_t* ids, int32_t T, int32_t k,
                           int32_t h, int32_t E, int32_t C, void* xl, int32_t* offsets_l, int32_t* back,
                           int32_t* pos_ep, void* workspace, smo_stream stream) {
  return smo::run_guarded([&] {
    ep_check(g, rank, T, k, h, E, C);
    SMO_REQUIRE(x && ids && xl && offsets_l && back && pos_ep && workspace, "ep dispatch: null pointer");
    const int P = g->t->P, E_loc = E / P, PT = T * k;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    EpWs w = ep_ws(workspace, P, T, k, h, E, C);
    smo::ep_remap(ids, PT, P, E_loc, w.oid, st);
    smo::permute(w.oid, T, k, E, x, h, w.offsets, w.perm, w.pos, w.xp, st);
    smo::ep_pack(w.xp, w.offsets, P, E_loc, C, h, w.blk_d, w.send, st, nullptr);
    smo::ep_pos(w.oid, w.pos, w.offsets, PT, E_loc, C, pos_ep, st);
    g->t->alltoall(rank, w.send, w.recv, w.blk_d, st);
    smo::ep_unpack(w.recv, P, E_loc, C, h, w.blk_d, xl, offsets_l, back, st);
  });
}

smo_status smo_ep_combine(smo_ep_group* g, int32_t rank, const float* yl, const int32_t* back,
                          const int32_t* offsets_l, const int32_t* pos_ep, const float* weights, int32_t T,
                          int32_t k, int32_t h, int32_t E, int32_t C, float* x, void* workspace, smo_stream stream) {
  return smo::run_guarded([&] {
    ep_check(g, rank, T, k, h, E, C);
    SMO_REQUIRE(yl && back && offsets_l && pos_ep && weights && x && workspace, "ep combine: null pointer");
    const int P = g->t->P, E_loc = E / P;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    EpWs w = ep_ws(workspace, P, T, k, h, E, C);
    smo::ep_pack_back(yl, back, offsets_l, E_loc, h, w.sendback, st, 1, 0, nullptr, 1);
    g->t->alltoall(rank, w.sendback, w.recvback, size_t(C) * h * sizeof(float), st);
    smo::unpermute_combine(w.recvback, pos_ep, weights, T, k, h, x, st);
  });
}

smo_status smo_ep_group_destroy(smo_ep_group* g) {
  return smo::run_guarded([&] { delete g; });
}

}  // extern "C"
