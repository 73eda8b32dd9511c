// Microbenchmark: cycles per tcgen05.mma for the shapes K1/K4 issue.
//   SS  : A, B from shared memory (K-major, SW128)        M=128 N=128 K=16
//   SSn : as SS with B MN-major (V-like)                   M=128 N=128 K=16
//   TS  : A from TMEM, B MN-major from smem (K1 PV)        M=128 N=128 K=16
//   SS256: SS with N=256
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include
//        -I paper_2508_21706_b200/csrc tools/mma_bench.cu -o build/mma_bench -lcuda
#include <cstdio>

#include "common.cuh"

using namespace smo;

template <int mode>
__global__ void __launch_bounds__(128, 1) bench(int iters, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t done;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  fence_proxy_async();
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    constexpr int N = (mode == 3 || mode == 7) ? 256 : (mode == 5 ? 64 : 128);
    constexpr uint32_t id = make_idesc_bf16(128, N, (mode == 1 || mode == 2 || mode == 5 || mode == 8) ? 1 : 0,
                                            (mode == 6 || mode == 8) ? 1 : 0);
    uint64_t ad[8], bd[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const bool amn = mode == 6 || mode == 8, bmn = mode == 1 || mode == 2 || mode == 5 || mode == 8;
      ad[kk] = amn ? make_sdesc_sw128(a + kk * 2048, 16384, 1024)
                   : make_sdesc_sw128(a + (kk % 4) * 32 + (kk / 4) * 16384, 16, 1024);
      bd[kk] = bmn ? make_sdesc_sw128(b + kk * 2048, 16384, 1024)
                   : make_sdesc_sw128(b + (kk % 4) * 32 + (kk / 4) * 16384, 16, 1024);
    }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if constexpr (mode == 2 || mode == 4 || mode == 7)
          umma_bf16_ts(tmem + 256, tmem + kk * 8, bd[kk], id, 1u);
        else
          umma_bf16(tmem, ad[kk], bd[kk], id, 1u);
      }
    }
    umma_commit(&done);
    mbar_wait(&done, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  const char* names[] = {"SS  A K  B K   N=128", "SS  A K  B MN  N=128", "TS  A=TMEM B MN N=128", "SS  A K  B K   N=256",
                         "TS  A=TMEM B K  N=128", "SS  A K  B MN  N=64", "SS  A MN B K   N=128", "TS  A=TMEM B K  N=256",
                         "SS  A MN B MN  N=128"};
  auto run = [&](auto kern, int mode) {
    const int iters = 400, grid = 148;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    kern<<<grid, 128, 100 * 1024>>>(iters, d);
    kern<<<grid, 128, 100 * 1024>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("%-26s %.1f cycles/MMA  (%s)\n", names[mode], double(mx) / (iters * 8), cudaGetErrorString(e));
  };
  run(bench<0>, 0); run(bench<1>, 1); run(bench<2>, 2); run(bench<3>, 3); run(bench<4>, 4);
  run(bench<5>, 5); run(bench<6>, 6); run(bench<7>, 7); run(bench<8>, 8);
  return 0;
}
