// Does tcgen05.ld/st traffic from other warps slow tcgen05.mma?  One CTA per SM, 384 threads:
// warp 8 lane 0 issues n_mma M=128 N=64 K=16 MMAs back to back (into columns [0, 64)) and times
// them to the commit; warps 0-7 meanwhile loop tcgen05.ld.x32 + tcgen05.st.x32 on columns
// [256, 384) (mode 1) or idle (mode 0).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_tmem_contention mma_tmem_contention.cu
#include <cstdio>
#include "../../paper_2404_11068_b200/csrc/evo_common.cuh"
using namespace evo;

template <int MODE>
__global__ void __launch_bounds__(384, 1) k(unsigned long long* out, int n_mma, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int done;
  const uint32_t s0 = smem_u32(smem);
  const int w = threadIdx.x >> 5;
  if (w == 0) tmem_alloc<512>(smem_u32(&slot));
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_barrier_init();
    done = 0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (w == 8) {
    if ((threadIdx.x & 31) == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(128, 64, 0, 0);
      const uint64_t ad = make_sdesc(s0, 16, 512, kSw64), bd = make_sdesc(s0 + 65536, 16, 512, kSw64);
      unsigned long long t0 = clock64();
      for (int i = 0; i < n_mma; ++i) umma_bf16(tm, ad, bd, idesc, 1);
      umma_commit(smem_u32(&bar));
      mbar_wait(smem_u32(&bar), 0);
      unsigned long long t1 = clock64();
      if (blockIdx.x == 0) out[0] = t1 - t0;
      done = 1;
    }
  } else if (w < 8 && MODE == 1) {
    const uint32_t taddr = tm + 256 + (w >> 2) * 64 + (((uint32_t)(w & 3) * 32) << 16);
    uint32_t r[32];
    float acc = 0.f;
    int it = 0;
    while (!done) {
      tmem_ld32(taddr, r);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 32; ++c) r[c] += 1u;
      tmem_st32(taddr + 32, r);
      tmem_wait_st();
      acc += __uint_as_float(r[it & 31]);
      ++it;
    }
    if (acc == 12345.f) sink[0] = acc;
    if (blockIdx.x == 0 && threadIdx.x == 0) out[1] = it;
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tm);
}

int main() {
  unsigned long long* d;
  float* s;
  cudaMalloc(&d, 16);
  cudaMalloc(&s, 4);
  for (int mode = 0; mode < 2; ++mode) {
    auto f = mode ? k<1> : k<0>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    const int n = 4096;
    cudaMemset(d, 0, 16);
    f<<<148, 384, 131072>>>(d, 16, s);
    f<<<148, 384, 131072>>>(d, n, s);
    cudaDeviceSynchronize();
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %.1f cycles per N=64 K=16 MMA; ld/st iterations per warp: %llu\n", mode,
           mode ? "8 warps streaming tcgen05.ld/st" : "idle warps", (double)h[0] / n, h[1]);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
