// Microbenchmarks on one SM: tcgen05.ld throughput, MUFU ex2 throughput, FFMA2 throughput.
#include <cstdio>
#include "../../paper_2404_11068_b200/csrc/evo_common.cuh"
using namespace evo;

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(unsigned long long* out, int iters, float* sink) {
  __shared__ uint32_t slot;
  const int w = threadIdx.x >> 5;
  if (w == 0) tmem_alloc<512>(smem_u32(&slot));
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot + (((w & 3) * 32) << 16) + (w >> 2) * 128;
  float acc = threadIdx.x;
  __syncthreads();
  unsigned long long t0 = clock64();
  if (MODE == 0) {  // tcgen05.ld x32, wait per 4 loads
    for (int i = 0; i < iters; ++i) {
      uint32_t r0[32], r1[32], r2[32], r3[32];
      tmem_ld32(tm, r0); tmem_ld32(tm + 32, r1); tmem_ld32(tm + 64, r2); tmem_ld32(tm + 96, r3);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 32; ++c) acc += __uint_as_float(r0[c] ^ r1[c] ^ r2[c] ^ r3[c]);
    }
  } else if (MODE == 1) {  // MUFU ex2: 64 independent per iter
    float x[64];
#pragma unroll
    for (int c = 0; c < 64; ++c) x[c] = acc * 1e-3f + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int c = 0; c < 64; ++c) x[c] = fast_exp2(x[c]) * -0.5f;
    }
#pragma unroll
    for (int c = 0; c < 64; ++c) acc += x[c];
  } else if (MODE == 2) {  // FFMA2: 32 independent pairs
    uint64_t x[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) x[c] = f2_pack(acc + c, acc - c);
    const uint64_t m = f2_pack(0.999f, 0.998f), ad = f2_pack(0.1f, 0.2f);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int c = 0; c < 32; ++c) x[c] = f2_fma(x[c], m, ad);
    }
#pragma unroll
    for (int c = 0; c < 32; ++c) { float a, b; f2_unpack(x[c], a, b); acc += a + b; }
  } else if (MODE == 3) {  // tcgen05.st x32
    uint32_t r[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) r[c] = __float_as_uint(acc + c);
    for (int i = 0; i < iters; ++i) {
      tmem_st32(tm, r); tmem_st32(tm + 32, r);
      tmem_wait_st();
      r[0] += 1;
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345.f) sink[0] = acc;
  tc_fence_before(); __syncthreads();
  if (w == 0) tmem_dealloc<512>(slot);
}

int main() {
  unsigned long long* d; float* s; cudaMalloc(&d, 8 * 148); cudaMalloc(&s, 4);
  unsigned long long h[148];
  const char* names[4] = {"tmem ld x32 (4/iter)", "mufu ex2 (64/iter)", "ffma2 (32/iter)", "tmem st x32 (2/iter)"};
  for (int mode = 0; mode < 4; ++mode)
    for (int nwarps : {4, 8, 16}) {
      int iters = 1000;
      auto f = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : k<3>;
      f<<<148, nwarps * 32>>>(d, 10, s);
      f<<<148, nwarps * 32>>>(d, iters, s);
      cudaDeviceSynchronize();
      cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
      double cyc = h[0];
      double per_iter = cyc / iters;
      double units = mode == 0 ? 4.0 * 4096 * nwarps : mode == 1 ? 64.0 * 32 * nwarps : mode == 2 ? 64.0 * 32 * nwarps : 2.0 * 4096 * nwarps;
      printf("%-24s warps=%2d  cycles/iter=%8.1f  -> %8.1f %s per clk per SM\n", names[mode], nwarps, per_iter,
             units / per_iter, mode == 0 || mode == 3 ? "bytes" : (mode == 1 ? "ex2" : "flop-lanes(fma)"));
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
