// Which pipe does the bf16x2 pack (cvt.rn.bf16x2.f32 = F2FP) use, and does it compete with MUFU
// ex2?  One SM-wide block per SM, 16 warps, independent chains; prints lanes per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xu_bench xu_bench.cu && ./xu_bench
#include <cstdio>
#include "../../paper_2404_11068_b200/csrc/evo_common.cuh"
using namespace evo;

__device__ __forceinline__ uint32_t pack_alu(float a, float b) {  // RNE bf16 pack on the ALU
  uint32_t ua = __float_as_uint(a), ub = __float_as_uint(b);
  ua += 0x7fffu + ((ua >> 16) & 1u);
  ub += 0x7fffu + ((ub >> 16) & 1u);
  return __byte_perm(ua, ub, 0x7632);
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(unsigned long long* out, int iters, float* sink) {
  float acc = threadIdx.x * 1e-3f;
  float x[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) x[c] = acc + c * 1e-2f;
  uint32_t h = 0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {  // 32 ex2
#pragma unroll
      for (int c = 0; c < 32; ++c) x[c] = fast_exp2(x[c]) * -0.5f;
    } else if (MODE == 1) {  // 16 F2FP
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        h ^= pack_bf16(x[2 * c], x[2 * c + 1]);
        x[2 * c] = __uint_as_float(__float_as_uint(x[2 * c]) ^ (h & 1u));
      }
    } else if (MODE == 2) {  // 32 ex2 + 16 F2FP (the forward's mix)
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const float p0 = fast_exp2(x[2 * c]), p1 = fast_exp2(x[2 * c + 1]);
        h ^= pack_bf16(p0, p1);
        x[2 * c] = p0 * -0.5f;
        x[2 * c + 1] = p1 * -0.5f;
      }
    } else if (MODE == 3) {  // 32 ex2 + 16 ALU packs
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const float p0 = fast_exp2(x[2 * c]), p1 = fast_exp2(x[2 * c + 1]);
        h ^= pack_alu(p0, p1);
        x[2 * c] = p0 * -0.5f;
        x[2 * c + 1] = p1 * -0.5f;
      }
    } else if (MODE == 4) {  // 32 ex2 + 32 F2FP (the backward's mix: P and dS packs)
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const float p0 = fast_exp2(x[2 * c]), p1 = fast_exp2(x[2 * c + 1]);
        h ^= pack_bf16(p0, p1) + pack_bf16(p0 * 0.3f, p1 * 0.7f);
        x[2 * c] = p0 * -0.5f;
        x[2 * c + 1] = p1 * -0.5f;
      }
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
#pragma unroll
  for (int c = 0; c < 32; ++c) acc += x[c];
  if (acc == 12345.f || h == 0x12345u) sink[0] = acc + h;
}

int main() {
  unsigned long long* d;
  float* s;
  cudaMalloc(&d, 8 * 148);
  cudaMalloc(&s, 4);
  unsigned long long hbuf[148];
  const char* names[5] = {"ex2 x32", "f2fp x16", "ex2 x32 + f2fp x16", "ex2 x32 + alu-pack x16",
                          "ex2 x32 + f2fp x32"};
  for (int mode = 0; mode < 5; ++mode) {
    const int nwarps = 16, iters = 2000;
    auto f = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : mode == 3 ? k<3> : k<4>;
    f<<<148, nwarps * 32>>>(d, 10, s);
    f<<<148, nwarps * 32>>>(d, iters, s);
    cudaDeviceSynchronize();
    cudaMemcpy(hbuf, d, 8 * 148, cudaMemcpyDeviceToHost);
    const double per_iter = (double)hbuf[0] / iters;  // cycles per iteration (whole SM)
    const double thr = 32.0 * nwarps;                 // threads per SM
    printf("%-26s cycles/iter=%8.1f  ex2-or-op lanes/clk/SM: ex2 %.2f  pack %.2f\n", names[mode],
           per_iter, (mode == 1 ? 0 : 32) * thr / per_iter,
           (mode == 0 ? 0 : mode == 4 ? 32 : 16) * thr / per_iter);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
