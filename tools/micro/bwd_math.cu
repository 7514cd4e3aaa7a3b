// Throughput of the backward's per-element math (the evo_bwd_pb.cu / round-1 fused kernel compute loop) on register
// data, 16 warps per SM (4 per sub-partition), in variants that drop one part at a time:
//   0 full:    x = bias·log2e - lse2 (FFMA2), x += S·scale·log2e (FFMA2), p = ex2 x2, dS = p·(dP - D)
//              (FADD2, FMUL2), Σ += dS (FADD2), pack p and dS to bf16x2 (2 F2FP)
//   1 no F2FP (packs by PRMT truncation)   2 no MUFU (ex2 -> FMUL)   3 only MUFU + F2FP
//   4 full, but P packed by F2FP and dS by PRMT
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o bwd_math bwd_math.cu
#include <cstdio>
#include "../../paper_2404_11068_b200/csrc/evo_common.cuh"
using namespace evo;

__device__ __forceinline__ uint32_t prmt_hi(float a, float b) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(__float_as_uint(a)), "r"(__float_as_uint(b)));
  return r;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(unsigned long long* out, int iters, uint32_t* sink) {
  const int tid = threadIdx.x;
  uint32_t rs[16], rd[16], acc[16], bu[8];
  float nl[16], nd[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    rs[i] = __float_as_uint(0.01f * (tid + i));
    rd[i] = __float_as_uint(0.02f * (tid - i));
    acc[i] = 0u;
    nl[i] = -1.f - 0.001f * i;
    nd[i] = -0.5f + 0.001f * i;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) bu[i] = 0x3f803f80u + i;
  const uint64_t sl2 = f2_pack(0.25f, 0.25f), l2e2 = f2_pack(kLog2e, kLog2e);
  uint32_t xo = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t pk[8], dk2[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int i = 2 * e;
      const uint64_t nl2 = f2_pack(nl[i], nl[i + 1]);
      const uint64_t nd2 = f2_pack(nd[i], nd[i + 1]);
      uint64_t x = f2_fma(bf16x2_to_f2(bu[e] ^ it), l2e2, nl2);
      x = f2_fma(((uint64_t)rs[i + 1] << 32) | rs[i], sl2, x);
      float x0, x1;
      f2_unpack(x, x0, x1);
      float p0, p1;
      if (MODE == 2) { p0 = x0 * 0.5f; p1 = x1 * 0.5f; }
      else { p0 = fast_exp2(x0); p1 = fast_exp2(x1); }
      if (MODE == 3) {
        pk[e] = pack_bf16(p0, p1);
        dk2[e] = pack_bf16(p1, p0);
        continue;
      }
      const uint64_t p2 = f2_pack(p0, p1);
      const uint64_t dd = f2_mul(p2, f2_add(((uint64_t)rd[i + 1] << 32) | rd[i], nd2));
      float d0, d1;
      f2_unpack(dd, d0, d1);
      const uint64_t s2 = f2_add(((uint64_t)acc[i + 1] << 32) | acc[i], dd);
      float a0, a1;
      f2_unpack(s2, a0, a1);
      acc[i] = __float_as_uint(a0);
      acc[i + 1] = __float_as_uint(a1);
      if (MODE == 1) { pk[e] = prmt_hi(p0, p1); dk2[e] = prmt_hi(d0, d1); }
      else if (MODE == 4) { pk[e] = pack_bf16(p0, p1); dk2[e] = prmt_hi(d0, d1); }
      else { pk[e] = pack_bf16(p0, p1); dk2[e] = pack_bf16(d0, d1); }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) xo ^= pk[e] + dk2[e];
#pragma unroll
    for (int i = 0; i < 16; ++i) rs[i] ^= xo & 1u;
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  uint32_t s = xo;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 0x12345678u) sink[0] = s;
}

int main() {
  unsigned long long* d;
  uint32_t* s;
  cudaMalloc(&d, 8 * 148);
  cudaMalloc(&s, 4);
  const char* names[5] = {"full", "no F2FP (PRMT packs)", "no MUFU", "MUFU + F2FP only", "dS by PRMT"};
  for (int mode = 0; mode < 5; ++mode)
    for (int nw : {8, 16}) {
      auto f = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : mode == 3 ? k<3> : k<4>;
      const int iters = 2000;
      f<<<148, nw * 32>>>(d, 10, s);
      f<<<148, nw * 32>>>(d, iters, s);
      cudaDeviceSynchronize();
      unsigned long long h;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      // elements per SM sub-partition per iteration: nw/4 warps x 32 lanes x 16 elements
      const double elems = nw / 4.0 * 32 * 16;
      printf("%-22s warps/SM=%2d: %.3f cycles per element per sub-partition (%.0f cycles per 2048)\n",
             names[mode], nw, (double)h / iters / elems, (double)h / iters / elems * 2048);
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
