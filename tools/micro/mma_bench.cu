// tcgen05.mma (kind::f16, bf16 in, fp32 accumulate, cta_group::1, M = 128) issue throughput and
// latency on one SM per CTA, for the small-N shapes the backward uses.  Operands are whatever
// the shared memory holds (timing only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_bench mma_bench.cu
#include <cstdio>
#include "../../paper_2404_11068_b200/csrc/evo_common.cuh"
using namespace evo;

// MODE 0: SS, 1: TS (A from TMEM), 2: SS with B MN-major, 3: SS with A and B MN-major (SW64,
// the backward's dV/dK and dQ operand forms).  NACC accumulators rotated or 1 (chained D).
template <int N, int MODE, int NACC>
__global__ void __launch_bounds__(128, 1) k(unsigned long long* out, int n_mma) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t s0 = smem_u32(smem);
  if (threadIdx.x < 32) tmem_alloc<512>(smem_u32(&slot));
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc_bf16(128, N, MODE == 3 ? 1 : 0, MODE >= 2 ? 1 : 0);
    const uint64_t ad = MODE == 3 ? make_sdesc(s0, 8192, 512, kSw64) : make_sdesc(s0, 16, 512, kSw64);
    const uint64_t bd = MODE >= 2 ? make_sdesc(s0 + 65536, 16384, 512, kSw64)
                                  : make_sdesc(s0 + 65536, 16, 512, kSw64);
    // latency: one MMA, commit, wait
    unsigned long long t0 = clock64();
    if (MODE != 1) umma_bf16(tm, ad, bd, idesc, 0);
    else umma_bf16_ts(tm, tm + 256, bd, idesc, 0);
    umma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    unsigned long long t1 = clock64();
    // throughput: n_mma back to back
    for (int i = 0; i < n_mma; ++i) {
      const uint32_t d = tm + (uint32_t)((i % NACC) * N) % 256;
      if (MODE != 1) umma_bf16(d, ad, bd, idesc, 1);
      else umma_bf16_ts(d, tm + 256, bd, idesc, 1);
    }
    umma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 1);
    unsigned long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tm);
}

template <int N, int MODE, int NACC>
void run(unsigned long long* d) {
  auto f = k<N, MODE, NACC>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  const int n = 4096;
  f<<<148, 128, 131072>>>(d, 16);
  f<<<148, 128, 131072>>>(d, n);
  cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double per = (double)h[1] / n;
  const char* mn[4] = {"SS", "TS", "SS-Bmn", "SS-ABmn"};
  printf("N=%3d %-7s nacc=%d: latency %5llu cyc, %6.1f cyc/MMA (K=16) -> %6.0f flop/clk/SM (%.0f%% of 8192)\n",
         N, mn[MODE], NACC, h[0], per, 2.0 * 128 * N * 16 / per,
         100.0 * 2.0 * 128 * N * 16 / per / 8192);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  run<32, 0, 1>(d);
  run<32, 0, 4>(d);
  run<32, 1, 1>(d);
  run<32, 1, 4>(d);
  run<64, 0, 1>(d);
  run<64, 0, 4>(d);
  run<128, 0, 1>(d);
  run<128, 0, 2>(d);
  run<256, 0, 1>(d);
  run<16, 0, 4>(d);
  run<32, 2, 1>(d);
  run<32, 2, 4>(d);
  run<32, 3, 1>(d);
  run<32, 3, 4>(d);
  run<64, 2, 1>(d);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
