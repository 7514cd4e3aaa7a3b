// tcgen05.mma (M = 128, K = 16, bf16) throughput when every MMA reads FRESH operands (A and B
// cycle through distinct shared-memory tiles, as in the backward), vs the same tile repeated.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_fresh mma_fresh.cu
#include <cstdio>
#include "../../paper_2404_11068_b200/csrc/evo_common.cuh"
using namespace evo;

// MODE 0: same A/B every MMA; 1: A and B rotate over 8 tiles (K-major SW64); 2: rotate, B MN-major;
// 3: TS (A from TMEM), B rotates MN-major; 4: rotate A K-major SW128 128-B rows (the Sᵀ form);
// 5: rotate, A AND B MN-major (the backward's dQ = dS·K: A read from the dSᵀ blocks)
template <int N, int MODE, int NACC = 2>
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
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u ^ i;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc_bf16(128, N, MODE == 5 ? 1 : 0, (MODE == 2 || MODE == 3 || MODE == 5) ? 1 : 0);
    unsigned long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const int r = MODE == 0 ? 0 : (i & 7);
      const uint32_t abase = s0 + r * 16384, bbase = s0 + 131072 + r * 8192;
      const uint64_t ad = MODE == 4 ? make_sdesc(abase, 16, 1024, kSw128)
                          : MODE == 5 ? make_sdesc(abase, 8192, 512, kSw64)
                                      : make_sdesc(abase, 16, 512, kSw64);
      const uint64_t bd = (MODE == 2 || MODE == 3 || MODE == 5) ? make_sdesc(bbase, 8192, 512, kSw64)
                                                                : make_sdesc(bbase, 16, 512, kSw64);
      const uint32_t d = tm + (uint32_t)((i % NACC) * N);
      if (MODE == 3) umma_bf16_ts(d, tm + 256 + (i & 7) * 8, bd, idesc, 1);
      else umma_bf16(d, ad, bd, idesc, 1);
    }
    umma_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tm);
}

template <int N, int MODE, int NACC = 2>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  auto f = k<N, MODE, NACC>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  f<<<148, 128, 200 * 1024>>>(d, 16);
  f<<<148, 128, 200 * 1024>>>(d, 4096);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("N=%3d nacc=%d %-34s %6.1f cyc/MMA [%s]\n", N, NACC, name, (double)h / 4096, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<32, 1, 1>("SS fresh, ONE accumulator (dependent)");
  run<32, 1, 2>("SS fresh, 2 accumulators alternating");
  run<32, 1, 4>("SS fresh, 4 accumulators");
  run<32, 2, 1>("SS fresh Bmn, ONE accumulator");
  run<32, 3, 1>("TS fresh, ONE accumulator");
  run<32, 3, 2>("TS fresh, 2 accumulators");
  run<64, 1, 1>("SS fresh N64, ONE accumulator");
  run<32, 0, 1>("SS same tiles, ONE accumulator");
  run<32, 0>("SS same tiles");
  run<32, 1>("SS fresh tiles (K-major)");
  run<32, 2>("SS fresh tiles (B MN-major)");
  run<32, 3>("TS fresh B (MN-major)");
  run<64, 0>("SS same tiles");
  run<64, 4>("SS fresh tiles (A SW128)");
  run<64, 1>("SS fresh tiles");
  run<128, 1>("SS fresh tiles");
  run<256, 1>("SS fresh tiles");
  run<128, 0>("SS same tiles");
  run<32, 5, 1>("SS fresh A+B MN-major (dQ), ONE acc");
  run<32, 5>("SS fresh A+B MN-major (dQ)");
  return 0;
}
