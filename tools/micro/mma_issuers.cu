// tcgen05.mma issue-rate probes for the backward's small-N MMAs (M = 128 / 64, N = 32):
//   (1) 1, 2 or 4 issuing threads (one per warp, disjoint accumulators) on one SM: is the
//       ~46-cycle-per-MMA floor per issuing thread or per SM tensor pipe?
//   (2) M = 64, N = 32 (cta_group::1)
//   (3) cta_group::2, M = 256, N = 32 on a CTA pair (cluster of 2): cycles per pair MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_issuers mma_issuers.cu
#include <cstdio>
#include "../../paper_2404_11068_b200/csrc/evo_common.cuh"
using namespace evo;

template <int M, int N, int NISS>
__global__ void __launch_bounds__(128, 1) k1(unsigned long long* out, int n_mma) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[4];
  const uint32_t s0 = smem_u32(smem);
  const int w = threadIdx.x >> 5;
  if (threadIdx.x < 32) tmem_alloc<512>(smem_u32(&slot));
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&bar[i]), 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  __syncthreads();
  unsigned long long t0 = clock64();
  if (w < NISS && (threadIdx.x & 31) == 0) {
    constexpr uint32_t idesc = make_idesc_bf16(M, N, 0, 0);
    const uint64_t ad = make_sdesc(s0 + w * 16384, 16, 512, kSw64);
    const uint64_t bd = make_sdesc(s0 + 65536 + w * 8192, 16, 512, kSw64);
    const uint32_t d = tm + (uint32_t)(w * 64);
    for (int i = 0; i < n_mma; ++i) umma_bf16(d + (i & 1) * N, ad, bd, idesc, 1);
    umma_commit(smem_u32(&bar[w]));
    mbar_wait(smem_u32(&bar[w]), 0);
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tm);
}

__device__ __forceinline__ uint32_t my_cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int N, bool FRESH = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k2(unsigned long long* out, int n_mma) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t s0 = smem_u32(smem);
  const uint32_t rank = my_cta_rank();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tm = slot;
  unsigned long long t0 = clock64();
  if (rank == 0 && threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc_bf16(256, N, 0, 0);
    for (int i = 0; i < n_mma; ++i) {
      const int r = FRESH ? (i & 7) : 0;
      const uint64_t ad = make_sdesc(s0 + r * 8192, 16, 512, kSw64);
      const uint64_t bd = make_sdesc(s0 + 65536 + r * 4096, 16, 512, kSw64);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm + (uint32_t)((i & 1) * N)),
          "l"(ad), "l"(bd), "r"(idesc), "r"(1u)
          : "memory");
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)),
        "h"((uint16_t)3)
        : "memory");
  }
  if (threadIdx.x == 0) mbar_wait(smem_u32(&bar), 0);
  __syncthreads();
  unsigned long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <class F>
void run(F f, const char* name, int grid, double mmas_per_cta_per_n, double flop_per_mma) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  const int n = 2048;
  f<<<grid, 128, 131072>>>(d, 16);
  f<<<grid, 128, 131072>>>(d, n);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / (n * mmas_per_cta_per_n);
  printf("%-34s %7.1f cyc per MMA per CTA  -> %6.0f flop/clk/SM  [%s]\n", name, per,
         flop_per_mma / per, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run(k1<128, 32, 1>, "M128 N32, 1 issuer", 148, 1, 2.0 * 128 * 32 * 16);
  run(k1<128, 32, 2>, "M128 N32, 2 issuers", 148, 2, 2.0 * 128 * 32 * 16);
  run(k1<128, 32, 4>, "M128 N32, 4 issuers", 148, 4, 2.0 * 128 * 32 * 16);
  run(k1<128, 64, 2>, "M128 N64, 2 issuers", 148, 2, 2.0 * 128 * 64 * 16);
  run(k1<128, 128, 1>, "M128 N128, 1 issuer", 148, 1, 2.0 * 128 * 128 * 16);
  run(k1<64, 32, 1>, "M64 N32, 1 issuer", 148, 1, 2.0 * 64 * 32 * 16);
  run(k1<64, 64, 1>, "M64 N64, 1 issuer", 148, 1, 2.0 * 64 * 64 * 16);
  // pair: each pair MMA does 2*256*N*16 flops over 2 SMs -> per SM 256*N*16
  run(k2<32>, "cta_group::2 M256 N32 (per SM)", 148, 1, 2.0 * 128 * 32 * 16);
  run(k2<64>, "cta_group::2 M256 N64 (per SM)", 148, 1, 2.0 * 128 * 64 * 16);
  run(k2<128>, "cta_group::2 M256 N128 (per SM)", 148, 1, 2.0 * 128 * 128 * 16);
  run(k2<32, true>, "cta_group::2 M256 N32 fresh", 148, 1, 2.0 * 128 * 32 * 16);
  run(k2<64, true>, "cta_group::2 M256 N64 fresh", 148, 1, 2.0 * 128 * 64 * 16);
  run(k2<128, true>, "cta_group::2 M256 N128 fresh", 148, 1, 2.0 * 128 * 128 * 16);
  run(k2<256, true>, "cta_group::2 M256 N256 fresh", 148, 1, 2.0 * 128 * 256 * 16);
  return 0;
}
