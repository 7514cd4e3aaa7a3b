// The fused backward's per-sub-tile-pair MMA mix, issued back to back on fresh operands (one
// thread, no synchronisation), to separate the tcgen05 cost of the mix itself from the kernel's
// hand-off pipeline: per pair  Sᵀ,dPᵀ (SS, N=64, K-major SW64, 2 K-steps each at D=32),
// then per sub-tile (x2) dV (TS, N=32, B MN-major) x2 K-steps and dK (SS, A K-major SW64 /
// B MN-major) x2, plus half a tile's dQ (SS, A and B MN-major) x4.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_mix mma_mix.cu
#include <cstdio>
#include "../../paper_2404_11068_b200/csrc/evo_common.cuh"
using namespace evo;

template <int MODE>
__global__ void __launch_bounds__(128, 1) k(unsigned long long* out, int npairs) {
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
    constexpr uint32_t kRow = 64;  // DP = 32 rows
    constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, 0, 0);
    constexpr uint32_t idesc_kv = make_idesc_bf16(128, 32, 0, 1);
    constexpr uint32_t idesc_q = make_idesc_bf16(128, 32, 1, 1);
    const uint32_t tS = tm + 256, tdV = tm + 384, tdK = tm + 416, tdQ = tm + 448, tP = tm + 480;
    unsigned long long t0 = clock64();
    for (int p = 0; p < npairs; ++p) {
      const uint32_t r = (uint32_t)(p & 3);
      const uint32_t kb = s0 + r * 16384, qb = s0 + 65536 + r * 16384, db = s0 + 131072 + r * 8192;
      if (MODE != 2) {
        for (int kk = 0; kk < 2; ++kk)
          umma_bf16(tS, make_sdesc(kb + kk * 32, 16, 8 * kRow, kSw64), make_sdesc(qb + kk * 32, 16, 8 * kRow, kSw64),
                    idesc_s, kk > 0);
        for (int kk = 0; kk < 2; ++kk)
          umma_bf16(tS + 64, make_sdesc(kb + 8192 + kk * 32, 16, 8 * kRow, kSw64),
                    make_sdesc(qb + 8192 + kk * 32, 16, 8 * kRow, kSw64), idesc_s, kk > 0);
      }
      if (MODE != 1) {
        for (int sub = 0; sub < 2; ++sub) {
          for (int kk = 0; kk < 2; ++kk)
            umma_bf16_ts(tdV, tP + sub * 16 + kk * 8, make_sdesc(qb + 8192 + kk * 16 * kRow, 16384, 8 * kRow, kSw64),
                         idesc_kv, 1);
          for (int kk = 0; kk < 2; ++kk)
            umma_bf16(tdK, make_sdesc(db + kk * 32, 16, 512, kSw64),
                      make_sdesc(qb + kk * 16 * kRow, 16384, 8 * kRow, kSw64), idesc_kv, 1);
        }
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(tdQ, make_sdesc(db + kk * 1024, 8192, 512, kSw64),
                    make_sdesc(kb + kk * 16 * kRow, 16384, 8 * kRow, kSw64), idesc_q, 1);
      }
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

template <int MODE>
void run(const char* name, int mmas_per_pair) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  auto f = k<MODE>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  f<<<148, 128, 200 * 1024>>>(d, 8);
  const int np = 1024;
  f<<<148, 128, 200 * 1024>>>(d, np);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-44s %7.1f cyc per pair, %5.1f per MMA [%s]\n", name, (double)h / np,
         (double)h / np / mmas_per_pair, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>("full mix (S/dP 4 + dV 4 + dK 4 + dQ 4)", 16);
  run<1>("S/dP only (4, N=64)", 4);
  run<2>("gradients only (dV 4 TS + dK 4 + dQ 4)", 12);
  return 0;
}
