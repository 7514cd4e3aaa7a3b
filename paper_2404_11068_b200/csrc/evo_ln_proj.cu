// evo_ln_proj.cu — fused LayerNorm + batched q/k/v/g projection (include/evo_ln_proj.h;
// SURVEY.md §8(f) row f2; "fused LayerNorm, MHA and its previous four GEMMs",
// L296-297 GEMM batching of the four independent linear layers).
//
// One CTA per 128-row tile of x, 256 threads:
//   warp 0      TMA producer: the x tile once (C/64 boxes of [128 rows][64 c], SW128), then the
//               W tiles [NT rows of W][64 c] through a kStages ring, in (n-tile, k-block) order
//   warp 1      tcgen05.mma issuer: acc[nt&1] (TMEM, 128 lanes x NT fp32) = y_tile · W_tileᵀ
//   warp 2      TMEM allocator (512 columns: two NT <= 256 accumulators)
//   warps 4..7  thread t = row t: LayerNorm of the tile IN PLACE in shared memory (two passes
//               over the row for μ and σ², a third writes y in the same swizzled layout — the
//               MMA A operand), then the epilogue of every n-tile: tcgen05.ld, + b, bf16, store.
// The stacked weight matrix ([4·H·D, C] bf16, <= 2 MB) stays L2-resident across CTAs; x is read
// once and `out` written once, so the op is HBM-bound for the AF2 shapes.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>

#include "evo_kernels.cuh"
#include "evo_ln_proj.h"

namespace evo {
namespace {

constexpr int kStages = 4;
constexpr int kThreads = 256;

struct LnProjArgs {
  int64_t M;
  int N, NT;
  float eps;
  int64_t out_ld;
  const float *gamma, *beta, *b;
  __nv_bfloat16* out;
  float *mean, *rstd;
};

EVO_DEV void tma_load_2d(uint32_t dst, const void* tmap, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}

template <int C>
__global__ void __launch_bounds__(kThreads, 1)
    ln_proj_fwd_kernel(const __grid_constant__ CUtensorMap tm_x,
                       const __grid_constant__ CUtensorMap tm_w, const LnProjArgs a) {
  constexpr int KB = C / 64;                 // 64-channel K blocks
  constexpr uint32_t kXBlock = 128 * 128;    // [128 rows][64 c] bf16
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sX = base;
  const uint32_t sW = sX + KB * kXBlock;
  const uint32_t stage_bytes = (uint32_t)a.NT * 128u;
  const uint32_t sBar = sW + kStages * 256u * 128u;
  const uint32_t bar_x = sBar, bar_y = sBar + 8;
  const uint32_t wfull = sBar + 16, wfree = wfull + 8 * kStages;
  const uint32_t accfull = wfree + 8 * kStages, accfree = accfull + 16;
  const uint32_t tmem_slot = accfree + 16;

  const uint32_t warp = warp_id(), lane = lane_id();
  const int64_t row0 = (int64_t)blockIdx.x * 128;
  const int n_tiles = a.N / a.NT;

  if (threadIdx.x == 0) {
    mbar_init(bar_x, 1);
    mbar_init(bar_y, 128);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(wfull + 8 * s, 1);
      mbar_init(wfree + 8 * s, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(accfull + 8 * i, 1);
      mbar_init(accfree + 8 * i, 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem_raw + (tmem_slot - smem_u32(smem_raw)));

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_x);
      tma_prefetch_desc(&tm_w);
      mbar_arrive_expect_tx(bar_x, KB * kXBlock);
      for (int kb = 0; kb < KB; ++kb)
        tma_load_2d(sX + kb * kXBlock, &tm_x, bar_x, kb * 64, (int)row0);
      int it = 0;
      for (int nt = 0; nt < n_tiles; ++nt)
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % kStages, round = it / kStages;
          if (round > 0) mbar_wait(wfree + 8 * s, (round - 1) & 1);
          mbar_arrive_expect_tx(wfull + 8 * s, stage_bytes);
          tma_load_2d(sW + s * 256u * 128u, &tm_w, wfull + 8 * s, kb * 64, nt * a.NT);
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc_bf16(128, (uint32_t)a.NT, 0, 0);
      mbar_wait(bar_y, 0);
      tc_fence_after();
      int it = 0;
      for (int nt = 0; nt < n_tiles; ++nt) {
        const int ab = nt & 1;
        if (nt >= 2) mbar_wait(accfree + 8 * ab, ((nt >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t tacc = tmem + ab * 256;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const int s = it % kStages, round = it / kStages;
          mbar_wait(wfull + 8 * s, round & 1);
          tc_fence_after();
          const uint32_t wb = sW + s * 256u * 128u, xb = sX + kb * kXBlock;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16(tacc, make_sdesc(xb + kk * 32, 16, 1024, kSw128),
                      make_sdesc(wb + kk * 32, 16, 1024, kSw128), idesc, (kb | kk) != 0);
          umma_commit(wfree + 8 * s);
        }
        umma_commit(accfull + 8 * ab);
      }
    }
  } else if (warp >= 4) {
    const uint32_t t = threadIdx.x - 128;  // tile row == TMEM lane
    const int64_t row = row0 + t;
    // ---- LayerNorm in place (row t of every K block; SW128: chunk ch at ch ^ (t & 7))
    mbar_wait(bar_x, 0);
    float sum = 0.f;
#pragma unroll 1
    for (int kb = 0; kb < KB; ++kb)
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        const uint4 v = ld_shared_v4(sX + kb * kXBlock + t * 128 + ((ch ^ (t & 7)) << 4));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) sum += bf16_lo(w[e]) + bf16_hi(w[e]);
      }
    const float mu = sum * (1.f / C);
    float ss = 0.f;
#pragma unroll 1
    for (int kb = 0; kb < KB; ++kb)
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        const uint4 v = ld_shared_v4(sX + kb * kXBlock + t * 128 + ((ch ^ (t & 7)) << 4));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float d0 = bf16_lo(w[e]) - mu, d1 = bf16_hi(w[e]) - mu;
          ss += d0 * d0 + d1 * d1;
        }
      }
    const float rs = rsqrtf(ss * (1.f / C) + a.eps);
    if (row < a.M) {
      if (a.mean) a.mean[row] = mu;
      if (a.rstd) a.rstd[row] = rs;
    }
#pragma unroll 1
    for (int kb = 0; kb < KB; ++kb)
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        const uint32_t addr = sX + kb * kXBlock + t * 128 + ((ch ^ (t & 7)) << 4);
        const uint4 v = ld_shared_v4(addr);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
        const int c0 = kb * 64 + ch * 8;
        const float4 g0 = __ldg(reinterpret_cast<const float4*>(a.gamma + c0));
        const float4 g1 = __ldg(reinterpret_cast<const float4*>(a.gamma + c0 + 4));
        const float4 b0 = __ldg(reinterpret_cast<const float4*>(a.beta + c0));
        const float4 b1 = __ldg(reinterpret_cast<const float4*>(a.beta + c0 + 4));
        const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
        uint32_t o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          o[e] = pack_bf16((bf16_lo(w[e]) - mu) * rs * gg[2 * e] + bb[2 * e],
                           (bf16_hi(w[e]) - mu) * rs * gg[2 * e + 1] + bb[2 * e + 1]);
        st_shared_v4(addr, o[0], o[1], o[2], o[3]);
      }
    fence_proxy_async_smem();
    mbar_arrive(bar_y);

    // ---- epilogue: acc[nt&1] -> (+ b) -> bf16 -> out[row, nt·NT + ...]
    const uint32_t lane_base = (uint32_t)(warp & 3) * 32u << 16;
    __nv_bfloat16* orow = a.out + row * a.out_ld;
#pragma unroll 1
    for (int nt = 0; nt < n_tiles; ++nt) {
      const int ab = nt & 1;
      mbar_wait(accfull + 8 * ab, (nt >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int cc = 0; cc < a.NT; cc += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_base + ab * 256 + cc, r);
        tmem_wait_ld();
        const int n0 = nt * a.NT + cc;
        if (row < a.M) {
          uint4* dst = reinterpret_cast<uint4*>(orow + n0);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float f[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(r[8 * q + e]);
            if (a.b) {
              const float4 b0 = __ldg(reinterpret_cast<const float4*>(a.b + n0 + 8 * q));
              const float4 b1 = __ldg(reinterpret_cast<const float4*>(a.b + n0 + 8 * q + 4));
              f[0] += b0.x; f[1] += b0.y; f[2] += b0.z; f[3] += b0.w;
              f[4] += b1.x; f[5] += b1.y; f[6] += b1.z; f[7] += b1.w;
            }
            dst[q] = make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]),
                                pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
          }
        }
      }
      tc_fence_before();
      mbar_arrive(accfree + 8 * ab);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

size_t smem_bytes(int C) { return 1024 + (size_t)(C / 64) * 16384 + kStages * 256 * 128 + 256; }

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

bool make_2d_map(CUtensorMap* m, const void* ptr, int64_t cols, int64_t rows, int64_t ld,
                 int box_rows) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)(rows > 0 ? rows : 1)};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

evo_status_t lp_fail(evo_status_t s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  set_error_detail(buf);  // evo_last_error_detail() (evo_api.cu)
  return s;
}
bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace
}  // namespace evo

extern "C" evo_status_t evo_ln_proj_fwd(const evo_ln_proj_desc_t* d, const void* x,
                                        const float* gamma, const float* beta, const void* W,
                                        const float* b, void* out, float* mean, float* rstd,
                                        void* stream) {
  using namespace evo;
  if (!d) return lp_fail(EVO_E_INVALID, "desc is NULL");
  if (d->rows < 0) return lp_fail(EVO_E_SHAPE, "rows = %lld < 0", (long long)d->rows);
  if (d->C != 64 && d->C != 128 && d->C != 256)
    return lp_fail(EVO_E_UNSUPPORTED, "C = %d (supported: 64, 128, 256)", d->C);
  if (d->N <= 0 || d->N % 64 != 0 || d->N > 4096)
    return lp_fail(EVO_E_UNSUPPORTED, "N = %d must be a positive multiple of 64, <= 4096", d->N);
  if (!(d->eps > 0.f)) return lp_fail(EVO_E_INVALID, "eps must be > 0");
  if (d->x_ld < d->C || d->x_ld % 8 != 0)
    return lp_fail(EVO_E_ALIGN, "x_ld = %lld must be >= C and a multiple of 8", (long long)d->x_ld);
  if (d->out_ld < d->N || d->out_ld % 8 != 0)
    return lp_fail(EVO_E_ALIGN, "out_ld = %lld must be >= N and a multiple of 8",
                   (long long)d->out_ld);
  if (d->rows == 0) return EVO_OK;
  if (!x || !gamma || !beta || !W || !out)
    return lp_fail(EVO_E_INVALID, "x, gamma, beta, W and out are required");
  if (!al16(x) || !al16(W) || !al16(out) || !al16(gamma) || !al16(beta) || (b && !al16(b)))
    return lp_fail(EVO_E_ALIGN, "tensors must be 16-byte aligned");

  LnProjArgs a{};
  a.M = d->rows;
  a.N = d->N;
  a.NT = d->N % 256 == 0 ? 256 : (d->N % 128 == 0 ? 128 : 64);
  a.eps = d->eps;
  a.out_ld = d->out_ld;
  a.gamma = gamma;
  a.beta = beta;
  a.b = b;
  a.out = static_cast<__nv_bfloat16*>(out);
  a.mean = mean;
  a.rstd = rstd;
  CUtensorMap tx, tw;
  if (!make_2d_map(&tx, x, d->C, d->rows, d->x_ld, 128) ||
      !make_2d_map(&tw, W, d->C, d->N, d->C, a.NT))
    return lp_fail(EVO_E_CUDA, "cuTensorMapEncodeTiled failed");
  const size_t smem = smem_bytes(d->C);
  const dim3 grid((unsigned)((d->rows + 127) / 128));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  switch (d->C) {
#define EVO_LP_CASE(CC)                                                                     \
  case CC:                                                                                  \
    e = cudaFuncSetAttribute(ln_proj_fwd_kernel<CC>,                                        \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);       \
    if (e == cudaSuccess) ln_proj_fwd_kernel<CC><<<grid, kThreads, smem, st>>>(tx, tw, a);  \
    break;
    EVO_LP_CASE(64)
    EVO_LP_CASE(128)
    EVO_LP_CASE(256)
#undef EVO_LP_CASE
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? EVO_OK : lp_fail(EVO_E_CUDA, "ln_proj_fwd: %s", cudaGetErrorString(e));
}
