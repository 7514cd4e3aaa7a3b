// evo_ln_proj.cu — fused LayerNorm + batched q/k/v/g projection (include/evo_ln_proj.h;
// SURVEY.md §8(f) row f2; "fused LayerNorm, MHA and its previous four GEMMs",
// L296-297 GEMM batching of the four independent linear layers).
//
// Persistent kernel on 2-CTA clusters, one CTA per SM, each CTA looping over 128-row tiles of x
// (the two CTAs of a cluster take adjacent tiles), 512 threads (16 warps):
//   warp 3      x producer: TMA of the tile's C/64 boxes [128 rows][64 c] (SW128) into one of two
//               x buffers, as soon as the MMAs of the tile two back released it
//   warps 8..15 LayerNorm, 4 lanes per row: the row is read once into registers (μ, then σ²
//               about μ, fp32), y = (x − μ)·rstd·γ + β written back IN PLACE (same swizzle: it
//               is the MMA A operand)
//   warp 0      W producer: stages [NT rows of W][64 c] through a kSt-deep ring, in (tile,
//               n-tile, k-block) order.  Both CTAs of the cluster need the same W sequence, so
//               each loads HALF of every stage with .multicast::cluster into both CTAs (halving
//               the L2 -> SM traffic that bounds this op: W is re-read per 128-row tile); a
//               stage is refilled once the MMAs of BOTH CTAs released it (commit multicast)
//   warp 1      tcgen05.mma issuer: acc[g & 1] (TMEM 128 lanes x NT <= 256 fp32) = y · W_ntᵀ
//   warp 2      TMEM allocator (512 columns = two accumulators)
//   warps 4..7  epilogue, thread = row: tcgen05.ld, + b, bf16, into the warp's own swizzled
//               [32 rows][32 cols] staging tile, TMA store by lane 0 (two buffers per warp,
//               bulk-group tracked; warps never wait on each other)
// γ, β and b are staged in shared memory once per CTA (lanes then read them as broadcasts).
// The x load and LayerNorm of tile i+1, the MMAs of tile i and the stores of tile i−1 overlap.
// HBM traffic = x read once + out written once (f2 row).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>

#include "evo_kernels.cuh"
#include "evo_ln_proj.h"

#ifndef LP_TL  // tools/lp_timeline.py: globaltimer stamps into a.mean (uint64 [grid][64])
#define LP_TL 0
#endif
#if LP_TL
#define LP_STAMP(slot)                                                                      \
  do {                                                                                      \
    uint64_t t_;                                                                            \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                  \
    reinterpret_cast<uint64_t*>(a.mean)[blockIdx.x * 64 + (slot)] = t_;                     \
  } while (0)
#else
#define LP_STAMP(slot) \
  do {                 \
  } while (0)
#endif

namespace evo {
namespace {

constexpr int kThreads = 512;
constexpr uint32_t kXBlock = 128 * 128;  // [128 rows][64 c] bf16, SW128
constexpr uint32_t kWStage = 256 * 128;  // [NT <= 256 rows][64 c] bf16, SW128
constexpr uint32_t kOStage = 128 * 64;   // 4 warps x [32 rows][32 cols] bf16 staging, SW64
constexpr int kMaxN = 2048;              // bias staged in smem

struct LnProjArgs {
  int64_t M;
  int N, NT, n_row_tiles, n_pairs;
  int ln;  // 1: LayerNorm the x tile first (evo_ln_proj_fwd); 0: plain linear (evo_linear_fwd)
  float eps;
  const float *gamma, *beta, *b;
  float *mean, *rstd;
};

template <int C>
__host__ __device__ constexpr int w_stages() { return C == 256 ? 2 : 4; }
template <int C>
constexpr size_t lp_smem() {
  return 1024 + 2 * (C / 64) * kXBlock + w_stages<C>() * kWStage + 2 * kOStage + 8 * C +
         4 * kMaxN + 256;
}

EVO_DEV void tma_load_2d(uint32_t dst, const void* tmap, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
// same box delivered to the same smem offset (and mbarrier offset) of every CTA in `mask`
EVO_DEV void tma_load_2d_mc(uint32_t dst, const void* tmap, uint32_t bar, int c0, int c1,
                            uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
// arrive on the mbarrier at this offset in every CTA of `mask` once this thread's MMAs complete
EVO_DEV void umma_commit_mc(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar),
      "h"(mask)
      : "memory");
}
EVO_DEV void tma_store_2d(const void* tmap, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(src), "r"(c0), "r"(c1)
               : "memory");
}
EVO_DEV float4 ld_shared_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
EVO_DEV void bulk_wait_group_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }

template <int C>
__global__ void __launch_bounds__(kThreads, 1)
    ln_proj_fwd_kernel(const __grid_constant__ CUtensorMap tm_x,
                       const __grid_constant__ CUtensorMap tm_w,
                       const __grid_constant__ CUtensorMap tm_o, const LnProjArgs a) {
  constexpr int KB = C / 64;  // 64-channel K blocks
  constexpr int kSt = w_stages<C>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sX = base;                   // x / y tiles: 2 x KB x kXBlock
  const uint32_t sW = sX + 2 * KB * kXBlock;  // W ring
  const uint32_t sO = sW + kSt * kWStage;     // output staging
  const uint32_t sGB = sO + 2 * kOStage;      // γ [C], β [C] fp32
  const uint32_t sB = sGB + 8 * C;            // b [N] fp32 (zeros when b == NULL)
  const uint32_t sBar = sB + 4 * kMaxN;
  const uint32_t xfull = sBar, xfree = sBar + 16, yready = sBar + 32;
  const uint32_t wfull = sBar + 48, wfree = wfull + 8 * kSt;
  const uint32_t accfull = wfree + 8 * kSt, accfree = accfull + 16;
  const uint32_t tmem_slot = accfree + 16;

  const uint32_t warp = warp_id(), lane = lane_id();
  const int rank = (int)cluster_ctarank();           // 0 / 1 within the CTA pair
  const int cid = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  const int n_tiles = a.N / a.NT;
  // tiles of this CTA: 2p + rank for pairs p = cid, cid + n_clusters, ...  (a tile index past
  // the end is a dummy: zero-filled load, no statistics, clipped stores — it keeps the pair's W
  // sequences in step)
#define LP_TILE_LOOP(i) \
  for (int p = cid, i = 0; p < a.n_pairs; p += n_clusters, ++i)

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(xfull + 8 * i, 1);
      mbar_init(xfree + 8 * i, 1);
      mbar_init(yready + 8 * i, 256);
    }
    for (int s = 0; s < kSt; ++s) {
      mbar_init(wfull + 8 * s, 1);
      mbar_init(wfree + 8 * s, 2);  // the MMA commits of both CTAs
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(accfull + 8 * i, 1);
      mbar_init(accfree + 8 * i, 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  {  // per-CTA parameter staging: every lane of a warp then reads the same word (broadcast)
    float* gb = reinterpret_cast<float*>(smem_raw + (sGB - smem_u32(smem_raw)));
    for (int k = threadIdx.x; k < 2 * C + a.N; k += kThreads)
      gb[k] = k < 2 * C ? (a.ln ? (k < C ? a.gamma[k] : a.beta[k - C]) : 0.f)
                        : (a.b ? a.b[k - 2 * C] : 0.f);
  }
  tc_fence_before();
  cluster_sync_all();  // barriers of both CTAs initialised before any multicast lands
  tc_fence_after();
  const uint32_t tmem =
      *reinterpret_cast<volatile uint32_t*>(smem_raw + (tmem_slot - smem_u32(smem_raw)));
  if (threadIdx.x == 0) LP_STAMP(0);

  if (warp == 3) {
    // ------------------------------------------------------------ x producer
    if (lane == 0) {
      tma_prefetch_desc(&tm_x);
      LP_TILE_LOOP(i) {
        const int b = i & 1, u = i >> 1, tile = 2 * p + rank;
        if (u > 0) mbar_wait_spin(xfree + 8 * b, (u - 1) & 1);
        mbar_arrive_expect_tx(xfull + 8 * b, KB * kXBlock);
        for (int kb = 0; kb < KB; ++kb)
          tma_load_2d(sX + (b * KB + kb) * kXBlock, &tm_x, xfull + 8 * b, kb * 64, tile * 128);
      }
    }
  } else if (warp == 0) {
    // ------------------------------------------------------------ W producer (half stages)
    if (lane == 0) {
      tma_prefetch_desc(&tm_w);
      const uint32_t half = (uint32_t)a.NT * 64u;  // bytes of this CTA's half of a stage
      int it = 0;
      LP_TILE_LOOP(i) {
        for (int nt = 0; nt < n_tiles; ++nt)
          for (int kb = 0; kb < KB; ++kb, ++it) {
            const int s = it % kSt, round = it / kSt;
            if (round > 0) mbar_wait_spin(wfree + 8 * s, (round - 1) & 1);
            mbar_arrive_expect_tx(wfull + 8 * s, 2 * half);
            tma_load_2d_mc(sW + s * kWStage + rank * half, &tm_w, wfull + 8 * s, kb * 64,
                           nt * a.NT + rank * (a.NT / 2), 0x3);
          }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = make_idesc_bf16(128, (uint32_t)a.NT, 0, 0);
      int it = 0, g = 0;
      LP_TILE_LOOP(i) {
        const int b = i & 1;
        mbar_wait_spin(yready + 8 * b, (i >> 1) & 1);
        if (i < 4) LP_STAMP(9 + i);
        tc_fence_after();
        for (int nt = 0; nt < n_tiles; ++nt, ++g) {
          const int ab = g & 1;
          if (g >= 2) mbar_wait_spin(accfree + 8 * ab, ((g >> 1) - 1) & 1);
          tc_fence_after();
          const uint32_t tacc = tmem + ab * 256;
          for (int kb = 0; kb < KB; ++kb, ++it) {
            const int s = it % kSt;
            mbar_wait_spin(wfull + 8 * s, (it / kSt) & 1);
            tc_fence_after();
            const uint32_t wb = sW + s * kWStage, xb = sX + (b * KB + kb) * kXBlock;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              umma_bf16(tacc, make_sdesc(xb + kk * 32, 16, 1024, kSw128),
                        make_sdesc(wb + kk * 32, 16, 1024, kSw128), idesc, (kb | kk) != 0);
            umma_commit_mc(wfree + 8 * s, 0x3);  // stage s free in both CTAs' view
          }
          umma_commit(accfull + 8 * ab);
        }
        umma_commit(xfree + 8 * b);  // all MMAs reading this x buffer done
        if (i < 4) LP_STAMP(13 + i);
      }
    }
  } else if (warp >= 8) {
    // ------------------------------------------------------------ LayerNorm, in place
    // 8 warps x 16 rows; per pass a warp covers 8 rows with 4 lanes per row: lane (r8, q) =
    // (lane & 7, lane >> 3) reads 16-byte chunks q and q+4 of every 64-channel block of row r8.
    // Each quarter-warp (8 consecutive lanes: one q, rows 0..7) then hits the 8 distinct SW128
    // chunk positions q ^ r8 — conflict-free; row sums by xor-shuffles over lanes 8 and 16.
    const uint32_t r8 = lane & 7, q = lane >> 3, sw = r8 << 4;
    LP_TILE_LOOP(i) {
      const int b = i & 1, tile = 2 * p + rank;
      mbar_wait(xfull + 8 * b, (i >> 1) & 1);
      if (warp == 8 && lane == 0 && i < 4) LP_STAMP(1 + i);
      if (!a.ln) {  // plain linear: the x tile is the A operand as loaded
        mbar_arrive(yready + 8 * b);
        continue;
      }
#pragma unroll 1
      for (int rg = 0; rg < 2; ++rg) {
        const uint32_t t = (warp - 8) * 16 + rg * 8 + r8;  // tile row
        const uint32_t xr = sX + b * KB * kXBlock + t * 128;
        uint4 v[2 * KB];  // the lane's 2·KB chunks of the row, read once
#pragma unroll
        for (int kb = 0; kb < KB; ++kb)
#pragma unroll
          for (int j = 0; j < 2; ++j)
            v[2 * kb + j] = ld_shared_v4(xr + kb * kXBlock + (((q + 4 * j) << 4) ^ sw));
        float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int m = 0; m < 2 * KB; ++m) {
          s4[0] += bf16_lo(v[m].x) + bf16_hi(v[m].x);
          s4[1] += bf16_lo(v[m].y) + bf16_hi(v[m].y);
          s4[2] += bf16_lo(v[m].z) + bf16_hi(v[m].z);
          s4[3] += bf16_lo(v[m].w) + bf16_hi(v[m].w);
        }
        float sum = (s4[0] + s4[1]) + (s4[2] + s4[3]);
        sum += __shfl_xor_sync(0xffffffffu, sum, 8);
        sum += __shfl_xor_sync(0xffffffffu, sum, 16);
        const float mu = sum * (1.f / C);
        float v4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int m = 0; m < 2 * KB; ++m) {
          const uint32_t w[4] = {v[m].x, v[m].y, v[m].z, v[m].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float d0 = bf16_lo(w[e]) - mu, d1 = bf16_hi(w[e]) - mu;
            v4[e] = fmaf(d0, d0, fmaf(d1, d1, v4[e]));
          }
        }
        float ss = (v4[0] + v4[1]) + (v4[2] + v4[3]);
        ss += __shfl_xor_sync(0xffffffffu, ss, 8);
        ss += __shfl_xor_sync(0xffffffffu, ss, 16);
        const float rs = rsqrtf(ss * (1.f / C) + a.eps);
        const int64_t row = (int64_t)tile * 128 + t;
        if (!LP_TL && q == 0 && row < a.M) {
          if (a.mean) a.mean[row] = mu;
          if (a.rstd) a.rstd[row] = rs;
        }
#pragma unroll
        for (int kb = 0; kb < KB; ++kb)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const uint32_t addr = xr + kb * kXBlock + (((q + 4 * j) << 4) ^ sw);
            const uint4 vv = v[2 * kb + j];
            const uint32_t w[4] = {vv.x, vv.y, vv.z, vv.w};
            const int c0 = kb * 64 + (q + 4 * j) * 8;
            const float4 g0 = ld_shared_f4(sGB + 4 * c0), g1 = ld_shared_f4(sGB + 4 * c0 + 16);
            const float4 b0 = ld_shared_f4(sGB + 4 * (C + c0)),
                         b1 = ld_shared_f4(sGB + 4 * (C + c0) + 16);
            const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
            const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
            uint32_t o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              o[e] = pack_bf16((bf16_lo(w[e]) - mu) * rs * gg[2 * e] + bb[2 * e],
                               (bf16_hi(w[e]) - mu) * rs * gg[2 * e + 1] + bb[2 * e + 1]);
            st_shared_v4(addr, o[0], o[1], o[2], o[3]);
          }
      }
      fence_proxy_async_smem();
      if (warp == 8 && lane == 0 && i < 4) LP_STAMP(5 + i);
      mbar_arrive(yready + 8 * b);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const uint32_t t = threadIdx.x - 128;  // tile row == TMEM lane
    const uint32_t lane_base = (uint32_t)(warp & 3) * 32u << 16;
    const uint32_t sw = ((t & 7) >> 1) << 4;  // SW64: 16-byte chunk c of row t at c ^ ((t & 7) >> 1)
    const int chunks = a.NT / 32;             // 32-column output chunks per accumulator
    int g = 0, oc = 0;
    LP_TILE_LOOP(i) {
      const int tile = 2 * p + rank;
      for (int nt = 0; nt < n_tiles; ++nt, ++g) {
        const int ab = g & 1;
        mbar_wait(accfull + 8 * ab, (g >> 1) & 1);
        if (t == 0 && nt == 0 && i < 4) LP_STAMP(33 + i);
        tc_fence_after();
        for (int ch = 0; ch < chunks; ++ch, ++oc) {
          const int n0 = nt * a.NT + ch * 32;
          uint32_t r[32];
          tmem_ld32(tmem + lane_base + ab * 256 + ch * 32, r);
          tmem_wait_ld();
          if (ch == chunks - 1) {
            tc_fence_before();
            mbar_arrive(accfree + 8 * ab);
          }
          // per-warp staging [32 rows][32 cols] (SW64), double-buffered, one TMA store per warp
          const uint32_t sbuf = sO + (warp & 3) * 4096 + (oc & 1) * 2048;
          if (lane == 0) bulk_wait_group_read1();  // this warp's store of chunk oc-2 was read
          __syncwarp();
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float4 b0 = ld_shared_f4(sB + 4 * (n0 + 8 * k));
            const float4 b1 = ld_shared_f4(sB + 4 * (n0 + 8 * k) + 16);
            const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
            float f[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(r[8 * k + e]) + bb[e];
            st_shared_v4(sbuf + lane * 64 + ((k << 4) ^ sw), pack_bf16(f[0], f[1]),
                         pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tm_o, sbuf, n0, tile * 128 + (int)(warp & 3) * 32);
            bulk_commit_group();
          }
        }
      }
    }
    if (lane == 0) bulk_wait_group0();
    if (t == 0) LP_STAMP(41);
  }
#undef LP_TILE_LOOP
  tc_fence_before();
  cluster_sync_all();  // no CTA exits while its peer may still multicast into it
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

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

// bf16 [rows][cols], row stride ld; box [box_rows][box_cols], 128-byte (64 cols) or 64-byte
// (32 cols) swizzle matching the box row
bool make_2d_map(CUtensorMap* m, const void* ptr, int64_t cols, int64_t rows, int64_t ld,
                 int box_rows, int box_cols = 64) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)(rows > 0 ? rows : 1)};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             box_cols == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
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

static evo_status_t ln_proj_launch(const evo_ln_proj_desc_t* d, const void* x, const float* gamma,
                                   const float* beta, const void* W, const float* b, void* out,
                                   float* mean, float* rstd, void* stream, int ln) {
  using namespace evo;
  if (!d) return lp_fail(EVO_E_INVALID, "desc is NULL");
  if (d->rows < 0) return lp_fail(EVO_E_SHAPE, "rows = %lld < 0", (long long)d->rows);
  if (d->C != 64 && d->C != 128 && d->C != 256)
    return lp_fail(EVO_E_UNSUPPORTED, "C = %d (supported: 64, 128, 256)", d->C);
  if (d->N <= 0 || d->N % 64 != 0 || d->N > kMaxN)
    return lp_fail(EVO_E_UNSUPPORTED, "N = %d must be a positive multiple of 64, <= %d", d->N,
                   kMaxN);
  if (ln && !(d->eps > 0.f)) return lp_fail(EVO_E_INVALID, "eps must be > 0");
  if (d->x_ld < d->C || d->x_ld % 8 != 0)
    return lp_fail(EVO_E_ALIGN, "x_ld = %lld must be >= C and a multiple of 8", (long long)d->x_ld);
  if (d->out_ld < d->N || d->out_ld % 8 != 0)
    return lp_fail(EVO_E_ALIGN, "out_ld = %lld must be >= N and a multiple of 8",
                   (long long)d->out_ld);
  if (d->rows == 0) return EVO_OK;
  if (!x || !W || !out || (ln && (!gamma || !beta)))
    return lp_fail(EVO_E_INVALID, ln ? "x, gamma, beta, W and out are required"
                                     : "x, W and out are required");
  if (!al16(x) || !al16(W) || !al16(out) || (b && !al16(b)))
    return lp_fail(EVO_E_ALIGN, "tensors must be 16-byte aligned");

  LnProjArgs a{};
  a.M = d->rows;
  a.N = d->N;
  a.NT = d->N % 256 == 0 ? 256 : (d->N % 128 == 0 ? 128 : 64);
  a.n_row_tiles = (int)((d->rows + 127) / 128);
  a.ln = ln;
  a.eps = d->eps;
  a.gamma = gamma;
  a.beta = beta;
  a.b = b;
  a.mean = ln ? mean : nullptr;
  a.rstd = ln ? rstd : nullptr;
  CUtensorMap tx, tw, to;
  if (!make_2d_map(&tx, x, d->C, d->rows, d->x_ld, 128) ||
      !make_2d_map(&tw, W, d->C, d->N, d->C, a.NT / 2) ||
      !make_2d_map(&to, out, d->N, d->rows, d->out_ld, 32, 32))
    return lp_fail(EVO_E_CUDA, "cuTensorMapEncodeTiled failed");
  a.n_pairs = (a.n_row_tiles + 1) / 2;
  static int n_sm = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const int n_clusters = (int)std::min<int64_t>(a.n_pairs, n_sm / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * n_clusters));
  cfg.blockDim = dim3(kThreads);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaSuccess;
  switch (d->C) {
#define EVO_LP_CASE(CC)                                                                      \
  case CC:                                                                                   \
    cfg.dynamicSmemBytes = lp_smem<CC>();                                                    \
    e = evo::set_smem_once(ln_proj_fwd_kernel<CC>, lp_smem<CC>());                         \
    if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, ln_proj_fwd_kernel<CC>, tx, tw, to, a); \
    break;
    EVO_LP_CASE(64)
    EVO_LP_CASE(128)
    EVO_LP_CASE(256)
#undef EVO_LP_CASE
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? EVO_OK : lp_fail(EVO_E_CUDA, "ln_proj_fwd: %s", cudaGetErrorString(e));
}

extern "C" evo_status_t evo_ln_proj_fwd(const evo_ln_proj_desc_t* d, const void* x,
                                        const float* gamma, const float* beta, const void* W,
                                        const float* b, void* out, float* mean, float* rstd,
                                        void* stream) {
  return ln_proj_launch(d, x, gamma, beta, W, b, out, mean, rstd, stream, 1);
}

extern "C" evo_status_t evo_linear_fwd(const evo_ln_proj_desc_t* d, const void* x, const void* W,
                                       const float* b, void* out, void* stream) {
  return ln_proj_launch(d, x, nullptr, nullptr, W, b, out, nullptr, nullptr, stream, 0);
}

// ===================================================================================== backward
// SURVEY.md §8(f) f2 backward (the gradient of evo_ln_proj_fwd / evo_linear_fwd):
//   dy  = dout · W                      [rows, C]   tcgen05 (dgrad kernel; LN backward fused in
//                                                   its epilogue, thread = row)
//   dx  = rstd·(dy⊙γ − mean_c(dy⊙γ) − x̂·mean_c(dy⊙γ⊙x̂))      (LayerNorm backward; = dy if no LN)
//   dγ  = Σ_rows dy⊙x̂,  dβ = Σ_rows dy  (per-128-row-tile partials, then a fixed-order sum)
//   dW  = doutᵀ · y                     [N, C]      tcgen05 (wgrad kernel, split over rows;
//                                                   y = bf16(x̂·γ + β), the forward's MMA operand,
//                                                   rebuilt once per row by the dgrad epilogue
//                                                   into the workspace — rebuilding it inside the
//                                                   wgrad cost one transform per n-tile, 8x at N=1024)
//   db  = Σ_rows dout                   (per-chunk partials, fixed-order sum)
// Every reduction is in a fixed order (bitwise repeatable).
namespace evo {
namespace {

constexpr uint32_t kBox64 = 64 * 128;  // [64 rows][64 cols] bf16, SW128 (8 KB)

struct LpBwdArgs {
  int64_t M;
  int N, ln, n_tiles_n, nsplit;
  int64_t rows_per_split;
  const float *gamma, *beta, *mean, *rstd;
  __nv_bfloat16* dx;
  int64_t dx_ld;
  float* part_gb;  // [n_row_tiles][2][C]
  float* part_w;   // [nsplit][N][C]
  __nv_bfloat16* y;  // LN: y = bf16(x̂·γ + β) [rows][C] written by dgrad, the wgrad's B operand
};

template <int C>
__host__ __device__ constexpr int dg_stages() { return C == 256 ? 2 : (C == 128 ? 3 : 4); }
template <int C>
constexpr uint32_t dg_stage_bytes() { return kXBlock + (C / 64) * kBox64; }  // dout + W boxes
template <int C>
constexpr size_t dg_smem() {
  return 1024 + (C / 64) * kXBlock + dg_stages<C>() * dg_stage_bytes<C>() + 8 * C + 256;
}
template <int C>
constexpr uint32_t wg_stage_bytes() { return 2 * kBox64 + (C / 64) * kBox64; }  // dout + x boxes
template <int C>
__host__ __device__ constexpr int wg_stages() { return C == 256 ? 4 : 6; }
template <int C>
constexpr size_t wg_smem() { return 1024 + wg_stages<C>() * wg_stage_bytes<C>() + 8 * C + 256; }

// dy = dout·W for one 128-row tile, then the LayerNorm backward of each row (thread = row).
template <int C>
__global__ void __launch_bounds__(256, 1)
    ln_proj_dgrad_kernel(const __grid_constant__ CUtensorMap tm_dout,
                         const __grid_constant__ CUtensorMap tm_w,
                         const __grid_constant__ CUtensorMap tm_x, const LpBwdArgs a) {
  constexpr int CB = C / 64, S = dg_stages<C>();
  constexpr uint32_t kSt = dg_stage_bytes<C>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sX = base;                 // x tile: CB x [128 rows][64 c]
  const uint32_t sR = sX + CB * kXBlock;    // ring: S x (dout [128 rows][64 n] | W CB x [64 n][64 c])
  const uint32_t sG = sR + S * kSt;         // γ [C], β [C] fp32
  const uint32_t sBar = sG + 8 * C;
  const uint32_t full = sBar, empty = sBar + 8 * S, xfull = sBar + 16 * S, accfull = xfull + 8;
  const uint32_t tmem_slot = accfull + 8;
  const uint32_t warp = warp_id(), lane = lane_id();
  const int tile = blockIdx.x, KB = a.N / 64;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, 1);
    }
    mbar_init(xfull, 1);
    mbar_init(accfull, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<C>(tmem_slot);
  if (a.ln) {
    float* g = reinterpret_cast<float*>(smem_raw + (sG - smem_u32(smem_raw)));
    for (int c = threadIdx.x; c < 2 * C; c += 256) g[c] = c < C ? a.gamma[c] : a.beta[c - C];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem_raw + (tmem_slot - smem_u32(smem_raw)));
  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      tma_prefetch_desc(&tm_dout);
      tma_prefetch_desc(&tm_w);
      if (a.ln) {
        tma_prefetch_desc(&tm_x);
        mbar_arrive_expect_tx(xfull, CB * kXBlock);
        for (int cb = 0; cb < CB; ++cb) tma_load_2d(sX + cb * kXBlock, &tm_x, xfull, cb * 64, tile * 128);
      }
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % S, round = kb / S;
        if (round > 0) mbar_wait_spin(empty + 8 * s, (round - 1) & 1);
        const uint32_t sb = sR + s * kSt;
        mbar_arrive_expect_tx(full + 8 * s, kSt);
        tma_load_2d(sb, &tm_dout, full + 8 * s, kb * 64, tile * 128);
        for (int cb = 0; cb < CB; ++cb)
          tma_load_2d(sb + kXBlock + cb * kBox64, &tm_w, full + 8 * s, cb * 64, kb * 64);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer: A = dout (K-major), B = W (MN-major: c contiguous)
      constexpr uint32_t idesc = make_idesc_bf16(128, C, 0, 1);
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % S;
        mbar_wait_spin(full + 8 * s, (kb / S) & 1);
        tc_fence_after();
        const uint32_t sb = sR + s * kSt;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(tmem, make_sdesc(sb + kk * 32, 16, 1024, kSw128),
                    make_sdesc(sb + kXBlock + kk * 2048, kBox64, 1024, kSw128), idesc,
                    (kb | kk) != 0);
        umma_commit(empty + 8 * s);
      }
      umma_commit(accfull);
    }
  } else if (warp >= 4) {
    // ---- epilogue: thread = row of the tile = TMEM lane
    const uint32_t t = threadIdx.x - 128;
    const uint32_t lane_base = (uint32_t)(warp & 3) * 32u << 16;
    const int64_t grow = (int64_t)tile * 128 + t;
    const bool valid = grow < a.M;
    mbar_wait(accfull, 0);
    if (a.ln) mbar_wait(xfull, 0);
    tc_fence_after();
    float mu = 0.f, rs = 0.f;
    if (a.ln && valid) { mu = a.mean[grow]; rs = a.rstd[grow]; }
    const float* g = reinterpret_cast<const float*>(smem_raw + (sG - smem_u32(smem_raw)));
    // x̂ of this row for 8 channels c0..c0+7 (the swizzled x tile)
    auto xhat8 = [&](int c0, float (&xh)[8]) {
      const uint32_t addr = sX + (c0 >> 6) * kXBlock + t * 128 + (((((c0 & 63) >> 3) ^ (t & 7))) << 4);
      const uint4 v = ld_shared_v4(addr);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        xh[2 * e] = (bf16_lo(w[e]) - mu) * rs;
        xh[2 * e + 1] = (bf16_hi(w[e]) - mu) * rs;
      }
    };
    float s1 = 0.f, s2 = 0.f;
    if (a.ln) {
      // pass 1: row sums of dy⊙γ and dy⊙γ⊙x̂, and the tile's column sums of dy⊙x̂ and dy
      // (dγ, dβ partials) through a padded [128][33] staging pair in the drained ring
      float* stg = reinterpret_cast<float*>(smem_raw + (sR - smem_u32(smem_raw)));
      for (int ch = 0; ch < C / 32; ++ch) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_base + ch * 32, r);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float xh[8];
          xhat8(ch * 32 + q * 8, xh);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int j = q * 8 + e;
            const float dy = __uint_as_float(r[j]);
            const float gg = dy * g[ch * 32 + j];
            s1 += gg;
            s2 += gg * xh[e];
            stg[t * 33 + j] = dy * xh[e];
            stg[128 * 33 + t * 33 + j] = dy;
          }
        }
        named_bar_sync(1, 128);
        if (t < 64) {  // column sums in row order (deterministic)
          const int j = t & 31, which = t >> 5;
          const float* col = stg + which * 128 * 33 + j;
          float acc = 0.f;
          for (int rr = 0; rr < 128; ++rr) acc += col[rr * 33];
          a.part_gb[((int64_t)tile * 2 + which) * C + ch * 32 + j] = acc;
        }
        named_bar_sync(1, 128);
      }
    }
    // pass 2: dx (bf16), 8 channels per 16-byte store
    const float inv_c = 1.f / C;
    for (int ch = 0; ch < C / 32; ++ch) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_base + ch * 32, r);
      tmem_wait_ld();
      if (!valid) continue;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float d[8];
        if (a.ln) {
          float xh[8], yv[8];
          xhat8(ch * 32 + q * 8, xh);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int j = q * 8 + e;
            const float gg = __uint_as_float(r[j]) * g[ch * 32 + j];
            d[e] = rs * (gg - s1 * inv_c - xh[e] * (s2 * inv_c));
            yv[e] = xh[e] * g[ch * 32 + j] + g[C + ch * 32 + j];
          }
          uint4 yo;  // the forward's MMA operand, rebuilt once per row for the wgrad
          yo.x = pack_bf16(yv[0], yv[1]); yo.y = pack_bf16(yv[2], yv[3]);
          yo.z = pack_bf16(yv[4], yv[5]); yo.w = pack_bf16(yv[6], yv[7]);
          *reinterpret_cast<uint4*>(a.y + grow * C + ch * 32 + q * 8) = yo;
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) d[e] = __uint_as_float(r[q * 8 + e]);
        }
        uint4 o;
        o.x = pack_bf16(d[0], d[1]); o.y = pack_bf16(d[2], d[3]);
        o.z = pack_bf16(d[4], d[5]); o.w = pack_bf16(d[6], d[7]);
        *reinterpret_cast<uint4*>(a.dx + grow * a.dx_ld + ch * 32 + q * 8) = o;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<C>(tmem);
}

// dW partial of one 128-row tile of W (n) over one range of rows: doutᵀ · y (y from the dgrad's
// workspace buffer; x itself for the plain linear backward).
template <int C>
__global__ void __launch_bounds__(256, 1)
    ln_proj_wgrad_kernel(const __grid_constant__ CUtensorMap tm_dout,
                         const __grid_constant__ CUtensorMap tm_x, const LpBwdArgs a) {
  constexpr int CB = C / 64, S = wg_stages<C>();
  constexpr uint32_t kSt = wg_stage_bytes<C>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sR = base;           // ring: S x (dout 2 x [64 rows][64 n] | x CB x [64 rows][64 c])
  const uint32_t sGB = sR + S * kSt;  // γ [C], β [C]
  const uint32_t sBar = sGB + 8 * C;
  const uint32_t full = sBar, empty = sBar + 8 * S, accfull = sBar + 16 * S;
  const uint32_t tmem_slot = accfull + 8;
  const uint32_t warp = warp_id(), lane = lane_id();
  const int nt = blockIdx.x % a.n_tiles_n, sp = blockIdx.x / a.n_tiles_n;
  const int64_t r0 = (int64_t)sp * a.rows_per_split;
  const int64_t r1 = r0 + a.rows_per_split < a.M ? r0 + a.rows_per_split : a.M;
  const int nkb = r1 > r0 ? (int)((r1 - r0 + 63) / 64) : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, 1);
    }
    mbar_init(accfull, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<C>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem_raw + (tmem_slot - smem_u32(smem_raw)));
  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      tma_prefetch_desc(&tm_dout);
      tma_prefetch_desc(&tm_x);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % S, round = kb / S;
        if (round > 0) mbar_wait_spin(empty + 8 * s, (round - 1) & 1);
        const uint32_t sb = sR + s * kSt;
        const int row = (int)(r0 + kb * 64);
        mbar_arrive_expect_tx(full + 8 * s, kSt);
        tma_load_2d(sb, &tm_dout, full + 8 * s, nt * 128, row);
        tma_load_2d(sb + kBox64, &tm_dout, full + 8 * s, nt * 128 + 64, row);
        for (int cb = 0; cb < CB; ++cb)
          tma_load_2d(sb + 2 * kBox64 + cb * kBox64, &tm_x, full + 8 * s, cb * 64, row);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer: A = doutᵀ (MN-major), B = y (MN-major)
      constexpr uint32_t idesc = make_idesc_bf16(128, C, 1, 1);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % S;
        mbar_wait_spin(full + 8 * s, (kb / S) & 1);
        tc_fence_after();
        const uint32_t sb = sR + s * kSt;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(tmem, make_sdesc(sb + kk * 2048, kBox64, 1024, kSw128),
                    make_sdesc(sb + 2 * kBox64 + kk * 2048, kBox64, 1024, kSw128), idesc,
                    (kb | kk) != 0);
        umma_commit(empty + 8 * s);
      }
      umma_commit(accfull);
    }
  }
  if (warp >= 4 && warp < 8) {
    const uint32_t t = threadIdx.x - 128;
    // ---- epilogue: thread = W row n; the partial [C] row, fp32
    const uint32_t lane_base = (uint32_t)(warp & 3) * 32u << 16;
    if (nkb > 0) mbar_wait(accfull, 0);
    tc_fence_after();
    const int n = nt * 128 + (int)t;
    float* dst = a.part_w + ((int64_t)sp * a.N + n) * C;
    for (int ch = 0; ch < C / 32; ++ch) {
      uint32_t r[32];
      if (nkb > 0) {
        tmem_ld32(tmem + lane_base + ch * 32, r);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = 0u;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
        reinterpret_cast<float4*>(dst + ch * 32)[i] =
            make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                        __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<C>(tmem);
}

// out[i] = Σ_p part[p·stride + i], p = 0, 1, ... (fixed order)
__global__ void __launch_bounds__(256) lp_sum_parts_kernel(const float* __restrict__ part,
                                                           int64_t nparts, int64_t stride,
                                                           int64_t n, float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int64_t p = 0; p < nparts; ++p) s += part[p * stride + i];
    out[i] = s;
  }
}

// out[i] = Σ_p part[p·stride + i] for few outputs and many parts: block i, 256 threads each sum
// parts t, t + 256, ... in order, then a fixed shuffle / shared-memory tree (deterministic)
__global__ void __launch_bounds__(256) lp_colsum_kernel(const float* __restrict__ part,
                                                        int64_t nparts, int64_t stride,
                                                        float* __restrict__ out) {
  __shared__ float red[8];
  const int64_t i = blockIdx.x;
  float s = 0.f;
  for (int64_t p = threadIdx.x; p < nparts; p += 256) s += part[p * stride + i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t += red[w];
    out[i] = t;
  }
}

// db partials: block k sums rows [k·R, (k+1)·R) of dout [rows][N] (row stride ld) into
// part[k][N]; thread = 8 columns, rows of the chunk in order
__global__ void __launch_bounds__(256) lp_db_partial_kernel(const __nv_bfloat16* __restrict__ dout,
                                                            int64_t M, int N, int64_t ld, int R,
                                                            float* __restrict__ part) {
  const int n8 = N / 8;
  const int64_t rbeg = (int64_t)blockIdx.x * R;
  const int64_t rend = rbeg + R < M ? rbeg + R : M;
  for (int c8 = threadIdx.x; c8 < n8; c8 += blockDim.x) {
    float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
    for (int64_t r = rbeg; r < rend; ++r) {
      const uint4 v = *reinterpret_cast<const uint4*>(dout + r * ld + c8 * 8);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        s[2 * e] += bf16_lo(w[e]);
        s[2 * e + 1] += bf16_hi(w[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) part[(int64_t)blockIdx.x * N + c8 * 8 + e] = s[e];
  }
}

struct LpBwdPlan {
  int64_t n_row_tiles, nsplit, rows_per_split, n_db_blocks, db_rows;
  size_t off_gb, off_w, off_db, off_y, bytes;
};
LpBwdPlan lp_bwd_plan(const evo_ln_proj_desc_t* d) {
  LpBwdPlan p{};
  static int n_sm = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  p.n_row_tiles = (d->rows + 127) / 128;
  const int64_t ntn = d->N / 128 > 0 ? d->N / 128 : 1;
  p.nsplit = std::max<int64_t>(1, std::min<int64_t>((n_sm + ntn - 1) / ntn, (d->rows + 63) / 64));
  p.rows_per_split = ((d->rows + p.nsplit - 1) / p.nsplit + 63) / 64 * 64;
  p.nsplit = std::max<int64_t>(1, (d->rows + p.rows_per_split - 1) / p.rows_per_split);
  p.db_rows = 32;
  p.n_db_blocks = std::max<int64_t>(1, (d->rows + p.db_rows - 1) / p.db_rows);
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t off = 0;
  p.off_gb = off; off = al(off + (size_t)p.n_row_tiles * 2 * d->C * 4);
  p.off_w = off;  off = al(off + (size_t)p.nsplit * d->N * d->C * 4);
  p.off_db = off; off = al(off + (size_t)p.n_db_blocks * d->N * 4);
  p.off_y = off;  off = al(off + (size_t)d->rows * d->C * 2);
  p.bytes = off;
  return p;
}

}  // namespace
}  // namespace evo

static evo_status_t ln_proj_bwd_launch(const evo_ln_proj_desc_t* d, const void* x,
                                       const float* gamma, const float* beta, const void* W,
                                       const float* mean, const float* rstd, const void* dout,
                                       int64_t dout_ld, void* dx, int64_t dx_ld, float* dgamma,
                                       float* dbeta, float* dW, float* db, void* ws,
                                       size_t ws_bytes, void* stream, int ln) {
  using namespace evo;
  if (!d) return lp_fail(EVO_E_INVALID, "desc is NULL");
  if (d->rows < 0) return lp_fail(EVO_E_SHAPE, "rows = %lld < 0", (long long)d->rows);
  if (d->C != 64 && d->C != 128 && d->C != 256)
    return lp_fail(EVO_E_UNSUPPORTED, "C = %d (supported: 64, 128, 256)", d->C);
  if (d->N <= 0 || d->N % 128 != 0 || d->N > kMaxN)
    return lp_fail(EVO_E_UNSUPPORTED, "backward: N = %d must be a positive multiple of 128, <= %d",
                   d->N, kMaxN);
  if (d->x_ld < d->C || d->x_ld % 8 != 0)
    return lp_fail(EVO_E_ALIGN, "x_ld = %lld must be >= C and a multiple of 8", (long long)d->x_ld);
  if (dout_ld < d->N || dout_ld % 8 != 0 || dx_ld < d->C || dx_ld % 8 != 0)
    return lp_fail(EVO_E_ALIGN, "dout_ld / dx_ld must cover N / C and be multiples of 8");
  const LpBwdPlan p = lp_bwd_plan(d);
  if (d->rows == 0) return EVO_OK;
  if (!dout || !W || !dx || !dW || (ln && (!x || !gamma || !beta || !mean || !rstd || !dgamma || !dbeta)) ||
      (!ln && !x))
    return lp_fail(EVO_E_INVALID, "a required pointer is NULL");
  if (!ws || ws_bytes < p.bytes)
    return lp_fail(EVO_E_WORKSPACE, "workspace %zu bytes < %zu", ws_bytes, p.bytes);
  if (!al16(x) || !al16(W) || !al16(dout) || !al16(dx) || !al16(dW) || !al16(ws))
    return lp_fail(EVO_E_ALIGN, "tensors must be 16-byte aligned");
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  LpBwdArgs a{};
  a.M = d->rows; a.N = d->N; a.ln = ln; a.n_tiles_n = d->N / 128; a.nsplit = (int)p.nsplit;
  a.rows_per_split = p.rows_per_split;
  a.gamma = gamma; a.beta = beta; a.mean = mean; a.rstd = rstd;
  a.dx = static_cast<__nv_bfloat16*>(dx); a.dx_ld = dx_ld;
  a.part_gb = reinterpret_cast<float*>(w8 + p.off_gb);
  a.part_w = reinterpret_cast<float*>(w8 + p.off_w);
  a.y = reinterpret_cast<__nv_bfloat16*>(w8 + p.off_y);
  CUtensorMap t_dout_a, t_w, t_x128, t_dout_b, t_x64;
  if (!make_2d_map(&t_dout_a, dout, d->N, d->rows, dout_ld, 128) ||
      !make_2d_map(&t_w, W, d->C, d->N, d->C, 64) ||
      !make_2d_map(&t_x128, x, d->C, d->rows, d->x_ld, 128) ||
      !make_2d_map(&t_dout_b, dout, d->N, d->rows, dout_ld, 64) ||
      !make_2d_map(&t_x64, ln ? (const void*)a.y : x, d->C, d->rows, ln ? d->C : d->x_ld, 64))
    return lp_fail(EVO_E_CUDA, "cuTensorMapEncodeTiled failed");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  switch (d->C) {
#define EVO_LPB_CASE(CC)                                                                        \
  case CC:                                                                                      \
    e = set_smem_once(ln_proj_dgrad_kernel<CC>, dg_smem<CC>());                               \
    if (e == cudaSuccess)                                                                       \
      ln_proj_dgrad_kernel<CC><<<(unsigned)p.n_row_tiles, 256, dg_smem<CC>(), st>>>(t_dout_a, t_w, \
                                                                                   t_x128, a);  \
    if (e == cudaSuccess) e = set_smem_once(ln_proj_wgrad_kernel<CC>, wg_smem<CC>());         \
    if (e == cudaSuccess)                                                                       \
      ln_proj_wgrad_kernel<CC><<<(unsigned)(a.n_tiles_n * p.nsplit), 256, wg_smem<CC>(), st>>>( \
          t_dout_b, t_x64, a);                                                                  \
    break;
    EVO_LPB_CASE(64)
    EVO_LPB_CASE(128)
    EVO_LPB_CASE(256)
#undef EVO_LPB_CASE
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  const int red_blocks = 2 * 148;
  if (e == cudaSuccess) {
    lp_sum_parts_kernel<<<red_blocks, 256, 0, st>>>(a.part_w, p.nsplit, (int64_t)d->N * d->C,
                                                    (int64_t)d->N * d->C, dW);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && ln) {
    lp_colsum_kernel<<<d->C, 256, 0, st>>>(a.part_gb, p.n_row_tiles, 2 * d->C, dgamma);
    lp_colsum_kernel<<<d->C, 256, 0, st>>>(a.part_gb + d->C, p.n_row_tiles, 2 * d->C, dbeta);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && db) {
    float* pdb = reinterpret_cast<float*>(w8 + p.off_db);
    lp_db_partial_kernel<<<(unsigned)p.n_db_blocks, 128, 0, st>>>(
        static_cast<const __nv_bfloat16*>(dout), d->rows, d->N, dout_ld, (int)p.db_rows, pdb);
    lp_colsum_kernel<<<d->N, 256, 0, st>>>(pdb, p.n_db_blocks, d->N, db);
    e = cudaGetLastError();
  }
  return e == cudaSuccess ? EVO_OK : lp_fail(EVO_E_CUDA, "ln_proj_bwd: %s", cudaGetErrorString(e));
}

extern "C" size_t evo_ln_proj_bwd_workspace_bytes(const evo_ln_proj_desc_t* d) {
  if (!d || d->rows <= 0 || d->N <= 0 || d->C <= 0) return 0;
  return evo::lp_bwd_plan(d).bytes;
}

extern "C" evo_status_t evo_ln_proj_bwd(const evo_ln_proj_desc_t* d, const void* x,
                                        const float* gamma, const float* beta, const void* W,
                                        const float* mean, const float* rstd, const void* dout,
                                        void* dx, float* dgamma, float* dbeta, float* dW,
                                        float* db, void* workspace, size_t workspace_bytes,
                                        void* stream) {
  if (!d) return evo::lp_fail(EVO_E_INVALID, "desc is NULL");
  return ln_proj_bwd_launch(d, x, gamma, beta, W, mean, rstd, dout, d->out_ld, dx, d->x_ld, dgamma,
                            dbeta, dW, db, workspace, workspace_bytes, stream, 1);
}

extern "C" evo_status_t evo_linear_bwd(const evo_ln_proj_desc_t* d, const void* x, const void* W,
                                       const void* dout, void* dx, float* dW, float* db,
                                       void* workspace, size_t workspace_bytes, void* stream) {
  if (!d) return evo::lp_fail(EVO_E_INVALID, "desc is NULL");
  return ln_proj_bwd_launch(d, x, nullptr, nullptr, W, nullptr, nullptr, dout, d->out_ld, dx,
                            d->x_ld, nullptr, nullptr, dW, db, workspace, workspace_bytes, stream, 0);
}
