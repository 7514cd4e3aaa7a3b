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
