// evo_pair_bias.cu — pair-bias side path (include/evo_pair_bias.h):
// LayerNorm(z) + LinearNoBias(c_z -> H) into the head-major attention bias, and its backward.
//
// thread blocks process many rows; the statistics in a single pass (Σz and
// Σz² in fp32); the parameter gradients by a two-step reduction (per-block partials, then a
// column reduction) with no atomics.  HBM-bound: z is read once (fwd) / twice (fwd + bwd) and
// dz written once.
//
// Mapping: one warp per pair row at a time (lanes across channels), 64 consecutive rows per warp;
// see the kernels below.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <string>

#include "evo_kernels.cuh"
#include "evo_pair_bias.h"

namespace evo {

struct PbArgs {
  int64_t Li, Lj;
  int C, H;
  float eps;
  int64_t z_si, z_sj, b_sh, b_si, b_sj;
  const __nv_bfloat16* z;
  const float *gamma, *beta, *W;
  __nv_bfloat16* bias;
  float *mean, *rstd;
  // backward
  const float* dbias;
  __nv_bfloat16* dz;
  float* partial;  // [nblocks][C·H + 2C]
  int rows_per_block;
};

// Warp per pair row, lanes across channels (NC = C/32 channels per lane, 8-byte-aligned runs):
// a row is one coalesced 2·C-byte read; the per-lane W slice (NC x H) stays in registers for the
// whole kernel; reductions over the row are warp butterflies (every lane ends with the sum).
// A warp walks ROWS_PER_WARP consecutive rows (consecutive j), so the per-head bias values of
// 32 rows land in 32 lanes and leave as coalesced stores.
constexpr int kFwdRowsPerWarp = 4;   // forward: rows per warp (all loads issued up front)
constexpr int kRowsPerWarp = 16;     // backward: rows per warp (amortises the dW/dγ/dβ partials)

template <int NC>
EVO_DEV void load_nc(const __nv_bfloat16* p, float (&v)[NC]) {
  if constexpr (NC == 1) {
    v[0] = __bfloat162float(*p);
  } else if constexpr (NC == 2) {
    const uint32_t u = *reinterpret_cast<const uint32_t*>(p);
    v[0] = bf16_lo(u); v[1] = bf16_hi(u);
  } else if constexpr (NC == 4) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    v[0] = bf16_lo(u.x); v[1] = bf16_hi(u.x); v[2] = bf16_lo(u.y); v[3] = bf16_hi(u.y);
  } else {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) { v[2 * e] = bf16_lo(w[e]); v[2 * e + 1] = bf16_hi(w[e]); }
  }
}

// Reduce-scatter of H per-lane partials across the warp: log2(H) halving steps (lanes with the
// offset bit set keep the upper half) then full butterflies; H - 1 + (5 - log2 H) shuffles
// instead of 5·H.  Afterwards lane l holds the full sum of head (l >> (5 - log2 H)).
template <int H>
EVO_DEV float warp_reduce_scatter(float (&v)[H], int lane) {
#pragma unroll
  for (int off = 16, n = H; off >= 1; off >>= 1) {
    if (n > 1) {
      const int half = n / 2;
      const bool up = (lane & off) != 0;
#pragma unroll
      for (int t = 0; t < H / 2; ++t) {
        if (t < half) {
          const float send = up ? v[t] : v[t + half];
          const float keep = up ? v[t + half] : v[t];
          v[t] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      n = half;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
    }
  }
  return v[0];
}

EVO_DEV float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// ------------------------------------------------------------------ forward
template <int C, int H>
__global__ void __launch_bounds__(256) pair_bias_fwd_kernel(const PbArgs a) {
  constexpr int NC = C / 32;
  const int lane = threadIdx.x & 31;
  const int64_t nrows = a.Li * a.Lj;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t r0 = warp * kFwdRowsPerWarp;
  if (r0 >= nrows) return;
  float w[NC][H], gm[NC], bt[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int cc = lane * NC + c;
    gm[c] = a.gamma[cc];
    bt[c] = a.beta[cc];
#pragma unroll
    for (int h = 0; h < H; ++h) w[c][h] = a.W[cc * H + h];
  }
  // rows r0.. are consecutive: one division per warp, then (i, j) steps (no 64-bit division per row)
  int64_t ri[kFwdRowsPerWarp], rj[kFwdRowsPerWarp];
  {
    int64_t i = r0 / a.Lj, j = r0 - i * a.Lj;
#pragma unroll
    for (int k = 0; k < kFwdRowsPerWarp; ++k) {
      ri[k] = i; rj[k] = j;
      if (++j == a.Lj) { j = 0; ++i; }
    }
  }
  float v[kFwdRowsPerWarp][NC];  // all rows' loads in flight first
#pragma unroll
  for (int k = 0; k < kFwdRowsPerWarp; ++k) {
    const bool ok = r0 + k < nrows;
    load_nc<NC>(a.z + (ok ? ri[k] : ri[0]) * a.z_si + (ok ? rj[k] : rj[0]) * a.z_sj + lane * NC, v[k]);
  }
#pragma unroll
  for (int k = 0; k < kFwdRowsPerWarp; ++k) {
    const int64_t r = r0 + k;
    float s = 0.f, ss = 0.f;  // one pass: Σz, Σz²
#pragma unroll
    for (int c = 0; c < NC; ++c) { s += v[k][c]; ss = fmaf(v[k][c], v[k][c], ss); }
    s = warp_sum(s);
    ss = warp_sum(ss);
    const float mean = s / C;
    const float rstd = rsqrtf(fmaxf(ss / C - mean * mean, 0.f) + a.eps);
    float dot[H];
#pragma unroll
    for (int h = 0; h < H; ++h) dot[h] = 0.f;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const float y = fmaf((v[k][c] - mean) * rstd, gm[c], bt[c]);
#pragma unroll
      for (int h = 0; h < H; ++h) dot[h] = fmaf(y, w[c][h], dot[h]);
    }
    constexpr int kSh = H == 4 ? 3 : (H == 8 ? 2 : 1);  // lane >> kSh = head of the sum
    const float mine = warp_reduce_scatter<H>(dot, lane);
    if (r < nrows) {
      const int64_t i = ri[k], j = rj[k];
      if ((lane & ((1 << kSh) - 1)) == 0)
        a.bias[(lane >> kSh) * a.b_sh + i * a.b_si + j * a.b_sj] = __float2bfloat16_rn(mine);
      if (lane == 0) { a.mean[r] = mean; a.rstd[r] = rstd; }
    }
  }
}

// Two threads per pair row (lanes 2t, 2t+1 take the two channel halves), one pass over z (the
// forward the bench path uses).  With G[c,h] = γ_c·W[c,h], gsum_h = Σ_c G[c,h] and
// bsum_h = Σ_c β_c·W[c,h] (per block, from W/γ/β in shared memory):
//   bias_h = Σ_c ((z_c − mean)·rstd·γ_c + β_c)·W[c,h] = rstd·(Σ_c z_c·G[c,h] − mean·gsum_h) + bsum_h
// so the row is read once, as the statistics are (the paper's single-pass LN):
// each thread issues all its 16-byte loads first (before the block's parameter set-up, so their
// latency covers it), then accumulates Σz, Σz² and the H dot products, and the lane pair combines
// them with one xor-shuffle each.  Consecutive pairs take consecutive j, so the head-major bias
// (j unit-stride) and mean/rstd leave as coalesced stores.
template <int C, int H>
__global__ void __launch_bounds__(256) pair_bias_fwd_row_kernel(const PbArgs a, const FastDiv fd_Lj) {
  // G[c][h] with the second channel half shifted by 4 floats: the two halves of a lane pair read
  // channels c and c + C/2 at the same time, which would otherwise share banks
  constexpr int kHalfOff = C / 2 * H + 4;
  __shared__ __align__(16) float sG[2 * kHalfOff];
  __shared__ float sBW[C][H];   // β_c·W[c,h]
  __shared__ float sSum[2][H];  // gsum, bsum
  constexpr int NCH = C / 16;   // 16-byte chunks per half row
  const uint32_t nrows = (uint32_t)(a.Li * a.Lj);
  const uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 1;
  const int half = threadIdx.x & 1;
  const bool ok = r < nrows;
  const uint32_t i = fdiv(ok ? r : 0u, fd_Lj), j = (ok ? r : 0u) - i * (uint32_t)a.Lj;
  uint4 u[NCH];
  {
    const uint4* zp = reinterpret_cast<const uint4*>(a.z + (int64_t)i * a.z_si + (int64_t)j * a.z_sj) +
                      half * NCH;
#pragma unroll
    for (int k = 0; k < NCH; ++k) u[k] = ok ? __ldg(zp + k) : make_uint4(0, 0, 0, 0);
  }
  for (int x = threadIdx.x; x < C * H; x += blockDim.x) {
    const int c = x / H;
    const float wv = a.W[x];
    sG[(c >= C / 2) * kHalfOff + (c % (C / 2)) * H + x % H] = a.gamma[c] * wv;
    sBW[c][x % H] = a.beta[c] * wv;
  }
  __syncthreads();
  if (threadIdx.x < 2 * H) {  // gsum_h, bsum_h: column sums of the tables, fixed channel order
    const int h = threadIdx.x % H;
    const bool isb = threadIdx.x >= H;
    auto tab = [&](int c) {
      return isb ? sBW[c][h] : sG[(c >= C / 2) * kHalfOff + (c % (C / 2)) * H + h];
    };
    float t0 = 0.f, t1 = 0.f, t2 = 0.f, t3 = 0.f;
#pragma unroll 8
    for (int c = 0; c < C; c += 4) {
      t0 += tab(c);
      t1 += tab(c + 1);
      t2 += tab(c + 2);
      t3 += tab(c + 3);
    }
    sSum[threadIdx.x >= H][h] = (t0 + t1) + (t2 + t3);
  }
  __syncthreads();
  // Σz, Σz² and the dot products in packed fp32 pairs (FFMA2): dot2[p] holds heads 2p, 2p+1
  uint64_t st2 = 0, dot2[H / 2];
#pragma unroll
  for (int p2 = 0; p2 < H / 2; ++p2) dot2[p2] = 0;
#pragma unroll
  for (int k = 0; k < NCH; ++k) {
    const uint32_t w4[4] = {u[k].x, u[k].y, u[k].z, u[k].w};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float z = (e & 1) ? bf16_hi(w4[e >> 1]) : bf16_lo(w4[e >> 1]);
      const uint64_t zz = f2_pack(z, z);
      st2 = f2_fma(zz, f2_pack(1.f, z), st2);  // (Σz, Σz²)
      const uint4* g = reinterpret_cast<const uint4*>(sG + half * kHalfOff + (k * 8 + e) * H);
#pragma unroll
      for (int q = 0; q < H / 4; ++q) {
        const uint4 gv = g[q];
        dot2[2 * q] = f2_fma(zz, ((uint64_t)gv.y << 32) | gv.x, dot2[2 * q]);
        dot2[2 * q + 1] = f2_fma(zz, ((uint64_t)gv.w << 32) | gv.z, dot2[2 * q + 1]);
      }
    }
  }
  float s, ss, dot[H];
  f2_unpack(st2, s, ss);
#pragma unroll
  for (int p2 = 0; p2 < H / 2; ++p2) f2_unpack(dot2[p2], dot[2 * p2], dot[2 * p2 + 1]);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  ss += __shfl_xor_sync(0xffffffffu, ss, 1);
#pragma unroll
  for (int h = 0; h < H; ++h) dot[h] += __shfl_xor_sync(0xffffffffu, dot[h], 1);
  if (!ok) return;
  const float mean = s * (1.f / C);
  const float rstd = rsqrtf(fmaxf(ss * (1.f / C) - mean * mean, 0.f) + a.eps);
#pragma unroll
  for (int h = 0; h < H; ++h)  // the pair splits the heads' stores
    if ((h & 1) == half)
      a.bias[h * a.b_sh + (int64_t)i * a.b_si + (int64_t)j * a.b_sj] =
          __float2bfloat16_rn(fmaf(rstd, dot[h] - mean * sSum[0][h], sSum[1][h]));
  if (half == 0) {
    a.mean[r] = mean;
    a.rstd[r] = rstd;
  }
}

// ------------------------------------------------------------------ backward
// Same warp-per-row walk; every lane accumulates the parameter gradients of its NC channels over
// the warp's rows in registers (dW NC x H, dγ, dβ), the block's 8 warps are summed in a fixed
// order through shared memory into one partial per block, and pair_bias_reduce_kernel sums the
// block partials column by column (the paper's two-step reduction; no atomics, deterministic).
template <int C, int H>
__global__ void __launch_bounds__(256) pair_bias_bwd_kernel(const PbArgs a) {
  constexpr int NC = C / 32;
  constexpr int NOUT = C * H + 2 * C;
  extern __shared__ float red_raw[];
  float (*red)[NOUT] = reinterpret_cast<float (*)[NOUT]>(red_raw);  // [8 warps][NOUT]
  const int lane = threadIdx.x & 31, wv = threadIdx.x >> 5;
  const int64_t nrows = a.Li * a.Lj;
  const int64_t r0 = ((int64_t)blockIdx.x * 8 + wv) * kRowsPerWarp;
  float w[NC][H], gm[NC], bt[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int cc = lane * NC + c;
    gm[c] = a.gamma[cc];
    bt[c] = a.beta[cc];
#pragma unroll
    for (int h = 0; h < H; ++h) w[c][h] = a.W[cc * H + h];
  }
  float dw[NC][H], dg[NC], dbt[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    dg[c] = 0.f;
    dbt[c] = 0.f;
#pragma unroll
    for (int h = 0; h < H; ++h) dw[c][h] = 0.f;
  }
  for (int rb = 0; rb < kRowsPerWarp; rb += 32) {
    // dbias, mean, rstd of up to 32 rows: one coalesced load per head, then broadcast per row
    float dbl[H], ml = 0.f, rl = 0.f;
    int64_t i0 = (r0 + rb) / a.Lj, j0 = (r0 + rb) - ((r0 + rb) / a.Lj) * a.Lj;  // first row
    {
      const int64_t r = r0 + rb + lane;
      const bool ok = r < nrows && lane < kRowsPerWarp;
      const int64_t i = ok ? r / a.Lj : 0, j = ok ? r % a.Lj : 0;
#pragma unroll
      for (int h = 0; h < H; ++h) dbl[h] = ok ? a.dbias[h * a.b_sh + i * a.b_si + j * a.b_sj] : 0.f;
      if (ok) { ml = a.mean[r]; rl = a.rstd[r]; }
    }
    for (int k = 0; k < 32 && rb + k < kRowsPerWarp; ++k) {
      const int64_t r = r0 + rb + k;
      if (r >= nrows) break;  // warp-uniform
      const int64_t i = i0, j = j0;
      if (++j0 == a.Lj) { j0 = 0; ++i0; }
      float v[NC];
      load_nc<NC>(a.z + i * a.z_si + j * a.z_sj + lane * NC, v);
      const float mean = __shfl_sync(0xffffffffu, ml, k), rstd = __shfl_sync(0xffffffffu, rl, k);
      float db[H];
#pragma unroll
      for (int h = 0; h < H; ++h) db[h] = __shfl_sync(0xffffffffu, dbl[h], k);
      float zh[NC], g[NC], sg = 0.f, sgz = 0.f;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        zh[c] = (v[c] - mean) * rstd;
        const float y = fmaf(zh[c], gm[c], bt[c]);
        float dy = 0.f;
#pragma unroll
        for (int h = 0; h < H; ++h) {
          dy = fmaf(db[h], w[c][h], dy);
          dw[c][h] = fmaf(y, db[h], dw[c][h]);
        }
        dg[c] = fmaf(dy, zh[c], dg[c]);
        dbt[c] += dy;
        g[c] = dy * gm[c];
        sg += g[c];
        sgz = fmaf(g[c], zh[c], sgz);
      }
      sg = warp_sum(sg) / C;
      sgz = warp_sum(sgz) / C;
      float d[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) d[c] = rstd * (g[c] - sg - zh[c] * sgz);
      __nv_bfloat16* dp = a.dz + i * a.z_si + j * a.z_sj + lane * NC;
      if constexpr (NC == 1) {
        *dp = __float2bfloat16_rn(d[0]);
      } else if constexpr (NC == 2) {
        *reinterpret_cast<uint32_t*>(dp) = pack_bf16(d[0], d[1]);
      } else if constexpr (NC == 4) {
        *reinterpret_cast<uint2*>(dp) = make_uint2(pack_bf16(d[0], d[1]), pack_bf16(d[2], d[3]));
      } else {
        *reinterpret_cast<uint4*>(dp) = make_uint4(pack_bf16(d[0], d[1]), pack_bf16(d[2], d[3]),
                                                   pack_bf16(d[4], d[5]), pack_bf16(d[6], d[7]));
      }
    }
  }
  // block partial: warp w's per-channel sums into red[w], then a fixed-order sum over warps
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int cc = lane * NC + c;
#pragma unroll
    for (int h = 0; h < H; ++h) red[wv][cc * H + h] = dw[c][h];
    red[wv][C * H + cc] = dg[c];
    red[wv][C * H + C + cc] = dbt[c];
  }
  __syncthreads();
  float* part = a.partial + (int64_t)blockIdx.x * NOUT;
  for (int o = threadIdx.x; o < NOUT; o += blockDim.x) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][o];
    part[o] = t;
  }
}

// Backward for C <= 128, 128 pair rows per 256-thread block, in two phases:
//  1. two threads per row (channel halves, as the forward): ẑ from z/mean/rstd, dy_c = Σ_h dbias_h·W[c,h]
//     (W from shared memory), g = dy·γ, the row sums Σg and Σg·ẑ (one xor-shuffle), then
//     dz_c = rstd·(g_c − Σg/C − ẑ_c·Σgẑ/C) straight to global memory (16-byte stores); ẑ and the row's
//     dbias go to shared memory;
//  2. one thread per (channel, half of the rows): the block's parameter-gradient partials
//     dW[c,h] = Σ_r y·dbias_h, dγ_c = Σ_r dy·ẑ, dβ_c = Σ_r dy from the staged ẑ/dbias (W row in
//     registers), the two row halves added in a fixed order; pair_bias_reduce_kernel sums the block
//     partials (the paper's two-step reduction; deterministic, no atomics).
// The rows' dbias values (consecutive j) and z loads are coalesced; no per-row warp reductions.
template <int C, int H>
__global__ void __launch_bounds__(256) pair_bias_bwd_row_kernel(const PbArgs a, const FastDiv fd_Lj) {
  constexpr int ROWS = 128, NCH = C / 16, CH = C / 2;  // chunks / channels per thread
  constexpr int kHalfOff = CH * H + 4;                  // bank-shifted halves of the W table
  constexpr int ZS = C + 1;                             // padded ẑ row stride (conflict-free)
  extern __shared__ __align__(16) float sm[];
  float* sW = sm;                        // [2 * kHalfOff]
  float* sZ = sW + 2 * kHalfOff;         // [ROWS][ZS]
  float* sDB = sZ + ROWS * ZS;           // [ROWS][H]
  float* sRed = sDB + ROWS * H;          // [C][H + 2] (phase-2 partials of the second row half)
  const int tid = threadIdx.x;
  const uint32_t nrows = (uint32_t)(a.Li * a.Lj);
  const int lrow = tid >> 1, half = tid & 1;
  const uint32_t r = blockIdx.x * ROWS + lrow;
  const bool ok = r < nrows;
  const uint32_t i = fdiv(ok ? r : 0u, fd_Lj), j = (ok ? r : 0u) - i * (uint32_t)a.Lj;
  // ---- phase 1 loads first (their latency covers the W table set-up)
  uint4 u[NCH];
  float db[H], mean = 0.f, rstd = 0.f;
  {
    const uint4* zp = reinterpret_cast<const uint4*>(a.z + (int64_t)i * a.z_si + (int64_t)j * a.z_sj) +
                      half * NCH;
#pragma unroll
    for (int k = 0; k < NCH; ++k) u[k] = ok ? __ldg(zp + k) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int h = 0; h < H; ++h) db[h] = ok ? __ldg(a.dbias + h * a.b_sh + (int64_t)i * a.b_si + (int64_t)j * a.b_sj) : 0.f;
    if (ok) { mean = __ldg(a.mean + r); rstd = __ldg(a.rstd + r); }
  }
  for (int x = tid; x < C * H; x += blockDim.x) {
    const int c = x / H;
    sW[(c >= CH) * kHalfOff + (c % CH) * H + x % H] = a.W[x];
  }
  __syncthreads();
  const float* wt = sW + half * kHalfOff;
  const float* gm = a.gamma + half * CH;
  float sg = 0.f, sgz = 0.f;
#pragma unroll
  for (int k = 0; k < NCH; ++k) {
    const uint32_t w4[4] = {u[k].x, u[k].y, u[k].z, u[k].w};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int c = k * 8 + e;
      const float zh = (((e & 1) ? bf16_hi(w4[e >> 1]) : bf16_lo(w4[e >> 1])) - mean) * rstd;
      float dy = 0.f;
#pragma unroll
      for (int h = 0; h < H; ++h) dy = fmaf(db[h], wt[c * H + h], dy);
      const float g = dy * __ldg(gm + c);
      sg += g;
      sgz = fmaf(g, zh, sgz);
      sZ[lrow * ZS + half * CH + c] = zh;
    }
  }
  sg += __shfl_xor_sync(0xffffffffu, sg, 1);
  sgz += __shfl_xor_sync(0xffffffffu, sgz, 1);
  sg *= 1.f / C;
  sgz *= 1.f / C;
  if (ok) {
    __nv_bfloat16* dzp = a.dz + (int64_t)i * a.z_si + (int64_t)j * a.z_sj + half * CH;
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      uint32_t pk[4];
#pragma unroll
      for (int e2 = 0; e2 < 4; ++e2) {
        float d2[2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int c = k * 8 + 2 * e2 + t;
          const float zh = sZ[lrow * ZS + half * CH + c];
          float dy = 0.f;
#pragma unroll
          for (int h = 0; h < H; ++h) dy = fmaf(db[h], wt[c * H + h], dy);
          d2[t] = rstd * (dy * __ldg(gm + c) - sg - zh * sgz);
        }
        pk[e2] = pack_bf16(d2[0], d2[1]);
      }
      *reinterpret_cast<uint4*>(dzp + k * 8) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
  }
  if (half == 0) {
#pragma unroll
    for (int h = 0; h < H; ++h) sDB[lrow * H + h] = db[h];  // 0 for rows past the end
  }
  __syncthreads();
  // ---- phase 2: thread (c, row half) accumulates the block's parameter gradients
  const int c = tid % C, rh = tid / C;  // 256 threads: C = 128 -> 2 row halves, C = 64 -> 4, ...
  constexpr int NRH = 256 / C;
  float wc[H], dw[H], dg = 0.f, dbt = 0.f;
#pragma unroll
  for (int h = 0; h < H; ++h) { wc[h] = a.W[c * H + h]; dw[h] = 0.f; }
  const float gc = a.gamma[c], bc = a.beta[c];
  const int nr = (int)min((uint32_t)ROWS, nrows - blockIdx.x * ROWS);
  for (int rr = rh; rr < nr; rr += NRH) {
    const float zh = sZ[rr * ZS + c];
    const float y = fmaf(zh, gc, bc);
    float dy = 0.f;
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const float dbh = sDB[rr * H + h];
      dy = fmaf(dbh, wc[h], dy);
      dw[h] = fmaf(y, dbh, dw[h]);
    }
    dg = fmaf(dy, zh, dg);
    dbt += dy;
  }
  // fixed-order combination of the row groups through shared memory (reusing sZ)
  __syncthreads();
  float* red = sZ;  // [NRH][C][H + 2]
#pragma unroll
  for (int h = 0; h < H; ++h) red[(rh * C + c) * (H + 2) + h] = dw[h];
  red[(rh * C + c) * (H + 2) + H] = dg;
  red[(rh * C + c) * (H + 2) + H + 1] = dbt;
  __syncthreads();
  if (rh == 0) {
    float* part = a.partial + (int64_t)blockIdx.x * (C * H + 2 * C);
#pragma unroll
    for (int h = 0; h < H + 2; ++h) {
      float t = 0.f;
#pragma unroll
      for (int g2 = 0; g2 < NRH; ++g2) t += red[(g2 * C + c) * (H + 2) + h];
      if (h < H) part[c * H + h] = t;
      else if (h == H) part[C * H + c] = t;
      else part[C * H + C + c] = t;
    }
  }
  (void)sRed;
}

// step 2 of the parameter-gradient reduction: column sums over the block partials, fixed order.
// 32 columns x 32 partial groups per 1024-thread block: each thread sums its group's partials
// (8 loads in flight per round), then the 32 group sums of a column are added in order.
__global__ void __launch_bounds__(1024) pair_bias_reduce_kernel(const float* __restrict__ part,
                                                                int nblocks, int nout, int C, int H,
                                                                float* dW, float* dgamma,
                                                                float* dbeta) {
  __shared__ float red[32][33];
  const int col = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int o = blockIdx.x * 32 + col;
  const int per = (nblocks + 31) / 32, b0 = grp * per, b1 = min(nblocks, b0 + per);
  float acc = 0.f;
  if (o < nout) {
    for (int b = b0; b < b1; b += 8) {
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = b + k < b1 ? __ldg(part + (int64_t)(b + k) * nout + o) : 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += v[k];
    }
  }
  red[grp][col] = acc;
  __syncthreads();
  if (grp == 0 && o < nout) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 32; ++k) t += red[k][col];
    if (o < C * H) dW[o] = t;
    else if (o < C * H + C) dgamma[o - C * H] = t;
    else dbeta[o - C * H - C] = t;
  }
}

inline int64_t pb_warps(const PbArgs& a) { return (a.Li * a.Lj + kRowsPerWarp - 1) / kRowsPerWarp; }

template <int C>
static cudaError_t launch_fwd_c(const PbArgs& a, cudaStream_t st) {
  const int64_t rows = a.Li * a.Lj;
  if (rows < ((int64_t)1 << 31)) {  // else the warp-per-row kernel (64-bit row indices)
    const unsigned grid = (unsigned)((rows + 127) / 128);  // 128 rows (two threads each) per block
    const FastDiv fd = make_fastdiv((uint32_t)a.Lj);
    if (a.H == 4) pair_bias_fwd_row_kernel<C, 4><<<grid, 256, 0, st>>>(a, fd);
    else if (a.H == 8) pair_bias_fwd_row_kernel<C, 8><<<grid, 256, 0, st>>>(a, fd);
    else pair_bias_fwd_row_kernel<C, 16><<<grid, 256, 0, st>>>(a, fd);
    return cudaGetLastError();
  }
  const int64_t warps = (a.Li * a.Lj + kFwdRowsPerWarp - 1) / kFwdRowsPerWarp;
  const unsigned grid = (unsigned)((warps + 7) / 8);
  if (a.H == 4) pair_bias_fwd_kernel<C, 4><<<grid, 256, 0, st>>>(a);
  else if (a.H == 8) pair_bias_fwd_kernel<C, 8><<<grid, 256, 0, st>>>(a);
  else pair_bias_fwd_kernel<C, 16><<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

template <int C, int H>
static cudaError_t launch_bwd_ch(const PbArgs& a, cudaStream_t st) {
  if constexpr (C <= 128) {  // else (c_z = 256, or 2^31 rows) the warp-per-row kernel
    if (a.Li * a.Lj < ((int64_t)1 << 31)) {
      // 128 rows per block: the same block count (and partial layout) as the warp kernel
      const unsigned grid = (unsigned)((a.Li * a.Lj + 127) / 128);
      auto k = pair_bias_bwd_row_kernel<C, H>;
      constexpr size_t smem = (2 * (C / 2 * H + 4) + 128 * (C + 1) + 128 * H + C * (H + 2)) * 4;
      cudaError_t e = set_smem_once(k, smem);
      if (e != cudaSuccess) return e;
      k<<<grid, 256, smem, st>>>(a, make_fastdiv((uint32_t)a.Lj));
      return cudaGetLastError();
    }
  }
  const unsigned grid = (unsigned)((pb_warps(a) + 7) / 8);
  auto k = pair_bias_bwd_kernel<C, H>;
  constexpr size_t smem = 8 * (C * H + 2 * C) * 4;
  cudaError_t e = set_smem_once(k, smem);
  if (e != cudaSuccess) return e;
  k<<<grid, 256, smem, st>>>(a);
  return cudaGetLastError();
}

template <int C>
static cudaError_t launch_bwd_c(const PbArgs& a, cudaStream_t st) {
  if (a.H == 4) return launch_bwd_ch<C, 4>(a, st);
  if (a.H == 8) return launch_bwd_ch<C, 8>(a, st);
  return launch_bwd_ch<C, 16>(a, st);
}

}  // namespace evo

// ====================================================================== C ABI
namespace {
evo_status_t pb_fail(evo_status_t s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  evo::set_error_detail(buf);  // evo_last_error_detail() (evo_api.cu)
  return s;
}
bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

evo_status_t check_desc(const evo_pair_bias_desc_t* d) {
  if (!d) return pb_fail(EVO_E_INVALID, "desc is NULL");
  if (d->Li < 0 || d->Lj < 0) return pb_fail(EVO_E_SHAPE, "negative pair extent");
  if (d->C != 32 && d->C != 64 && d->C != 128 && d->C != 256)
    return pb_fail(EVO_E_UNSUPPORTED, "C = %d (supported: 32, 64, 128, 256)", d->C);
  if (d->H != 4 && d->H != 8 && d->H != 16)
    return pb_fail(EVO_E_UNSUPPORTED, "H = %d (supported: 4, 8, 16)", d->H);
  if (!(d->eps > 0.f)) return pb_fail(EVO_E_INVALID, "eps must be > 0");
  if (d->z_str[2] != 1) return pb_fail(EVO_E_ALIGN, "z channel stride must be 1");
  if ((d->z_str[0] * 2) % 16 || (d->z_str[1] * 2) % 16)
    return pb_fail(EVO_E_ALIGN, "z row strides must be multiples of 16 bytes");
  return EVO_OK;
}

evo::PbArgs make_args(const evo_pair_bias_desc_t* d) {
  evo::PbArgs a{};
  a.Li = d->Li; a.Lj = d->Lj; a.C = d->C; a.H = d->H; a.eps = d->eps;
  a.z_si = d->z_str[0]; a.z_sj = d->z_str[1];
  a.b_sh = d->b_str[0]; a.b_si = d->b_str[1]; a.b_sj = d->b_str[2];
  return a;
}

cudaError_t launch_fwd(const evo::PbArgs& a, cudaStream_t st) {
  switch (a.C) {
    case 32: return evo::launch_fwd_c<32>(a, st);
    case 64: return evo::launch_fwd_c<64>(a, st);
    case 128: return evo::launch_fwd_c<128>(a, st);
    default: return evo::launch_fwd_c<256>(a, st);
  }
}
cudaError_t launch_bwd(const evo::PbArgs& a, cudaStream_t st) {
  switch (a.C) {
    case 32: return evo::launch_bwd_c<32>(a, st);
    case 64: return evo::launch_bwd_c<64>(a, st);
    case 128: return evo::launch_bwd_c<128>(a, st);
    default: return evo::launch_bwd_c<256>(a, st);
  }
}
int64_t bwd_blocks(const evo_pair_bias_desc_t* d) {
  const int64_t warps = (d->Li * d->Lj + evo::kRowsPerWarp - 1) / evo::kRowsPerWarp;
  return (warps + 7) / 8;
}
}  // namespace

extern "C" {

evo_status_t evo_pair_bias_fwd(const evo_pair_bias_desc_t* d, const void* z, const float* gamma,
                               const float* beta, const float* W, void* bias, float* mean,
                               float* rstd, void* stream) {
  evo_status_t s = check_desc(d);
  if (s) return s;
  if (!z || !gamma || !beta || !W || !bias || !mean || !rstd)
    return pb_fail(EVO_E_INVALID, "z, gamma, beta, W, bias, mean, rstd are required");
  if (!al16(z)) return pb_fail(EVO_E_ALIGN, "z is not 16-byte aligned");
  if (d->Li * d->Lj == 0) return EVO_OK;
  evo::PbArgs a = make_args(d);
  a.z = (const __nv_bfloat16*)z; a.gamma = gamma; a.beta = beta; a.W = W;
  a.bias = (__nv_bfloat16*)bias; a.mean = mean; a.rstd = rstd;
  cudaError_t e = launch_fwd(a, reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? EVO_OK : pb_fail(EVO_E_CUDA, "pair_bias_fwd: %s", cudaGetErrorString(e));
}

size_t evo_pair_bias_bwd_workspace_bytes(const evo_pair_bias_desc_t* d) {
  if (check_desc(d) != EVO_OK) return 0;
  return (size_t)bwd_blocks(d) * (size_t)(d->C * d->H + 2 * d->C) * 4;
}

evo_status_t evo_pair_bias_bwd(const evo_pair_bias_desc_t* d, const void* z, const float* gamma,
                               const float* beta, const float* W, const float* mean,
                               const float* rstd, const float* dbias, void* dz, float* dgamma,
                               float* dbeta, float* dW, void* workspace, size_t workspace_bytes,
                               void* stream) {
  evo_status_t s = check_desc(d);
  if (s) return s;
  if (!z || !gamma || !beta || !W || !mean || !rstd || !dbias || !dz || !dgamma || !dbeta || !dW)
    return pb_fail(EVO_E_INVALID, "every tensor argument is required");
  if (!al16(z) || !al16(dz)) return pb_fail(EVO_E_ALIGN, "z / dz not 16-byte aligned");
  const size_t need = evo_pair_bias_bwd_workspace_bytes(d);
  if (need && (!workspace || workspace_bytes < need))
    return pb_fail(EVO_E_WORKSPACE, "workspace needs %zu bytes, got %zu", need, workspace_bytes);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int nout = d->C * d->H + 2 * d->C;
  if (d->Li * d->Lj == 0) {  // empty: zero parameter gradients
    cudaMemsetAsync(dW, 0, (size_t)d->C * d->H * 4, st);
    cudaMemsetAsync(dgamma, 0, (size_t)d->C * 4, st);
    cudaMemsetAsync(dbeta, 0, (size_t)d->C * 4, st);
    return EVO_OK;
  }
  evo::PbArgs a = make_args(d);
  a.z = (const __nv_bfloat16*)z; a.gamma = gamma; a.beta = beta; a.W = W;
  a.mean = const_cast<float*>(mean); a.rstd = const_cast<float*>(rstd);
  a.dbias = dbias; a.dz = (__nv_bfloat16*)dz; a.partial = (float*)workspace;
  cudaError_t e = launch_bwd(a, st);
  if (e != cudaSuccess) return pb_fail(EVO_E_CUDA, "pair_bias_bwd: %s", cudaGetErrorString(e));
  const int nb = (int)bwd_blocks(d);
  evo::pair_bias_reduce_kernel<<<(nout + 31) / 32, 1024, 0, st>>>(a.partial, nb, nout, d->C, d->H,
                                                                  dW, dgamma, dbeta);
  e = cudaGetLastError();
  return e == cudaSuccess ? EVO_OK : pb_fail(EVO_E_CUDA, "pair_bias_reduce: %s", cudaGetErrorString(e));
}

}  // extern "C"
