// evo_pair_bias.cu — pair-bias side path (include/evo_pair_bias.h):
// LayerNorm(z) + LinearNoBias(c_z -> H) into the head-major attention bias, and its backward.
//
// thread blocks process many rows; the statistics in a single pass (Σz and
// Σz² in fp32); the parameter gradients by a two-step reduction (per-block partials, then a
// column reduction) with no atomics.  HBM-bound: z is read once (fwd) / twice (fwd + bwd) and
// dz written once.
//
// Mapping: TPR = max(1, C/64) threads per pair row, each holding C/TPR channels (≤ 64) of the
// row in registers; rows of a warp are consecutive along j, so the z loads (16 B per thread)
// and the per-head bias stores (consecutive j) are coalesced.  W, γ, β live in shared memory
// (broadcast reads).
#include <cuda_runtime.h>

#include <cstdarg>
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

template <int CP>  // channels per thread (C / TPR)
EVO_DEV void load_row(const __nv_bfloat16* p, float (&v)[CP]) {
#pragma unroll
  for (int c = 0; c < CP; c += 8) {
    const uint4 u = *reinterpret_cast<const uint4*>(p + c);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[c + 2 * e] = bf16_lo(w[e]);
      v[c + 2 * e + 1] = bf16_hi(w[e]);
    }
  }
}

template <int TPR>
EVO_DEV float group_sum(float x) {  // sum over the TPR consecutive lanes of one row
#pragma unroll
  for (int o = 1; o < TPR; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// ------------------------------------------------------------------ forward
template <int C, int TPR, int H>
__global__ void __launch_bounds__(256) pair_bias_fwd_kernel(const PbArgs a) {
  constexpr int CP = C / TPR;
  __shared__ float sW[C * H], sG[C], sB[C];
  for (int i = threadIdx.x; i < C * H; i += blockDim.x) sW[i] = a.W[i];
  for (int i = threadIdx.x; i < C; i += blockDim.x) { sG[i] = a.gamma[i]; sB[i] = a.beta[i]; }
  __syncthreads();
  const int64_t nrows = a.Li * a.Lj;
  const int sub = threadIdx.x % TPR;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / TPR;
  const bool valid = r < nrows;
  const int64_t i = valid ? r / a.Lj : 0, j = valid ? r % a.Lj : 0;
  float v[CP];
#pragma unroll
  for (int c = 0; c < CP; ++c) v[c] = 0.f;
  if (valid) load_row<CP>(a.z + i * a.z_si + j * a.z_sj + sub * CP, v);
  float s = 0.f, ss = 0.f;  // single pass: Σz, Σz²
#pragma unroll
  for (int c = 0; c < CP; ++c) { s += v[c]; ss = fmaf(v[c], v[c], ss); }
  s = group_sum<TPR>(s);
  ss = group_sum<TPR>(ss);
  const float mean = s / C;
  const float var = fmaxf(ss / C - mean * mean, 0.f);
  const float rstd = rsqrtf(var + a.eps);
  float dot[H];
#pragma unroll
  for (int h = 0; h < H; ++h) dot[h] = 0.f;
#pragma unroll
  for (int c = 0; c < CP; ++c) {
    const int cc = sub * CP + c;
    const float y = fmaf((v[c] - mean) * rstd, sG[cc], sB[cc]);
#pragma unroll
    for (int h = 0; h < H; ++h) dot[h] = fmaf(y, sW[cc * H + h], dot[h]);
  }
#pragma unroll
  for (int h = 0; h < H; ++h) dot[h] = group_sum<TPR>(dot[h]);
  if (valid && sub == 0) {
#pragma unroll
    for (int h = 0; h < H; ++h)
      a.bias[h * a.b_sh + i * a.b_si + j * a.b_sj] = __float2bfloat16_rn(dot[h]);
    a.mean[r] = mean;
    a.rstd[r] = rstd;
  }
}

// ------------------------------------------------------------------ backward
// Block = rows_per_block rows (RB = 8192 / C).  Phase 1 (TPR threads per row): dz, and the
// row's ẑ, y, dy into shared memory; phase 2 (thread per output): the block's partial of dW, dγ,
// dβ as plain sums over its rows, in row order.
template <int C, int TPR, int H>
__global__ void __launch_bounds__(256) pair_bias_bwd_kernel(const PbArgs a) {
  constexpr int CP = C / TPR;
  constexpr int RB = 8192 / C;
  extern __shared__ float sm[];
  float* sY = sm;                 // [RB][C]
  float* sDY = sY + RB * C;       // [RB][C]
  float* sZH = sDY + RB * C;      // [RB][C]
  float* sDB = sZH + RB * C;      // [RB][H]
  float* sW = sDB + RB * H;       // [C][H]
  float* sG = sW + C * H;         // [C]
  float* sB = sG + C;             // [C]
  for (int t = threadIdx.x; t < C * H; t += blockDim.x) sW[t] = a.W[t];
  for (int t = threadIdx.x; t < C; t += blockDim.x) { sG[t] = a.gamma[t]; sB[t] = a.beta[t]; }
  __syncthreads();
  const int64_t nrows = a.Li * a.Lj;
  const int sub = threadIdx.x % TPR;
  const int rl = threadIdx.x / TPR;  // row within the block
  const int64_t r = (int64_t)blockIdx.x * RB + rl;
  const bool valid = r < nrows;
  const int64_t i = valid ? r / a.Lj : 0, j = valid ? r % a.Lj : 0;
  float v[CP];
#pragma unroll
  for (int c = 0; c < CP; ++c) v[c] = 0.f;
  if (valid) load_row<CP>(a.z + i * a.z_si + j * a.z_sj + sub * CP, v);
  const float mean = valid ? a.mean[r] : 0.f, rstd = valid ? a.rstd[r] : 0.f;
  float db[H];
#pragma unroll
  for (int h = 0; h < H; ++h) db[h] = valid ? a.dbias[h * a.b_sh + i * a.b_si + j * a.b_sj] : 0.f;
  if (sub == 0) {
#pragma unroll
    for (int h = 0; h < H; ++h) sDB[rl * H + h] = db[h];
  }
  float g[CP];
  float sg = 0.f, sgz = 0.f;
#pragma unroll
  for (int c = 0; c < CP; ++c) {
    const int cc = sub * CP + c;
    const float zh = (v[c] - mean) * rstd;
    float dy = 0.f;
#pragma unroll
    for (int h = 0; h < H; ++h) dy = fmaf(db[h], sW[cc * H + h], dy);
    sY[rl * C + cc] = fmaf(zh, sG[cc], sB[cc]);
    sDY[rl * C + cc] = dy;
    sZH[rl * C + cc] = zh;
    g[c] = dy * sG[cc];
    sg += g[c];
    sgz = fmaf(g[c], zh, sgz);
    v[c] = zh;
  }
  sg = group_sum<TPR>(sg) / C;
  sgz = group_sum<TPR>(sgz) / C;
  if (valid) {
    __nv_bfloat16* dp = a.dz + i * a.z_si + j * a.z_sj + sub * CP;
#pragma unroll
    for (int c = 0; c < CP; c += 8) {
      float d[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) d[e] = rstd * (g[c + e] - sg - v[c + e] * sgz);
      uint4 u;
      u.x = pack_bf16(d[0], d[1]); u.y = pack_bf16(d[2], d[3]);
      u.z = pack_bf16(d[4], d[5]); u.w = pack_bf16(d[6], d[7]);
      *reinterpret_cast<uint4*>(dp + c) = u;
    }
  }
  __syncthreads();
  const int nout = C * H + 2 * C;
  const int64_t left = nrows - (int64_t)blockIdx.x * RB;
  const int rows_here = left < RB ? (int)left : RB;
  float* part = a.partial + (int64_t)blockIdx.x * nout;
  for (int o = threadIdx.x; o < nout; o += blockDim.x) {
    float acc = 0.f;
    if (o < C * H) {  // dW[c][h] = Σ_rows y_c · dbias_h
      const int c = o / H, h = o % H;
      for (int q = 0; q < rows_here; ++q) acc = fmaf(sY[q * C + c], sDB[q * H + h], acc);
    } else if (o < C * H + C) {  // dγ_c = Σ_rows dy_c · ẑ_c
      const int c = o - C * H;
      for (int q = 0; q < rows_here; ++q) acc = fmaf(sDY[q * C + c], sZH[q * C + c], acc);
    } else {  // dβ_c = Σ_rows dy_c
      const int c = o - C * H - C;
      for (int q = 0; q < rows_here; ++q) acc += sDY[q * C + c];
    }
    part[o] = acc;
  }
}

// step 2 of the parameter-gradient reduction: column sums over the block partials, fixed order
__global__ void __launch_bounds__(256) pair_bias_reduce_kernel(const float* __restrict__ part,
                                                               int nblocks, int nout, int C, int H,
                                                               float* dW, float* dgamma,
                                                               float* dbeta) {
  __shared__ float red[8][33];
  const int o = blockIdx.x * 32 + (threadIdx.x & 31);
  const int wv = threadIdx.x >> 5;
  float acc = 0.f;
  if (o < nout)
    for (int b = wv; b < nblocks; b += 8) acc += part[(int64_t)b * nout + o];
  red[wv][threadIdx.x & 31] = acc;
  __syncthreads();
  if (wv == 0 && o < nout) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][threadIdx.x & 31];
    if (o < C * H) dW[o] = t;
    else if (o < C * H + C) dgamma[o - C * H] = t;
    else dbeta[o - C * H - C] = t;
  }
}

template <int C, int TPR>
static cudaError_t launch_fwd_c(const PbArgs& a, cudaStream_t st) {
  const int64_t threads = a.Li * a.Lj * TPR;
  const unsigned grid = (unsigned)((threads + 255) / 256);
#define EVO_PB_H(hh) \
  if (a.H <= hh) { pair_bias_fwd_kernel<C, TPR, hh><<<grid, 256, 0, st>>>(a); return cudaGetLastError(); }
  EVO_PB_H(4) EVO_PB_H(8) EVO_PB_H(16)
#undef EVO_PB_H
  return cudaErrorInvalidValue;
}

template <int C, int TPR, int H>
static cudaError_t launch_bwd_ch(const PbArgs& a, cudaStream_t st) {
  constexpr int RB = 8192 / C;
  const size_t smem = (size_t)(3 * RB * C + RB * H + C * H + 2 * C) * 4;
  auto k = pair_bias_bwd_kernel<C, TPR, H>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const unsigned grid = (unsigned)((a.Li * a.Lj + RB - 1) / RB);
  k<<<grid, RB * TPR, smem, st>>>(a);
  return cudaGetLastError();
}

template <int C, int TPR>
static cudaError_t launch_bwd_c(const PbArgs& a, cudaStream_t st) {
  if (a.H <= 4) return launch_bwd_ch<C, TPR, 4>(a, st);
  if (a.H <= 8) return launch_bwd_ch<C, TPR, 8>(a, st);
  return launch_bwd_ch<C, TPR, 16>(a, st);
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
    case 32: return evo::launch_fwd_c<32, 1>(a, st);
    case 64: return evo::launch_fwd_c<64, 1>(a, st);
    case 128: return evo::launch_fwd_c<128, 2>(a, st);
    default: return evo::launch_fwd_c<256, 4>(a, st);
  }
}
cudaError_t launch_bwd(const evo::PbArgs& a, cudaStream_t st) {
  switch (a.C) {
    case 32: return evo::launch_bwd_c<32, 1>(a, st);
    case 64: return evo::launch_bwd_c<64, 1>(a, st);
    case 128: return evo::launch_bwd_c<128, 2>(a, st);
    default: return evo::launch_bwd_c<256, 4>(a, st);
  }
}
int64_t bwd_blocks(const evo_pair_bias_desc_t* d) { return (d->Li * d->Lj + 8192 / d->C - 1) / (8192 / d->C); }
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
  evo::pair_bias_reduce_kernel<<<(nout + 31) / 32, 256, 0, st>>>(a.partial, nb, nout, d->C, d->H,
                                                                 dW, dgamma, dbeta);
  e = cudaGetLastError();
  return e == cudaSuccess ? EVO_OK : pb_fail(EVO_E_CUDA, "pair_bias_reduce: %s", cudaGetErrorString(e));
}

}  // extern "C"
