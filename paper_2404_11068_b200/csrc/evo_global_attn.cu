// evo_global_attn.cu — extra-MSA global column attention core (include/evo_global_attn.h;
// SURVEY.md §8(f) f3; AF2 Alg. 19 lines 3, 5, 6 cited at PAPER.md L178).
//
// One CTA per column b (256 threads).  The work per column is a handful of tiny contractions
// (one query per head against S keys of a single shared K/V head), so there is nothing for the
// tensor cores: the kernel is HBM-bound on q, g, o (and dout, dq, dg in the backward), streamed
// in coalesced 16-byte chunks, with the per-head score rows of the column in shared memory.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>

#include "evo_global_attn.h"
#include "evo_kernels.cuh"

namespace evo {

struct GaArgs {
  int64_t B;
  int S, H, D;
  float scale;
  int64_t q_sb, q_ss, q_sh, k_sb, k_ss, v_sb, v_ss, g_sb, g_ss, g_sh, o_sb, o_ss, o_sh;
  const uint8_t* mask;
  int64_t m_sb, m_ss;
  const __nv_bfloat16 *q, *k, *v, *g, *dout;
  __nv_bfloat16 *o, *dq, *dk, *dv, *dg;
  float *lse, *qbar;
  const float *lse_in, *qbar_in;
};

constexpr int kGaThreads = 512;

EVO_DEV float ga_sigmoid(float x) { return 1.f / (1.f + __expf(-x)); }

template <int D>
EVO_DEV void ga_load(const __nv_bfloat16* p, float (&r)[D]) {
#pragma unroll
  for (int c = 0; c < D; c += 8) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p + c));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) { r[c + 2 * e] = bf16_lo(w[e]); r[c + 2 * e + 1] = bf16_hi(w[e]); }
  }
}

EVO_DEV bool ga_keep(const GaArgs& a, int64_t b, int s) {
  return a.mask ? a.mask[b * a.m_sb + (int64_t)s * a.m_ss] != 0 : true;
}

// block-wide sum of one float per thread (all threads get the result)
EVO_DEV float block_sum(float x, float* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = x;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < kGaThreads / 32; ++i) t += red[i];
  return t;
}
EVO_DEV float block_max(float x, float* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = x;
  __syncthreads();
  float t = -INFINITY;
  for (int i = 0; i < kGaThreads / 32; ++i) t = fmaxf(t, red[i]);
  return t;
}

// block-wide reduction of H <= 16 values per thread at once (max or sum; every thread gets the
// H results): one shuffle tree per head and a single pair of barriers instead of one per head
template <bool MAX>
EVO_DEV void block_reduce_heads(float (&v)[16], int H, float* red) {
#pragma unroll
  for (int h = 0; h < 16; ++h) {
    if (h >= H) break;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float u = __shfl_xor_sync(0xffffffffu, v[h], o);
      v[h] = MAX ? fmaxf(v[h], u) : v[h] + u;
    }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0)
#pragma unroll
    for (int h = 0; h < 16; ++h)
      if (h < H) red[w * 16 + h] = v[h];
  __syncthreads();
#pragma unroll
  for (int h = 0; h < 16; ++h) {
    if (h >= H) break;
    float t = MAX ? -INFINITY : 0.f;
    for (int i = 0; i < kGaThreads / 32; ++i) t = MAX ? fmaxf(t, red[i * 16 + h]) : t + red[i * 16 + h];
    v[h] = t;
  }
  __syncthreads();  // red may be reused right after
}

// Σ over the column's kept sequences of x[b,s,h,:] (slot layout: (s, h, 8-chunk)); result
// (H·D floats) in out[], divided by `div`
template <int D>
EVO_DEV void ga_mean_over_s(const GaArgs& a, int64_t b, const __nv_bfloat16* x, int64_t sb,
                            int64_t ss, int64_t sh, float div, float* red, float* out) {
  constexpr int NC = D / 8;
  const int HC = a.H * NC;
  const int ngrp = kGaThreads / HC;  // s-groups (threads beyond ngrp·HC idle)
  const int slot = threadIdx.x % HC, grp = threadIdx.x / HC;
  const int h = slot / NC, c = slot % NC;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (grp < ngrp) {
    for (int s0 = grp; s0 < a.S; s0 += 4 * ngrp) {  // four rows' loads in flight together
      uint4 u[4];
      bool ok[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int s = s0 + j * ngrp;
        ok[j] = s < a.S && ga_keep(a, b, s);
        u[j] = ok[j] ? __ldg(reinterpret_cast<const uint4*>(x + b * sb + (int64_t)s * ss +
                                                            (int64_t)h * sh + c * 8))
                     : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {  // rows summed in s order (fixed per thread)
        const uint32_t w[4] = {u[j].x, u[j].y, u[j].z, u[j].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) { acc[2 * e] += bf16_lo(w[e]); acc[2 * e + 1] += bf16_hi(w[e]); }
      }
    }
  }
  __syncthreads();
  if (grp < ngrp)
#pragma unroll
    for (int e = 0; e < 8; ++e) red[grp * (HC * 8) + slot * 8 + e] = acc[e];
  __syncthreads();
  for (int i = threadIdx.x; i < HC * 8; i += kGaThreads) {
    float t = 0.f;
    for (int gI = 0; gI < ngrp; ++gI) t += red[gI * (HC * 8) + i];
    out[i] = t / div;  // i = h·D + d (slot·8 + e with slot = h·NC + c)
  }
  __syncthreads();
}

template <int D>
EVO_DEV int ga_count(const GaArgs& a, int64_t b, float* red) {
  float c = 0.f;
  for (int s = threadIdx.x; s < a.S; s += kGaThreads) c += ga_keep(a, b, s) ? 1.f : 0.f;
  return (int)block_sum(c, red);
}

// scores of every kept key for every head into sA[h][t] (−inf when masked); returns nothing
template <int D>
EVO_DEV void ga_scores(const GaArgs& a, int64_t b, const float* sQ, float* sA) {
  for (int t = threadIdx.x; t < a.S; t += kGaThreads) {
    const bool keep = ga_keep(a, b, t);
    float kv[D];
    ga_load<D>(a.k + b * a.k_sb + (int64_t)t * a.k_ss, kv);
    for (int h = 0; h < a.H; ++h) {
      float l = 0.f;
#pragma unroll
      for (int d = 0; d < D; ++d) l = fmaf(sQ[h * D + d], kv[d], l);
      sA[h * a.S + t] = keep ? l * a.scale : -INFINITY;
    }
  }
}

// attn[h][d] = Σ_t sA[h][t]·v[t][d] / norm[h]   (threads: (h, t-group))
template <int D>
EVO_DEV void ga_weighted_v(const GaArgs& a, int64_t b, const float* sA, const float* norm,
                           float* red, float* out) {
  const int ntg = kGaThreads / a.H;
  const int h = threadIdx.x % a.H, tg = threadIdx.x / a.H;
  float acc[D];
#pragma unroll
  for (int d = 0; d < D; ++d) acc[d] = 0.f;
  if (tg < ntg) {
    for (int t = tg; t < a.S; t += ntg) {
      const float w = sA[h * a.S + t];
      if (w == 0.f) continue;
      float vv[D];
      ga_load<D>(a.v + b * a.v_sb + (int64_t)t * a.v_ss, vv);
#pragma unroll
      for (int d = 0; d < D; ++d) acc[d] = fmaf(w, vv[d], acc[d]);
    }
  }
  __syncthreads();
  if (tg < ntg)
#pragma unroll
    for (int d = 0; d < D; ++d) red[tg * (a.H * D) + h * D + d] = acc[d];
  __syncthreads();
  for (int i = threadIdx.x; i < a.H * D; i += kGaThreads) {
    float t = 0.f;
    for (int gI = 0; gI < ntg; ++gI) t += red[gI * (a.H * D) + i];
    out[i] = t * norm[i / D];
  }
  __syncthreads();
}

// ------------------------------------------------------------------ forward
template <int D>
__global__ void __launch_bounds__(kGaThreads) global_attn_fwd_kernel(const GaArgs a) {
  extern __shared__ float sm[];
  float* sA = sm;                              // [H][S]
  float* sQ = sA + a.H * a.S;                  // [H·D]  q̄
  float* sAt = sQ + a.H * D;                   // [H·D]  attn
  float* sN = sAt + a.H * D;                   // [H]    1/Σ
  float* red = sN + 16;                        // reductions
  const int64_t b = blockIdx.x;
  const int cnt = ga_count<D>(a, b, red);
  ga_mean_over_s<D>(a, b, a.q, a.q_sb, a.q_ss, a.q_sh, cnt > 0 ? (float)cnt : 1.f, red, sQ);
  if (cnt > 0) {
    ga_scores<D>(a, b, sQ, sA);
    __syncthreads();
    {  // softmax statistics of all heads at once (H <= 16)
      float m[16], sum[16];
#pragma unroll
      for (int h = 0; h < 16; ++h) { m[h] = -INFINITY; sum[h] = 0.f; }
      for (int t = threadIdx.x; t < a.S; t += kGaThreads)
#pragma unroll
        for (int h = 0; h < 16; ++h)
          if (h < a.H) m[h] = fmaxf(m[h], sA[h * a.S + t]);
      block_reduce_heads<true>(m, a.H, red);
      for (int t = threadIdx.x; t < a.S; t += kGaThreads)
#pragma unroll
        for (int h = 0; h < 16; ++h) {
          if (h >= a.H) break;
          const float x = sA[h * a.S + t];
          const float e = x == -INFINITY ? 0.f : __expf(x - m[h]);
          sA[h * a.S + t] = e;
          sum[h] += e;
        }
      block_reduce_heads<false>(sum, a.H, red);
      if (threadIdx.x == 0)
#pragma unroll
        for (int h = 0; h < 16; ++h)
          if (h < a.H) {
            sN[h] = 1.f / sum[h];
            a.lse[b * a.H + h] = m[h] + __logf(sum[h]);
          }
    }
    __syncthreads();
    ga_weighted_v<D>(a, b, sA, sN, red, sAt);
  } else {
    for (int i = threadIdx.x; i < a.H * D; i += kGaThreads) sAt[i] = 0.f;
    for (int h = threadIdx.x; h < a.H; h += kGaThreads) a.lse[b * a.H + h] = -INFINITY;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < a.H * D; i += kGaThreads) a.qbar[b * a.H * D + i] = sQ[i];
  // o[b,s,h,:] = σ(g) ⊙ attn[h]
  constexpr int NC = D / 8;
  const int HC = a.H * NC;
  const int64_t nout = (int64_t)a.S * HC;
  for (int64_t i0 = threadIdx.x; i0 < nout; i0 += 4 * kGaThreads) {  // 4 chunks in flight
    uint4 gu[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t idx = i0 + j * kGaThreads;
      const int s = (int)(idx / HC), slot = (int)(idx % HC), h = slot / NC, c = slot % NC;
      gu[j] = idx < nout ? __ldg(reinterpret_cast<const uint4*>(a.g + b * a.g_sb + (int64_t)s * a.g_ss +
                                                                (int64_t)h * a.g_sh + c * 8))
                         : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t idx = i0 + j * kGaThreads;
      if (idx >= nout) break;
      const int s = (int)(idx / HC), slot = (int)(idx % HC), h = slot / NC, c = slot % NC;
      const uint32_t gw[4] = {gu[j].x, gu[j].y, gu[j].z, gu[j].w};
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        w[e] = pack_bf16(ga_sigmoid(bf16_lo(gw[e])) * sAt[h * D + c * 8 + 2 * e],
                         ga_sigmoid(bf16_hi(gw[e])) * sAt[h * D + c * 8 + 2 * e + 1]);
      *reinterpret_cast<uint4*>(a.o + b * a.o_sb + (int64_t)s * a.o_ss + (int64_t)h * a.o_sh + c * 8) =
          make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// ------------------------------------------------------------------ backward
template <int D>
__global__ void __launch_bounds__(kGaThreads) global_attn_bwd_kernel(const GaArgs a) {
  extern __shared__ float sm[];
  float* sA = sm;                              // [H][S]  a, later dlogit
  float* sDA = sA + a.H * a.S;                 // [H][S]  da
  float* sQ = sDA + a.H * a.S;                 // [H·D]  q̄
  float* sAt = sQ + a.H * D;                   // [H·D]  attn
  float* sDt = sAt + a.H * D;                  // [H·D]  dattn, later dq̄
  float* sOne = sDt + a.H * D;                 // [16]   ones / Dh
  float* red = sOne + 16;
  const int64_t b = blockIdx.x;
  constexpr int NC = D / 8;
  const int HC = a.H * NC;
  const int cnt = ga_count<D>(a, b, red);
  for (int i = threadIdx.x; i < a.H * D; i += kGaThreads) sQ[i] = a.qbar_in[b * a.H * D + i];
  for (int i = threadIdx.x; i < 16; i += kGaThreads) sOne[i] = 1.f;
  __syncthreads();
  if (cnt == 0) {  // no kept sequence: every gradient is zero
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (int64_t idx = threadIdx.x; idx < (int64_t)a.S * HC; idx += kGaThreads) {
      const int s = (int)(idx / HC), slot = (int)(idx % HC), h = slot / NC, c = slot % NC;
      *reinterpret_cast<uint4*>(a.dq + b * a.q_sb + (int64_t)s * a.q_ss + (int64_t)h * a.q_sh + c * 8) = z;
      *reinterpret_cast<uint4*>(a.dg + b * a.g_sb + (int64_t)s * a.g_ss + (int64_t)h * a.g_sh + c * 8) = z;
    }
    for (int64_t idx = threadIdx.x; idx < (int64_t)a.S * NC; idx += kGaThreads) {
      const int t = (int)(idx / NC), c = (int)(idx % NC);
      *reinterpret_cast<uint4*>(a.dk + b * a.k_sb + (int64_t)t * a.k_ss + c * 8) = z;
      *reinterpret_cast<uint4*>(a.dv + b * a.v_sb + (int64_t)t * a.v_ss + c * 8) = z;
    }
    return;
  }
  // a = exp(scale·q̄·k − lse), attn = Σ_t a v
  ga_scores<D>(a, b, sQ, sA);
  __syncthreads();
  for (int i = threadIdx.x; i < a.H * a.S; i += kGaThreads) {
    const float l = sA[i];
    sA[i] = l == -INFINITY ? 0.f : __expf(l - a.lse_in[b * a.H + i / a.S]);
  }
  __syncthreads();
  ga_weighted_v<D>(a, b, sA, sOne, red, sAt);
  // dattn[h][:] = Σ_s dO ⊙ σ(g);  dg = dO ⊙ attn ⊙ σ(1−σ)   (stream over s)
  {
    const int ngrp = kGaThreads / HC;
    const int slot = threadIdx.x % HC, grp = threadIdx.x / HC;
    const int h = slot / NC, c = slot % NC;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (grp < ngrp) {
#pragma unroll 2
      for (int s = grp; s < a.S; s += ngrp) {
        float gv[8], dov[8];
        ga_load<8>(a.g + b * a.g_sb + (int64_t)s * a.g_ss + (int64_t)h * a.g_sh + c * 8, gv);
        ga_load<8>(a.dout + b * a.o_sb + (int64_t)s * a.o_ss + (int64_t)h * a.o_sh + c * 8, dov);
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          const float s0 = ga_sigmoid(gv[e]), s1 = ga_sigmoid(gv[e + 1]);
          acc[e] = fmaf(dov[e], s0, acc[e]);
          acc[e + 1] = fmaf(dov[e + 1], s1, acc[e + 1]);
          w[e / 2] = pack_bf16(dov[e] * sAt[h * D + c * 8 + e] * s0 * (1.f - s0),
                               dov[e + 1] * sAt[h * D + c * 8 + e + 1] * s1 * (1.f - s1));
        }
        *reinterpret_cast<uint4*>(a.dg + b * a.g_sb + (int64_t)s * a.g_ss + (int64_t)h * a.g_sh + c * 8) =
            make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    __syncthreads();
    if (grp < ngrp)
#pragma unroll
      for (int e = 0; e < 8; ++e) red[grp * (HC * 8) + slot * 8 + e] = acc[e];
    __syncthreads();
    for (int i = threadIdx.x; i < HC * 8; i += kGaThreads) {
      float t = 0.f;
      for (int gI = 0; gI < ngrp; ++gI) t += red[gI * (HC * 8) + i];
      sDt[i] = t;
    }
    __syncthreads();
  }
  // per key t: da_h = dattn_h·v_t, dv_t = Σ_h a_ht dattn_h; then Dh = Σ_t a·da
  float dh_part[16];
#pragma unroll
  for (int h = 0; h < 16; ++h) dh_part[h] = 0.f;
  for (int t = threadIdx.x; t < a.S; t += kGaThreads) {
    float vv[D], dvv[D];
    ga_load<D>(a.v + b * a.v_sb + (int64_t)t * a.v_ss, vv);
#pragma unroll
    for (int d = 0; d < D; ++d) dvv[d] = 0.f;
#pragma unroll
    for (int h = 0; h < 16; ++h) {  // (unrolled with a guard: dh_part stays in registers)
      if (h >= a.H) break;
      const float w = sA[h * a.S + t];
      float da = 0.f;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        da = fmaf(sDt[h * D + d], vv[d], da);
        dvv[d] = fmaf(w, sDt[h * D + d], dvv[d]);
      }
      sDA[h * a.S + t] = da;
      dh_part[h] = fmaf(w, da, dh_part[h]);
    }
#pragma unroll
    for (int c = 0; c < D; c += 8) {
      uint32_t w4[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) w4[e] = pack_bf16(dvv[c + 2 * e], dvv[c + 2 * e + 1]);
      *reinterpret_cast<uint4*>(a.dv + b * a.v_sb + (int64_t)t * a.v_ss + c) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
    }
  }
  block_reduce_heads<false>(dh_part, a.H, red);
  if (threadIdx.x == 0)
#pragma unroll
    for (int h = 0; h < 16; ++h)
      if (h < a.H) sOne[h] = dh_part[h];  // reuse: Dh per head
  __syncthreads();
  // dlogit = a ⊙ (da − Dh);  dk_t = scale·Σ_h dlogit_ht q̄_h
  for (int t = threadIdx.x; t < a.S; t += kGaThreads) {
    float dkv[D];
#pragma unroll
    for (int d = 0; d < D; ++d) dkv[d] = 0.f;
    for (int h = 0; h < a.H; ++h) {
      const float dl = sA[h * a.S + t] * (sDA[h * a.S + t] - sOne[h]);
      sA[h * a.S + t] = dl;
#pragma unroll
      for (int d = 0; d < D; ++d) dkv[d] = fmaf(dl, sQ[h * D + d], dkv[d]);
    }
#pragma unroll
    for (int c = 0; c < D; c += 8) {
      uint32_t w4[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) w4[e] = pack_bf16(dkv[c + 2 * e] * a.scale, dkv[c + 2 * e + 1] * a.scale);
      *reinterpret_cast<uint4*>(a.dk + b * a.k_sb + (int64_t)t * a.k_ss + c) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
    }
  }
  __syncthreads();
  // dq̄[h][:] = scale·Σ_t dlogit_ht k_t   (into sDt), then dq = m_s·dq̄ / cnt
  for (int i = threadIdx.x; i < 16; i += kGaThreads) sOne[i] = a.scale / (float)cnt;
  __syncthreads();
  {
    const int ntg = kGaThreads / a.H;
    const int h = threadIdx.x % a.H, tg = threadIdx.x / a.H;
    float acc[D];
#pragma unroll
    for (int d = 0; d < D; ++d) acc[d] = 0.f;
    if (tg < ntg) {
      for (int t = tg; t < a.S; t += ntg) {
        const float w = sA[h * a.S + t];
        if (w == 0.f) continue;
        float kv[D];
        ga_load<D>(a.k + b * a.k_sb + (int64_t)t * a.k_ss, kv);
#pragma unroll
        for (int d = 0; d < D; ++d) acc[d] = fmaf(w, kv[d], acc[d]);
      }
    }
    __syncthreads();
    if (tg < ntg)
#pragma unroll
      for (int d = 0; d < D; ++d) red[tg * (a.H * D) + h * D + d] = acc[d];
    __syncthreads();
    for (int i = threadIdx.x; i < a.H * D; i += kGaThreads) {
      float t = 0.f;
      for (int gI = 0; gI < ntg; ++gI) t += red[gI * (a.H * D) + i];
      sDt[i] = t * sOne[0];  // scale / cnt
    }
    __syncthreads();
  }
  for (int64_t idx = threadIdx.x; idx < (int64_t)a.S * HC; idx += kGaThreads) {
    const int s = (int)(idx / HC), slot = (int)(idx % HC), h = slot / NC, c = slot % NC;
    const bool keep = ga_keep(a, b, s);
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      w[e] = keep ? pack_bf16(sDt[h * D + c * 8 + 2 * e], sDt[h * D + c * 8 + 2 * e + 1]) : 0u;
    *reinterpret_cast<uint4*>(a.dq + b * a.q_sb + (int64_t)s * a.q_ss + (int64_t)h * a.q_sh + c * 8) =
        make_uint4(w[0], w[1], w[2], w[3]);
  }
}

template <int D>
static size_t ga_smem(const GaArgs& a, bool bwd) {
  // score rows (+ da rows in the backward) | q̄, attn, dattn (+1) x H·D | 16 | reductions
  const size_t red = (size_t)kGaThreads * (D > 8 ? D : 8);
  return ((bwd ? 2 : 1) * (size_t)a.H * a.S + 4 * (size_t)a.H * D + 16 + red) * 4;
}

template <int D>
static cudaError_t ga_launch(const GaArgs& a, bool bwd, cudaStream_t st) {
  const size_t smem = ga_smem<D>(a, bwd);
  if (bwd) {
    cudaError_t e = set_smem_once(global_attn_bwd_kernel<D>, smem);
    if (e != cudaSuccess) return e;
    global_attn_bwd_kernel<D><<<(unsigned)a.B, kGaThreads, smem, st>>>(a);
  } else {
    cudaError_t e = set_smem_once(global_attn_fwd_kernel<D>, smem);
    if (e != cudaSuccess) return e;
    global_attn_fwd_kernel<D><<<(unsigned)a.B, kGaThreads, smem, st>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace evo

namespace {
evo_status_t ga_fail(evo_status_t s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  evo::set_error_detail(buf);
  return s;
}
bool ga_al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

evo_status_t ga_check(const evo_global_attn_desc_t* d) {
  if (!d) return ga_fail(EVO_E_INVALID, "desc is NULL");
  if (d->B < 0 || d->S < 0 || d->H < 1) return ga_fail(EVO_E_SHAPE, "B, S >= 0 and H >= 1 required");
  if (d->D != 8 && d->D != 16 && d->D != 32)
    return ga_fail(EVO_E_UNSUPPORTED, "D = %d (supported: 8, 16, 32)", d->D);
  if (d->H > 16) return ga_fail(EVO_E_UNSUPPORTED, "H = %d > 16", d->H);
  if ((int64_t)d->H * d->S > 16384)
    return ga_fail(EVO_E_UNSUPPORTED, "H·S = %lld > 16384 (score rows in shared memory)",
                   (long long)d->H * d->S);
  if (!(d->scale > 0.f)) return ga_fail(EVO_E_INVALID, "scale must be > 0");
  const int64_t* strs[] = {d->q_str, d->g_str, d->o_str};
  for (auto p : strs)
    for (int i = 0; i < 3; ++i)
      if (p[i] % 8) return ga_fail(EVO_E_ALIGN, "q/g/o strides must be multiples of 8 elements");
  for (int i = 0; i < 2; ++i)
    if (d->k_str[i] % 8 || d->v_str[i] % 8)
      return ga_fail(EVO_E_ALIGN, "k/v strides must be multiples of 8 elements");
  return EVO_OK;
}

evo::GaArgs ga_args(const evo_global_attn_desc_t* d, const uint8_t* mask) {
  evo::GaArgs a{};
  a.B = d->B; a.S = d->S; a.H = d->H; a.D = d->D; a.scale = d->scale;
  a.q_sb = d->q_str[0]; a.q_ss = d->q_str[1]; a.q_sh = d->q_str[2];
  a.k_sb = d->k_str[0]; a.k_ss = d->k_str[1];
  a.v_sb = d->v_str[0]; a.v_ss = d->v_str[1];
  a.g_sb = d->g_str[0]; a.g_ss = d->g_str[1]; a.g_sh = d->g_str[2];
  a.o_sb = d->o_str[0]; a.o_ss = d->o_str[1]; a.o_sh = d->o_str[2];
  a.mask = d->has_mask ? mask : nullptr;
  a.m_sb = d->mask_str[0]; a.m_ss = d->mask_str[1];
  return a;
}

cudaError_t ga_dispatch(const evo::GaArgs& a, bool bwd, cudaStream_t st) {
  if (a.D == 8) return evo::ga_launch<8>(a, bwd, st);
  if (a.D == 16) return evo::ga_launch<16>(a, bwd, st);
  return evo::ga_launch<32>(a, bwd, st);
}
}  // namespace

extern "C" {

evo_status_t evo_global_attn_fwd(const evo_global_attn_desc_t* d, const void* q, const void* k,
                                 const void* v, const uint8_t* mask, const void* g, void* o,
                                 float* lse, float* qbar, void* stream) {
  evo_status_t s = ga_check(d);
  if (s) return s;
  if (!q || !k || !v || !g || !o || !lse || !qbar)
    return ga_fail(EVO_E_INVALID, "q, k, v, g, o, lse, qbar are required");
  if ((mask != nullptr) != (d->has_mask != 0)) return ga_fail(EVO_E_INVALID, "mask iff has_mask");
  for (const void* p : {q, k, v, g, (const void*)o})
    if (!ga_al16(p)) return ga_fail(EVO_E_ALIGN, "tensor pointer not 16-byte aligned");
  if (d->B == 0 || d->S == 0) return EVO_OK;
  evo::GaArgs a = ga_args(d, mask);
  a.q = (const __nv_bfloat16*)q; a.k = (const __nv_bfloat16*)k; a.v = (const __nv_bfloat16*)v;
  a.g = (const __nv_bfloat16*)g; a.o = (__nv_bfloat16*)o; a.lse = lse; a.qbar = qbar;
  cudaError_t e = ga_dispatch(a, false, reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? EVO_OK : ga_fail(EVO_E_CUDA, "global_attn_fwd: %s", cudaGetErrorString(e));
}

evo_status_t evo_global_attn_bwd(const evo_global_attn_desc_t* d, const void* q, const void* k,
                                 const void* v, const uint8_t* mask, const void* g,
                                 const float* lse, const float* qbar, const void* dout, void* dq,
                                 void* dk, void* dv, void* dg, void* stream) {
  evo_status_t s = ga_check(d);
  if (s) return s;
  if (!q || !k || !v || !g || !lse || !qbar || !dout || !dq || !dk || !dv || !dg)
    return ga_fail(EVO_E_INVALID, "every tensor argument is required");
  if ((mask != nullptr) != (d->has_mask != 0)) return ga_fail(EVO_E_INVALID, "mask iff has_mask");
  for (const void* p : {q, k, v, g, dout, (const void*)dq, (const void*)dk, (const void*)dv, (const void*)dg})
    if (!ga_al16(p)) return ga_fail(EVO_E_ALIGN, "tensor pointer not 16-byte aligned");
  if (d->B == 0 || d->S == 0) return EVO_OK;
  evo::GaArgs a = ga_args(d, mask);
  a.q = (const __nv_bfloat16*)q; a.k = (const __nv_bfloat16*)k; a.v = (const __nv_bfloat16*)v;
  a.g = (const __nv_bfloat16*)g; a.dout = (const __nv_bfloat16*)dout;
  a.dq = (__nv_bfloat16*)dq; a.dk = (__nv_bfloat16*)dk; a.dv = (__nv_bfloat16*)dv;
  a.dg = (__nv_bfloat16*)dg; a.lse_in = lse; a.qbar_in = qbar;
  cudaError_t e = ga_dispatch(a, true, reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? EVO_OK : ga_fail(EVO_E_CUDA, "global_attn_bwd: %s", cudaGetErrorString(e));
}

}  // extern "C"
