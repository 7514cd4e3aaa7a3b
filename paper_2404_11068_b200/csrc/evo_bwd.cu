// evo_bwd.cu — bf16 backward of Evoformer gated attention with pair bias on sm_100a.
//
// Recompute backward ("re-derive probabilities tile-by-tile from saved row
// statistics").  With A = Σ_k p_k V_k (ungated), o = σ(G)⊙A:
//   a7   bwd_pre:   D_q = Σ_d dO·o,  dA = dO⊙σ(G),  dG = dO⊙o⊙(1-σ(G)),  lse2 = lse·log2e
//   a8-12 bwd_main (CTA per (b, h, 128-key tile), loop over 128-query tiles, tcgen05):
//        Sᵀ = K·Qᵀ,  dPᵀ = V·dAᵀ                       (TMEM, M = keys)
//        Pᵀ = exp2(Sᵀ·scale·log2e + biasᵀ·log2e - lse2),  dSᵀ = Pᵀ⊙(dPᵀ - D)   (8 warps)
//        dV += Pᵀ·dA,  dK += dSᵀ·Q,  dQ_part = dS·K      (TMEM; dQ parts summed in fp32)
//   a13  bwd_bias  (CTA per (h, q tile, k tile, batch chunk)): dS recomputed, Σ_b dS held in
//        registers over the chunk -> fp32 partials -> deterministic reduce (no atomics on dbias)
//   a14  dq_convert: dq = bf16(scale · Σ dQ_part)
#include <cstdlib>

#include "evo_kernels.cuh"

namespace evo {

// =============================================================================== bwd_pre
// CTA per (b, 32 query rows) x all heads.  Rows are visited in the order of the smaller of the
// (h, l) strides of o, so a warp's 16-byte loads/stores cover consecutive memory; the per-row
// statistics go through shared memory and leave as coalesced [B*H][Lq_pad] vectors.
template <bool F32, int DP>
__global__ void __launch_bounds__(256) bwd_pre_kernel(const BwdPreArgs a) {
  constexpr int kHC = 16;  // heads per pass
  __shared__ float sD[kHC][32], sL[kHC][32];
  const int Lq_pad = ((a.Lq + 127) / 128) * 128;
  const int nqb = Lq_pad / 32;
  const bool hfast = a.o_sh < a.o_sl;
  const float sgn = a.negate ? -1.f : 1.f;
  // persistent over (b, 32-query block) items: a short-lived block per item left the SMs half
  // empty (one wave with a long ramp-down)
  const int64_t nitems = (int64_t)a.B * nqb;
  for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
  const int64_t b = item / nqb;
  const int q0 = (int)(item % nqb) * 32;
  for (int h0 = 0; h0 < a.H; h0 += kHC) {
    const int hc = min(kHC, a.H - h0);
    for (int r = threadIdx.x; r < 32 * hc; r += blockDim.x) {
      const int qi = hfast ? r / hc : r % 32, hi = hfast ? r % hc : r / 32;
      const int q = q0 + qi, h = h0 + hi;
      float Dq = 0.f, lv = F32 ? 0.f : sgn * INFINITY;  // padding rows: inert
      if (q < a.Lq) {
        const int64_t orow = b * a.o_sb + h * a.o_sh + (int64_t)q * a.o_sl;
        const int64_t grow = b * a.g_sb + h * a.g_sh + (int64_t)q * a.g_sl;
        const int64_t arow = b * a.a_sb + h * a.a_sh + (int64_t)q * a.a_sl;
        if (!F32) {
          // bf16: issue every load of the row (o, dO, g, lse) before the first store — the
          // stores may alias the inputs as far as the compiler knows, so it would not hoist them
          constexpr int NV = DP / 8;
          uint4 ov[NV], dv[NV], gv[NV];
          const __nv_bfloat16* o_p = reinterpret_cast<const __nv_bfloat16*>(a.o) + orow;
          const __nv_bfloat16* d_p = reinterpret_cast<const __nv_bfloat16*>(a.dout) + orow;
          const __nv_bfloat16* g_p = reinterpret_cast<const __nv_bfloat16*>(a.g) + grow;
#pragma unroll
          for (int x = 0; x < NV; ++x) {
            ov[x] = dv[x] = gv[x] = make_uint4(0, 0, 0, 0);
            if (x * 8 < a.D) {
              ov[x] = __ldg(reinterpret_cast<const uint4*>(o_p + x * 8));
              dv[x] = __ldg(reinterpret_cast<const uint4*>(d_p + x * 8));
              if (a.g) gv[x] = __ldg(reinterpret_cast<const uint4*>(g_p + x * 8));
            }
          }
          const float l = a.lse[(b * a.H + h) * a.Lq + q];
#pragma unroll
          for (int x = 0; x < NV; ++x) {
            if (x * 8 >= a.D) break;
            const uint32_t ou[4] = {ov[x].x, ov[x].y, ov[x].z, ov[x].w};
            const uint32_t du[4] = {dv[x].x, dv[x].y, dv[x].z, dv[x].w};
            const uint32_t gu[4] = {gv[x].x, gv[x].y, gv[x].z, gv[x].w};
            uint32_t pa[4], pg[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float o0 = bf16_lo(ou[e]), o1 = bf16_hi(ou[e]);
              const float d0v = bf16_lo(du[e]), d1v = bf16_hi(du[e]);
              Dq = fmaf(d0v, o0, fmaf(d1v, o1, Dq));
              if (a.g) {
                const float s0 = 1.f / (1.f + __expf(-bf16_lo(gu[e])));
                const float s1 = 1.f / (1.f + __expf(-bf16_hi(gu[e])));
                pa[e] = pack_bf16(d0v * s0, d1v * s1);
                pg[e] = pack_bf16(d0v * o0 * (1.f - s0), d1v * o1 * (1.f - s1));
              }
            }
            if (a.g) {
              *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.dA) + arow + x * 8) =
                  make_uint4(pa[0], pa[1], pa[2], pa[3]);
              *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.dg) + grow + x * 8) =
                  make_uint4(pg[0], pg[1], pg[2], pg[3]);
            }
          }
          lv = sgn * (l == -INFINITY ? INFINITY : l * kLog2e);  // no kept key -> P = 0
        } else {
#pragma unroll
        for (int d0 = 0; d0 < DP; d0 += 8) {  // fp32 verification path
          if (d0 >= a.D) break;
          float o8[8], do8[8], g8[8];
          if (F32) {
            const float* op = reinterpret_cast<const float*>(a.o) + orow + d0;
            const float* dp = reinterpret_cast<const float*>(a.dout) + orow + d0;
#pragma unroll
            for (int e = 0; e < 8; ++e) { o8[e] = op[e]; do8[e] = dp[e]; }
            if (a.g) {
              const float* gp = reinterpret_cast<const float*>(a.g) + grow + d0;
#pragma unroll
              for (int e = 0; e < 8; ++e) g8[e] = gp[e];
            }
          } else {
            const uint4 ov = *reinterpret_cast<const uint4*>(
                reinterpret_cast<const __nv_bfloat16*>(a.o) + orow + d0);
            const uint4 dv = *reinterpret_cast<const uint4*>(
                reinterpret_cast<const __nv_bfloat16*>(a.dout) + orow + d0);
            const uint32_t ou[4] = {ov.x, ov.y, ov.z, ov.w}, du[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              o8[2 * e] = bf16_lo(ou[e]); o8[2 * e + 1] = bf16_hi(ou[e]);
              do8[2 * e] = bf16_lo(du[e]); do8[2 * e + 1] = bf16_hi(du[e]);
            }
            if (a.g) {
              const uint4 gv = *reinterpret_cast<const uint4*>(
                  reinterpret_cast<const __nv_bfloat16*>(a.g) + grow + d0);
              const uint32_t gu[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) { g8[2 * e] = bf16_lo(gu[e]); g8[2 * e + 1] = bf16_hi(gu[e]); }
            }
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) Dq = fmaf(do8[e], o8[e], Dq);
          if (a.g) {
            float da[8], dg[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float sg = F32 ? 1.f / (1.f + expf(-g8[e])) : 1.f / (1.f + __expf(-g8[e]));
              da[e] = do8[e] * sg;
              dg[e] = do8[e] * o8[e] * (1.f - sg);
            }
            if (F32) {
              float* dap = reinterpret_cast<float*>(a.dA) + arow + d0;
              float* dgp = reinterpret_cast<float*>(a.dg) + grow + d0;
#pragma unroll
              for (int e = 0; e < 8; ++e) { dap[e] = da[e]; dgp[e] = dg[e]; }
            } else {
              uint4 x, y;
              x.x = pack_bf16(da[0], da[1]); x.y = pack_bf16(da[2], da[3]);
              x.z = pack_bf16(da[4], da[5]); x.w = pack_bf16(da[6], da[7]);
              y.x = pack_bf16(dg[0], dg[1]); y.y = pack_bf16(dg[2], dg[3]);
              y.z = pack_bf16(dg[4], dg[5]); y.w = pack_bf16(dg[6], dg[7]);
              *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.dA) + arow + d0) = x;
              *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.dg) + grow + d0) = y;
            }
          }
        }
        }
      }
      sD[hi][qi] = sgn * Dq;
      sL[hi][qi] = lv;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < 32 * hc; r += blockDim.x) {  // coalesced along q
      const int hi = r / 32, qi = r % 32;
      const int64_t v = (b * a.H + h0 + hi) * Lq_pad + q0 + qi;
      a.Dvec[v] = sD[hi][qi];
      if (!F32) a.lse2[v] = sL[hi][qi];
    }
    __syncthreads();
  }
  }
}

// bf16 path, chunk per thread: NCH = D/8 consecutive lanes share a row, one 16-byte chunk each,
// rows in the memory order of o (the smaller of its (h, l) strides fastest), so every warp-wide
// load/store covers 512 contiguous bytes when the rows are dense; Σ_d dO·o by xor-shuffles inside
// the row's lanes.  Two chunks per thread per iteration, all five loads in flight before the math.
template <int NCH>
__global__ void __launch_bounds__(256) bwd_pre_vec_kernel(const BwdPreArgs a) {
  const int Lq_pad = ((a.Lq + 127) / 128) * 128;
  const bool hfast = a.o_sh < a.o_sl;
  const float sgn = a.negate ? -1.f : 1.f;
  const uint32_t H = (uint32_t)a.H, Lq = (uint32_t)a.Lq;
  const uint32_t n = (uint32_t)a.B * H * Lq * NCH;
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t c = threadIdx.x % NCH;
  const __nv_bfloat16* o_p = reinterpret_cast<const __nv_bfloat16*>(a.o);
  const __nv_bfloat16* d_p = reinterpret_cast<const __nv_bfloat16*>(a.dout);
  const __nv_bfloat16* g_p = reinterpret_cast<const __nv_bfloat16*>(a.g);
  const uint64_t zpol = l2_policy_evict_last();
  for (uint32_t i0 = blockIdx.x * blockDim.x; i0 < n; i0 += 2 * stride) {  // block-uniform trip
    uint4 ov[2], dv[2], gv[2];
    float l[2];
    int64_t orow[2], grow[2], arow[2], vrow[2], zrow[2];
    bool ok[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t idx = i0 + u * stride + threadIdx.x;
      ok[u] = idx < n;
      uint32_t r = (ok[u] ? idx : 0u) / NCH, h, q, r2;
      if (hfast) {
        r2 = fdiv(r, a.fd_H); h = r - r2 * H; r = r2;
        r2 = fdiv(r, a.fd_Lq); q = r - r2 * Lq; r = r2;
      } else {
        r2 = fdiv(r, a.fd_Lq); q = r - r2 * Lq; r = r2;
        r2 = fdiv(r, a.fd_H); h = r - r2 * H; r = r2;
      }
      const int64_t b = r;
      orow[u] = b * a.o_sb + h * a.o_sh + (int64_t)q * a.o_sl + c * 8;
      grow[u] = b * a.g_sb + h * a.g_sh + (int64_t)q * a.g_sl + c * 8;
      arow[u] = b * a.a_sb + h * a.a_sh + (int64_t)q * a.a_sl + c * 8;
      vrow[u] = (b * H + h) * Lq_pad + q;
      zrow[u] = b * a.z_sb + h * a.z_sh + (int64_t)q * a.z_sl + c * 8;
      ov[u] = dv[u] = gv[u] = make_uint4(0, 0, 0, 0);
      l[u] = 0.f;
      if (ok[u]) {
        ov[u] = __ldg(reinterpret_cast<const uint4*>(o_p + orow[u]));
        dv[u] = __ldg(reinterpret_cast<const uint4*>(d_p + orow[u]));
        if (g_p) gv[u] = __ldg(reinterpret_cast<const uint4*>(g_p + grow[u]));
        l[u] = __ldg(a.lse + (b * H + h) * Lq + q);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t ou[4] = {ov[u].x, ov[u].y, ov[u].z, ov[u].w};
      const uint32_t du[4] = {dv[u].x, dv[u].y, dv[u].z, dv[u].w};
      const uint32_t gu[4] = {gv[u].x, gv[u].y, gv[u].z, gv[u].w};
      uint32_t pa[4], pg[4];
      float Dq = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float o0 = bf16_lo(ou[e]), o1 = bf16_hi(ou[e]);
        const float d0v = bf16_lo(du[e]), d1v = bf16_hi(du[e]);
        Dq = fmaf(d0v, o0, fmaf(d1v, o1, Dq));
        const float s0 = fast_sigmoid(bf16_lo(gu[e])), s1 = fast_sigmoid(bf16_hi(gu[e]));
        pa[e] = pack_bf16(d0v * s0, d1v * s1);
        pg[e] = pack_bf16(d0v * o0 * (1.f - s0), d1v * o1 * (1.f - s1));
      }
#pragma unroll
      for (int m = 1; m < NCH; m <<= 1) Dq += __shfl_xor_sync(0xffffffffu, Dq, m);
      if (!ok[u]) continue;
      if (a.zacc) {
        float4* z = reinterpret_cast<float4*>(a.zacc + zrow[u]);
        // evict_last: keep the zeroed lines in L2 for bwd_fused's adds
        asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %1, %1, %1}, %2;" ::"l"(z), "f"(0.f), "l"(zpol) : "memory");
        asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %1, %1, %1}, %2;" ::"l"(z + 1), "f"(0.f), "l"(zpol) : "memory");
      }
      if (g_p) {
        *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.dA) + arow[u]) =
            make_uint4(pa[0], pa[1], pa[2], pa[3]);
        *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.dg) + grow[u]) =
            make_uint4(pg[0], pg[1], pg[2], pg[3]);
      }
      if (c == 0) {
        a.Dvec[vrow[u]] = sgn * Dq;
        a.lse2[vrow[u]] = sgn * (l[u] == -INFINITY ? INFINITY : l[u] * kLog2e);  // no kept key -> P = 0
      }
    }
  }
  // padding query rows [Lq, Lq_pad) of the statistics vectors: inert (D = 0, P = 0)
  const uint32_t npad = (uint32_t)a.B * H * (uint32_t)(Lq_pad - a.Lq);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < npad; i += stride) {
    const uint32_t bh = i / (uint32_t)(Lq_pad - a.Lq), q = Lq + i % (uint32_t)(Lq_pad - a.Lq);
    a.Dvec[(int64_t)bh * Lq_pad + q] = 0.f;
    a.lse2[(int64_t)bh * Lq_pad + q] = sgn * INFINITY;
  }
}

cudaError_t launch_bwd_pre(const BwdPreArgs& a, int f32, cudaStream_t st) {
  const int Lq_pad = ((a.Lq + 127) / 128) * 128;
  const int64_t items = (int64_t)a.B * (Lq_pad / 32);
  if (items == 0) return cudaSuccess;
  const int64_t nvec = (int64_t)a.B * a.H * Lq_pad * (a.D / 8);
  // only the vector path zero-fills a dQ accumulator; the caller selects it whenever it asks
  if (a.zacc && !(!f32 && a.D % 8 == 0 && nvec < ((int64_t)1 << 31) )) return cudaErrorInvalidValue;
  if (!f32 && a.D % 8 == 0 && nvec < ((int64_t)1 << 31) ) {
    BwdPreArgs v = a;
    v.fd_H = make_fastdiv((uint32_t)a.H);
    v.fd_Lq = make_fastdiv((uint32_t)a.Lq);
    const int64_t blocks = (nvec + 511) / 512;  // two chunks per thread
    const unsigned g = (unsigned)(blocks < 148 * 8 ? blocks : 148 * 8);
    switch (a.D / 8) {
      case 1: bwd_pre_vec_kernel<1><<<g, 256, 0, st>>>(v); break;
      case 2: bwd_pre_vec_kernel<2><<<g, 256, 0, st>>>(v); break;
      case 4: bwd_pre_vec_kernel<4><<<g, 256, 0, st>>>(v); break;
      case 8: bwd_pre_vec_kernel<8><<<g, 256, 0, st>>>(v); break;
      default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
  }
  const unsigned g = (unsigned)(items < 148 * 6 ? items : 148 * 6);
  if (f32) {
    if (a.D <= 16) bwd_pre_kernel<true, 16><<<g, 256, 0, st>>>(a);
    else if (a.D <= 32) bwd_pre_kernel<true, 32><<<g, 256, 0, st>>>(a);
    else bwd_pre_kernel<true, 64><<<g, 256, 0, st>>>(a);
  } else {
    if (a.D <= 16) bwd_pre_kernel<false, 16><<<g, 256, 0, st>>>(a);
    else if (a.D <= 32) bwd_pre_kernel<false, 32><<<g, 256, 0, st>>>(a);
    else bwd_pre_kernel<false, 64><<<g, 256, 0, st>>>(a);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------- shared helpers
// Bias value at (q, k) of a 128x128 bias tile held as two 16 KB SW128 regions whose rows are
// the non-contiguous index and whose 64-wide column blocks are the contiguous index.
//   rows = q, cols = k  (k-contiguous bias, "mode 1")   or   rows = k, cols = q  ("mode 2")
EVO_DEV float bias_at(uint32_t sB, uint32_t r, uint32_t c) {
  return bf16_to_f(ld_shared_u16(sB + (c >> 6) * 16384 + r * 128 +
                                 ((((c & 63) >> 3) ^ (r & 7)) << 4) + (c & 7) * 2));
}
// 64 consecutive columns [64*half, 64*half+64) of row r, as fp32 scaled by log2(e), added to v
EVO_DEV void add_bias_row64(uint32_t sB, uint32_t r, uint32_t half, float (&v)[64]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint4 x = ld_shared_v4(sB + half * 16384 + swz_offset(r, c, 128));
    const uint32_t u[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[c * 8 + 2 * e] = fmaf(bf16_lo(u[e]), kLog2e, v[c * 8 + 2 * e]);
      v[c * 8 + 2 * e + 1] = fmaf(bf16_hi(u[e]), kLog2e, v[c * 8 + 2 * e + 1]);
    }
  }
}
EVO_DEV void tmem_ld64(uint32_t taddr, float (&v)[64], float mul) {
  uint32_t r[32];
  tmem_ld32(taddr, r);
  tmem_wait_ld();
#pragma unroll
  for (int c = 0; c < 32; ++c) v[c] = __uint_as_float(r[c]) * mul;
  tmem_ld32(taddr + 32, r);
  tmem_wait_ld();
#pragma unroll
  for (int c = 0; c < 32; ++c) v[32 + c] = __uint_as_float(r[c]) * mul;
}
EVO_DEV void store_row64_bf16(uint32_t base, uint32_t row, const float (&v)[64]) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
    st_shared_v4(base + swz_offset(row, c, 128), pack_bf16(v[8 * c], v[8 * c + 1]),
                 pack_bf16(v[8 * c + 2], v[8 * c + 3]), pack_bf16(v[8 * c + 4], v[8 * c + 5]),
                 pack_bf16(v[8 * c + 6], v[8 * c + 7]));
}

// =============================================================================== bwd_main
template <int DP, int BIAS>
__global__ void __launch_bounds__(256, 1) bwd_main_kernel(const __grid_constant__ CUtensorMap tm_q,
                                                           const __grid_constant__ CUtensorMap tm_k,
                                                           const __grid_constant__ CUtensorMap tm_v,
                                                           const __grid_constant__ CUtensorMap tm_da,
                                                           const __grid_constant__ CUtensorMap tm_b,
                                                           const BwdMainArgs a) {
  constexpr uint32_t kRowBytes = DP * 2;
  constexpr uint32_t kTileBytes = 128 * kRowBytes;
  constexpr uint32_t kSw = DP == 64 ? kSw128 : (DP == 32 ? kSw64 : kSw32);
  constexpr uint32_t kHalfCols = DP / 2;
  constexpr uint32_t kStageBytes = 2 * kTileBytes + (BIAS ? 32768u : 0u) + 1024u;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;  // dynamic smem base is 1024-aligned (no static smem); checked:
  if (smem_u32(smem) & 1023u) __trap();
  const uint32_t s0 = smem_u32(smem);
  const uint32_t sPt = s0;                 // 32 KB: Pᵀ  [128 keys][128 q] bf16, 2 SW128 regions
  const uint32_t sdSt = s0 + 32768;        // 32 KB: dSᵀ
  const uint32_t sBias = s0 + 65536;       // 2 x 32 KB (stage s)
  const uint32_t sK = s0 + 131072;
  const uint32_t sV = sK + kTileBytes;
  const uint32_t sQ = sV + kTileBytes;     // 2 stages
  const uint32_t sdA = sQ + 2 * kTileBytes;  // 2 stages
  const uint32_t sVec = sdA + 2 * kTileBytes;  // 2 stages x (lse2[128], D[128]) fp32
  float* vec = reinterpret_cast<float*>(smem + (sVec - s0));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (sVec - s0) + 2048);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);
  const uint32_t bar_kv = smem_u32(&bars[0]);
  const uint32_t bar_in0 = smem_u32(&bars[1]);  // +8: stage 1
  const uint32_t bar_sp = smem_u32(&bars[3]);
  const uint32_t bar_mm = smem_u32(&bars[4]);
  (void)kStageBytes;

  const uint32_t tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const uint32_t qd = w & 3, hh = w >> 2, row = qd * 32 + lane;
  const int nq = (a.Lq + 127) >> 7, nk = (a.Lk + 127) >> 7;
  const int Lq_pad = nq * 128;
  const int j = blockIdx.x % nk;
  const int bh = blockIdx.x / nk;
  const int h = bh % a.H;
  const int b = bh / a.H;
  const int k0 = j * 128;
  const int bcoord = a.bias_batched ? b : 0;

  if (w == 0) tmem_alloc<512>(smem_u32(tmem_slot));
  if (tid == 0) {
    mbar_init(bar_kv, 1);
    mbar_init(bar_in0, 1);
    mbar_init(bar_in0 + 8, 1);
    mbar_init(bar_sp, 1);
    mbar_init(bar_mm, 1);
    fence_barrier_init();
  }
  // this thread's key row (TMEM lane for Sᵀ/dPᵀ/dV/dK): validity incl. the hard mask
  const int kk = k0 + (int)row;
  bool keep = kk < a.Lk;
  if (keep && a.mask) keep = a.mask[(int64_t)b * a.mask_s0 + (int64_t)kk * a.mask_s1] != 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tSt = tmem, tdPt = tmem + 128, tdV = tmem + 256, tdK = tmem + 256 + DP,
                 tdQ = tmem + 256 + 2 * DP;
  const uint32_t lane_base = (qd * 32) << 16;

  constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, 0, 0);   // Sᵀ, dPᵀ
  constexpr uint32_t idesc_kv = make_idesc_bf16(128, DP, 0, 1);   // dV, dK (B MN-major)
  constexpr uint32_t idesc_q = make_idesc_bf16(128, DP, 1, 1);    // dQ (A and B MN-major)
  const float* vec_src_l = a.lse2 + (int64_t)bh * Lq_pad;
  const float* vec_src_d = a.Dvec + (int64_t)bh * Lq_pad;

  auto load_stage = [&](int s, int i) {  // Q_i, dA_i, bias(i, j), lse2/D of tile i
    const uint32_t bar = bar_in0 + 8 * s;
    mbar_arrive_expect_tx(bar, 2 * kTileBytes + (BIAS ? 32768u : 0u) + 1024u);
    tma_load_4d(sQ + s * kTileBytes, &tm_q, bar, 0, i * 128, h, b);
    tma_load_4d(sdA + s * kTileBytes, &tm_da, bar, 0, i * 128, h, b);
    if (BIAS) {
      for (int r = 0; r < 2; ++r) {
        if (BIAS == 1)  // rows q, cols k
          tma_load_4d(sBias + s * 32768 + r * 16384, &tm_b, bar, k0 + r * 64, i * 128, h, bcoord);
        else            // rows k, cols q
          tma_load_4d(sBias + s * 32768 + r * 16384, &tm_b, bar, i * 128 + r * 64, k0, h, bcoord);
      }
    }
    bulk_load(sVec + s * 1024, vec_src_l + i * 128, 512, bar);
    bulk_load(sVec + s * 1024 + 512, vec_src_d + i * 128, 512, bar);
  };
  auto issue_sp = [&](int s) {  // Sᵀ = K·Q_sᵀ, dPᵀ = V·dA_sᵀ
#pragma unroll
    for (int t = 0; t < DP / 16; ++t)
      umma_bf16(tSt, make_sdesc(sK + t * 32, 16, 8 * kRowBytes, kSw),
                make_sdesc(sQ + s * kTileBytes + t * 32, 16, 8 * kRowBytes, kSw), idesc_s, t > 0);
#pragma unroll
    for (int t = 0; t < DP / 16; ++t)
      umma_bf16(tdPt, make_sdesc(sV + t * 32, 16, 8 * kRowBytes, kSw),
                make_sdesc(sdA + s * kTileBytes + t * 32, 16, 8 * kRowBytes, kSw), idesc_s, t > 0);
    umma_commit(bar_sp);
  };

  if (tid == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_da);
    if (BIAS) tma_prefetch_desc(&tm_b);
    mbar_arrive_expect_tx(bar_kv, 2 * kTileBytes);
    tma_load_4d(sK, &tm_k, bar_kv, 0, k0, h, b);
    tma_load_4d(sV, &tm_v, bar_kv, 0, k0, h, b);
    for (int s = 0; s < 2 && s < nq; ++s) load_stage(s, s);
    mbar_wait(bar_kv, 0);
    mbar_wait(bar_in0, 0);
    tc_fence_after();
    issue_sp(0);
  }

  for (int i = 0; i < nq; ++i) {
    const int s = i & 1;
    const uint32_t sB = sBias + s * 32768;
    const float* lse2v = vec + s * 256;
    const float* Dv = lse2v + 128;
    mbar_wait(bar_in0 + 8 * s, (i >> 1) & 1);  // vectors + bias of tile i visible
    mbar_wait(bar_sp, i & 1);
    tc_fence_after();
    float p[64], ds[64];
    tmem_ld64(tSt + lane_base + hh * 64, p, a.scale_log2);
    if (BIAS == 1) {  // bias tile rows q, cols k: column `row`
#pragma unroll
      for (int c = 0; c < 64; ++c) p[c] = fmaf(bias_at(sB, hh * 64 + c, row), kLog2e, p[c]);
    } else if (BIAS == 2) {  // rows k, cols q: row `row`, block hh
      add_bias_row64(sB, row, hh, p);
    }
#pragma unroll
    for (int c = 0; c < 64; ++c) p[c] = keep ? fast_exp2(p[c] - lse2v[hh * 64 + c]) : 0.f;
    tmem_ld64(tdPt + lane_base + hh * 64, ds, 1.f);
#pragma unroll
    for (int c = 0; c < 64; ++c) ds[c] = p[c] * (ds[c] - Dv[hh * 64 + c]);
    store_row64_bf16(sPt + hh * 16384, row, p);
    store_row64_bf16(sdSt + hh * 16384, row, ds);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t qb = sQ + s * kTileBytes, ab = sdA + s * kTileBytes;
#pragma unroll
      for (int t = 0; t < 8; ++t) {  // dV += Pᵀ·dA_i
        umma_bf16(tdV, make_sdesc(sPt + (t >> 2) * 16384 + (t & 3) * 32, 16, 1024, kSw128),
                  make_sdesc(ab + t * 16 * kRowBytes, 16384, 8 * kRowBytes, kSw), idesc_kv,
                  (i > 0 || t > 0) ? 1u : 0u);
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) {  // dK += dSᵀ·Q_i
        umma_bf16(tdK, make_sdesc(sdSt + (t >> 2) * 16384 + (t & 3) * 32, 16, 1024, kSw128),
                  make_sdesc(qb + t * 16 * kRowBytes, 16384, 8 * kRowBytes, kSw), idesc_kv,
                  (i > 0 || t > 0) ? 1u : 0u);
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) {  // dQ_part = dS·K_j  (A = dSᵀ buffer read MN-major)
        umma_bf16(tdQ, make_sdesc(sdSt + t * 2048, 16384, 1024, kSw128),
                  make_sdesc(sK + t * 16 * kRowBytes, 16384, 8 * kRowBytes, kSw), idesc_q,
                  t > 0 ? 1u : 0u);
      }
      umma_commit(bar_mm);
      if (i + 1 < nq) {
        mbar_wait(bar_in0 + 8 * (s ^ 1), ((i + 1) >> 1) & 1);
        tc_fence_after();
        issue_sp(s ^ 1);
      }
    }
    mbar_wait(bar_mm, i & 1);
    tc_fence_after();
    if (tid == 0 && i + 2 < nq) load_stage(s, i + 2);
    // dQ part: TMEM lane = query row
    const int q = i * 128 + (int)row;
    const bool qvalid = q < a.Lq;
#pragma unroll
    for (int c0 = 0; c0 < (int)kHalfCols; c0 += 8) {
      const int d0 = hh * kHalfCols + c0;
      uint32_t r[8];
      tmem_ld8(tdQ + lane_base + d0, r);
      tmem_wait_ld();
      if (qvalid && d0 < a.D) {
        if (nk == 1) {
          uint4 st;
          st.x = pack_bf16(__uint_as_float(r[0]) * a.scale, __uint_as_float(r[1]) * a.scale);
          st.y = pack_bf16(__uint_as_float(r[2]) * a.scale, __uint_as_float(r[3]) * a.scale);
          st.z = pack_bf16(__uint_as_float(r[4]) * a.scale, __uint_as_float(r[5]) * a.scale);
          st.w = pack_bf16(__uint_as_float(r[6]) * a.scale, __uint_as_float(r[7]) * a.scale);
          *reinterpret_cast<uint4*>(a.dq + (int64_t)b * a.q_sb + (int64_t)h * a.q_sh +
                                    (int64_t)q * a.q_sl + d0) = st;
        } else {
          // this key tile's own fp32 part (plain stores): dq_convert sums the nk parts in
          // key-tile order, so dq does not depend on the CTAs' completion order
          float4* dst = reinterpret_cast<float4*>(
              a.dq_acc + ((int64_t)j * a.B * a.H + bh) * (int64_t)a.Lq * a.D + (int64_t)q * a.D + d0);
          dst[0] = make_float4(__uint_as_float(r[0]), __uint_as_float(r[1]), __uint_as_float(r[2]),
                               __uint_as_float(r[3]));
          dst[1] = make_float4(__uint_as_float(r[4]), __uint_as_float(r[5]), __uint_as_float(r[6]),
                               __uint_as_float(r[7]));
        }
      }
    }
    tc_fence_before();
  }

  // dK, dV: TMEM lane = key row
  const bool kvalid = kk < a.Lk;
#pragma unroll
  for (int c0 = 0; c0 < (int)kHalfCols; c0 += 8) {
    const int d0 = hh * kHalfCols + c0;
    uint32_t rk[8], rv[8];
    tmem_ld8(tdK + lane_base + d0, rk);
    tmem_ld8(tdV + lane_base + d0, rv);
    tmem_wait_ld();
    if (kvalid && d0 < a.D) {
      uint4 x, y;
      x.x = pack_bf16(__uint_as_float(rk[0]) * a.scale, __uint_as_float(rk[1]) * a.scale);
      x.y = pack_bf16(__uint_as_float(rk[2]) * a.scale, __uint_as_float(rk[3]) * a.scale);
      x.z = pack_bf16(__uint_as_float(rk[4]) * a.scale, __uint_as_float(rk[5]) * a.scale);
      x.w = pack_bf16(__uint_as_float(rk[6]) * a.scale, __uint_as_float(rk[7]) * a.scale);
      y.x = pack_bf16(__uint_as_float(rv[0]), __uint_as_float(rv[1]));
      y.y = pack_bf16(__uint_as_float(rv[2]), __uint_as_float(rv[3]));
      y.z = pack_bf16(__uint_as_float(rv[4]), __uint_as_float(rv[5]));
      y.w = pack_bf16(__uint_as_float(rv[6]), __uint_as_float(rv[7]));
      *reinterpret_cast<uint4*>(a.dk + (int64_t)b * a.k_sb + (int64_t)h * a.k_sh +
                                (int64_t)kk * a.k_sl + d0) = x;
      *reinterpret_cast<uint4*>(a.dv + (int64_t)b * a.v_sb + (int64_t)h * a.v_sh +
                                (int64_t)kk * a.v_sl + d0) = y;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tmem);
}

template <int DP, int BIAS>
static cudaError_t launch_bwd_main_t(const BwdMainLaunch& L, cudaStream_t st) {
  auto kern = bwd_main_kernel<DP, BIAS>;
  const size_t smem = bwd_main_smem_bytes(DP);
  cudaError_t e = set_smem_once(kern, smem);
  if (e != cudaSuccess) return e;
  const int nk = (L.args.Lk + 127) / 128;
  const long long grid = (long long)L.args.B * L.args.H * nk;
  if (grid == 0) return cudaSuccess;
  kern<<<(unsigned)grid, 256, smem, st>>>(L.tm_q, L.tm_k, L.tm_v, L.tm_da, L.tm_b, L.args);
  return cudaGetLastError();
}

cudaError_t launch_bwd_main_bf16(const BwdMainLaunch& L, int DP, int bias_mode, cudaStream_t st) {
#define EVO_BWD_CASE(dp, bm) \
  if (DP == dp && bias_mode == bm) return launch_bwd_main_t<dp, bm>(L, st);
  EVO_BWD_CASE(16, 0) EVO_BWD_CASE(16, 1) EVO_BWD_CASE(16, 2)
  EVO_BWD_CASE(32, 0) EVO_BWD_CASE(32, 1) EVO_BWD_CASE(32, 2)
  EVO_BWD_CASE(64, 0) EVO_BWD_CASE(64, 1) EVO_BWD_CASE(64, 2)
#undef EVO_BWD_CASE
  return cudaErrorInvalidValue;
}

// =============================================================================== bwd_bias
// CTA per (h, q tile i, k tile j, batch chunk).  Thread = query row (TMEM lane) x key half.
// dS[b] for b in the chunk is recomputed with two tcgen05.mma (S = Q·Kᵀ, dP = dA·Vᵀ) into a
// double-buffered TMEM pair and summed in 64 fp32 registers per thread; the chunk's sum is
// written once as an fp32 partial (shared bias) or dS is written per b (per-batch bias).
template <int DP, int BIAS>
__global__ void __launch_bounds__(256, 1) bwd_bias_kernel(const __grid_constant__ CUtensorMap tm_q,
                                                           const __grid_constant__ CUtensorMap tm_k,
                                                           const __grid_constant__ CUtensorMap tm_v,
                                                           const __grid_constant__ CUtensorMap tm_da,
                                                           const __grid_constant__ CUtensorMap tm_b,
                                                           const BwdBiasArgs a) {
  constexpr uint32_t kRowBytes = DP * 2;
  constexpr uint32_t kTileBytes = 128 * kRowBytes;
  constexpr uint32_t kSw = DP == 64 ? kSw128 : (DP == 32 ? kSw64 : kSw32);
  constexpr uint32_t kStage = 4 * kTileBytes + 32768 + 1024;  // Q K V dA | bias | vectors

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;  // dynamic smem base is 1024-aligned (no static smem); checked:
  if (smem_u32(smem) & 1023u) __trap();
  const uint32_t s0 = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * kStage);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);
  const uint32_t bar_in0 = smem_u32(&bars[0]);  // +8 stage 1
  const uint32_t bar_sp0 = smem_u32(&bars[2]);  // +8 buffer 1

  const uint32_t tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const uint32_t qd = w & 3, hh = w >> 2, row = qd * 32 + lane;
  const int nq = (a.Lq + 127) >> 7, nk = (a.Lk + 127) >> 7;
  const int Lq_pad = nq * 128, Lk_pad = nk * 128;
  int u = blockIdx.x;
  const int c = u % a.nchunks; u /= a.nchunks;
  const int j = u % nk; u /= nk;
  const int i = u % nq;
  const int h = u / nq;
  const int b0 = c * a.chunk;
  const int nb = min(a.B - b0, a.chunk);
  const int q0 = i * 128, k0 = j * 128;
  if (nb <= 0) return;

  if (w == 0) tmem_alloc<512>(smem_u32(tmem_slot));
  if (tid == 0) {
    mbar_init(bar_in0, 1);
    mbar_init(bar_in0 + 8, 1);
    mbar_init(bar_sp0, 1);
    mbar_init(bar_sp0 + 8, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = (qd * 32) << 16;
  constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, 0, 0);

  auto stage_base = [&](int s) { return s0 + (uint32_t)s * kStage; };
  auto load_stage = [&](int s, int b, bool with_bias) {
    const uint32_t sb = stage_base(s), bar = bar_in0 + 8 * s;
    mbar_arrive_expect_tx(bar, 4 * kTileBytes + (with_bias ? 32768u : 0u) + 1024u);
    tma_load_4d(sb, &tm_q, bar, 0, q0, h, b);
    tma_load_4d(sb + kTileBytes, &tm_k, bar, 0, k0, h, b);
    tma_load_4d(sb + 2 * kTileBytes, &tm_v, bar, 0, k0, h, b);
    tma_load_4d(sb + 3 * kTileBytes, &tm_da, bar, 0, q0, h, b);
    if (with_bias) {
      const int bc = a.bias_batched ? b : 0;
      for (int r = 0; r < 2; ++r) {
        if (BIAS == 1)
          tma_load_4d(sb + 4 * kTileBytes + r * 16384, &tm_b, bar, k0 + r * 64, q0, h, bc);
        else
          tma_load_4d(sb + 4 * kTileBytes + r * 16384, &tm_b, bar, q0 + r * 64, k0, h, bc);
      }
    }
    const int64_t vrow = ((int64_t)b * a.H + h) * Lq_pad + q0;
    bulk_load(sb + 4 * kTileBytes + 32768, a.lse2 + vrow, 512, bar);
    bulk_load(sb + 4 * kTileBytes + 32768 + 512, a.Dvec + vrow, 512, bar);
  };
  auto issue_sp = [&](int s) {
    const uint32_t sb = stage_base(s);
    const uint32_t tS = tmem + s * 256, tdP = tS + 128;
#pragma unroll
    for (int t = 0; t < DP / 16; ++t)
      umma_bf16(tS, make_sdesc(sb + t * 32, 16, 8 * kRowBytes, kSw),
                make_sdesc(sb + kTileBytes + t * 32, 16, 8 * kRowBytes, kSw), idesc_s, t > 0);
#pragma unroll
    for (int t = 0; t < DP / 16; ++t)
      umma_bf16(tdP, make_sdesc(sb + 3 * kTileBytes + t * 32, 16, 8 * kRowBytes, kSw),
                make_sdesc(sb + 2 * kTileBytes + t * 32, 16, 8 * kRowBytes, kSw), idesc_s, t > 0);
    umma_commit(bar_sp0 + 8 * s);
  };

  if (tid == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_da);
    tma_prefetch_desc(&tm_b);
    for (int n = 0; n < 2 && n < nb; ++n) load_stage(n, b0 + n, a.bias_batched || n == 0);
    mbar_wait(bar_in0, 0);
    tc_fence_after();
    issue_sp(0);
  }

  float acc[64];
#pragma unroll
  for (int cc = 0; cc < 64; ++cc) acc[cc] = 0.f;
  const int qrow = q0 + (int)row;

  for (int n = 0; n < nb; ++n) {
    const int s = n & 1;
    const int b = b0 + n;
    const uint32_t sb = stage_base(s);
    const uint32_t sBias = (a.bias_batched ? sb : stage_base(0)) + 4 * kTileBytes;
    const float* vec = reinterpret_cast<const float*>(smem + (sb - s0) + 4 * kTileBytes + 32768);
    // key validity bits for keys [k0 + 64hh, +64)
    const int ka = k0 + (int)hh * 64 + (int)lane, kb2 = ka + 32;
    bool ok_a = ka < a.Lk, ok_b = kb2 < a.Lk;
    if (a.mask) {
      if (ok_a) ok_a = a.mask[(int64_t)b * a.mask_s0 + (int64_t)ka * a.mask_s1] != 0;
      if (ok_b) ok_b = a.mask[(int64_t)b * a.mask_s0 + (int64_t)kb2 * a.mask_s1] != 0;
    }
    const uint32_t m0 = __ballot_sync(0xffffffffu, ok_a), m1 = __ballot_sync(0xffffffffu, ok_b);
    mbar_wait(bar_in0 + 8 * s, (n >> 1) & 1);
    mbar_wait(bar_sp0 + 8 * s, (n >> 1) & 1);
    tc_fence_after();
    const float lse2 = vec[row], Dq = vec[128 + row];
    float p[64], dp[64];
    tmem_ld64(tmem + s * 256 + lane_base + hh * 64, p, a.scale_log2);
    if (BIAS == 1) {
      add_bias_row64(sBias, row, hh, p);
    } else {
#pragma unroll
      for (int cc = 0; cc < 64; ++cc) p[cc] = fmaf(bias_at(sBias, hh * 64 + cc, row), kLog2e, p[cc]);
    }
    tmem_ld64(tmem + s * 256 + 128 + lane_base + hh * 64, dp, 1.f);
#pragma unroll
    for (int cc = 0; cc < 64; ++cc) {
      const uint32_t bit = (cc < 32 ? (m0 >> cc) : (m1 >> (cc - 32))) & 1u;
      const float pv = bit ? fast_exp2(p[cc] - lse2) : 0.f;
      const float dsv = pv * (dp[cc] - Dq);
      if (a.bias_batched) acc[cc] = dsv;
      else acc[cc] += dsv;
    }
    if (a.bias_batched && qrow < a.Lq) {  // per-batch bias: dbias[b] = dS[b] directly
      float* dst = a.partial + (((int64_t)b * a.H + h) * Lq_pad + qrow) * Lk_pad + k0 + hh * 64;
#pragma unroll
      for (int cc = 0; cc < 64; cc += 4)
        *reinterpret_cast<float4*>(dst + cc) = make_float4(acc[cc], acc[cc + 1], acc[cc + 2], acc[cc + 3]);
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      if (n + 2 < nb) load_stage(s, b + 2, a.bias_batched != 0);
      if (n + 1 < nb) {
        mbar_wait(bar_in0 + 8 * (s ^ 1), ((n + 1) >> 1) & 1);
        tc_fence_after();
        issue_sp(s ^ 1);
      }
    }
  }
  if (!a.bias_batched && qrow < a.Lq) {
    float* dst = a.partial + (((int64_t)c * a.H + h) * Lq_pad + qrow) * Lk_pad + k0 + hh * 64;
#pragma unroll
    for (int cc = 0; cc < 64; cc += 4)
      *reinterpret_cast<float4*>(dst + cc) = make_float4(acc[cc], acc[cc + 1], acc[cc + 2], acc[cc + 3]);
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tmem);
}

template <int DP, int BIAS>
static cudaError_t launch_bwd_bias_t(const BwdBiasLaunch& L, cudaStream_t st) {
  auto kern = bwd_bias_kernel<DP, BIAS>;
  const size_t smem = bwd_bias_smem_bytes(DP);
  cudaError_t e = set_smem_once(kern, smem);
  if (e != cudaSuccess) return e;
  const int nq = (L.args.Lq + 127) / 128, nk = (L.args.Lk + 127) / 128;
  const long long grid = (long long)L.args.H * nq * nk * L.args.nchunks;
  if (grid == 0) return cudaSuccess;
  kern<<<(unsigned)grid, 256, smem, st>>>(L.tm_q, L.tm_k, L.tm_v, L.tm_da, L.tm_b, L.args);
  return cudaGetLastError();
}

cudaError_t launch_bwd_bias_bf16(const BwdBiasLaunch& L, int DP, int bias_mode, cudaStream_t st) {
#define EVO_BIAS_CASE(dp, bm) \
  if (DP == dp && bias_mode == bm) return launch_bwd_bias_t<dp, bm>(L, st);
  EVO_BIAS_CASE(16, 1) EVO_BIAS_CASE(16, 2)
  EVO_BIAS_CASE(32, 1) EVO_BIAS_CASE(32, 2)
  EVO_BIAS_CASE(64, 1) EVO_BIAS_CASE(64, 2)
#undef EVO_BIAS_CASE
  return cudaErrorInvalidValue;
}

// =============================================================================== reduce / convert
// dbias[(b,) h, q, k] = Σ_c partial[c][(b,) h][q][k]   (partials padded to [.][Lq_pad][Lk_pad]).
// Latency-bound (the partials are ~19 MB, ~0.13 MB per SM), so every thread issues the loads of
// ALL its parts at once (NP >= nparts registers, predicated) and sums them in part order
// (deterministic); no grid-stride loop, so the whole reduction is in flight.
//
// q-contiguous destination (end-node bias view): 32 q x 32 k tiles, 256 threads (4 rows each),
// parts read along k (coalesced), transposed through shared memory, written along q.
template <int NP>
__global__ void __launch_bounds__(256) dbias_reduce_kernel(const ReduceArgs a) {
  __shared__ float tile[32][33];
  const int Lq_pad = ((a.Lq + 127) / 128) * 128, Lk_pad = ((a.Lk + 127) / 128) * 128;
  const int64_t plane = (int64_t)a.H * Lq_pad * Lk_pad;
  const int nqt = (a.Lq + 31) / 32, nkt = (a.Lk + 31) / 32;
  int64_t u = blockIdx.x;
  const int kt = (int)(u % nkt); u /= nkt;
  const int qt = (int)(u % nqt); u /= nqt;
  const int h = (int)(u % a.H);
  const int64_t bb = u / a.H;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int k = kt * 32 + tx;
  const float* src = a.partial + ((bb * a.H + h) * Lq_pad + qt * 32 + ty) * (int64_t)Lk_pad + k;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int c0 = 0; c0 < a.nparts; c0 += NP) {  // one round unless nparts > NP
    float v[4][NP];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int c = 0; c < NP; ++c)
        v[i][c] = c0 + c < a.nparts ? __ldg(src + (int64_t)(8 * i) * Lk_pad + (int64_t)(c0 + c) * plane) : 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int c = 0; c < NP; ++c) acc[i] += v[i][c];  // fixed order: deterministic
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) tile[ty + 8 * i][tx] = acc[i];
  __syncthreads();
  if (a.q_fast) {  // destination q-contiguous: lanes along q
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int ki = ty + 8 * i, q = qt * 32 + tx, kk = kt * 32 + ki;
      if (q < a.Lq && kk < a.Lk)
        a.dbias[bb * a.s_b + h * a.s_h + (int64_t)q * a.s_q + (int64_t)kk * a.s_k] = tile[tx][ki];
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int qi = ty + 8 * i, q = qt * 32 + qi;
      if (q < a.Lq && k < a.Lk)
        a.dbias[bb * a.s_b + h * a.s_h + (int64_t)q * a.s_q + (int64_t)k * a.s_k] = tile[qi][tx];
    }
  }
}

// k-contiguous destination (the common case): a thread per 4 consecutive keys of a row, every
// part's float4 in flight before the (fixed-order) sum, one float4 store
template <int NP>
__global__ void __launch_bounds__(256) dbias_reduce_k4_kernel(const ReduceArgs a) {
  const int Lq_pad = ((a.Lq + 127) / 128) * 128, Lk_pad = ((a.Lk + 127) / 128) * 128;
  const int64_t plane = (int64_t)a.H * Lq_pad * Lk_pad;
  const int nk4 = (a.Lk + 3) / 4;
  const int64_t n = a.nb * a.H * (int64_t)a.Lq * nk4;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n) return;
  const int k = (int)(idx % nk4) * 4;
  int64_t t = idx / nk4;
  const int q = (int)(t % a.Lq);
  t /= a.Lq;
  const int h = (int)(t % a.H);
  const int64_t bb = t / a.H;
  const float4* src = reinterpret_cast<const float4*>(
      a.partial + ((bb * a.H + h) * Lq_pad + q) * (int64_t)Lk_pad + k);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int c0 = 0; c0 < a.nparts; c0 += NP) {  // one round unless nparts > NP
    float4 v[NP];
#pragma unroll
    for (int c = 0; c < NP; ++c)
      v[c] = c0 + c < a.nparts ? __ldg(src + (int64_t)(c0 + c) * (plane / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int c = 0; c < NP; ++c) { acc.x += v[c].x; acc.y += v[c].y; acc.z += v[c].z; acc.w += v[c].w; }
  }
  float* dst = a.dbias + bb * a.s_b + h * a.s_h + (int64_t)q * a.s_q + k;
  if (k + 3 < a.Lk && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
    *reinterpret_cast<float4*>(dst) = acc;
  } else {
    const float e4[4] = {acc.x, acc.y, acc.z, acc.w};
    for (int e = 0; e < 4 && k + e < a.Lk; ++e) dst[e] = e4[e];
  }
}

cudaError_t launch_dbias_reduce(const ReduceArgs& a, cudaStream_t st) {
  if (!a.q_fast && a.s_k == 1) {
    const int64_t n = a.nb * a.H * (int64_t)a.Lq * ((a.Lk + 3) / 4);
    if (n == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((n + 255) / 256);
    if (a.nparts <= 8) dbias_reduce_k4_kernel<8><<<blocks, 256, 0, st>>>(a);
    else if (a.nparts <= 16) dbias_reduce_k4_kernel<16><<<blocks, 256, 0, st>>>(a);
    else dbias_reduce_k4_kernel<32><<<blocks, 256, 0, st>>>(a);
    return cudaGetLastError();
  }
  const int64_t blocks = a.nb * a.H * (int64_t)((a.Lq + 31) / 32) * ((a.Lk + 31) / 32);
  if (blocks == 0) return cudaSuccess;
  if (a.nparts <= 8) dbias_reduce_kernel<8><<<(unsigned)blocks, 256, 0, st>>>(a);
  else dbias_reduce_kernel<16><<<(unsigned)blocks, 256, 0, st>>>(a);  // 4 rows x 16 in flight
  return cudaGetLastError();
}

// dq = bf16(scale · Σ_p part_p): 8 elements per thread (adjacent threads on adjacent 32-byte
// chunks: coalesced), rows visited in the order of the smaller of the (h, l) strides of dq (the
// parts use the same order, see ws_layout); 32-bit index math (rows < 2^31 checked by the launcher)
template <int DP>
__global__ void __launch_bounds__(256) dq_convert_kernel(const ConvertArgs a) {
  constexpr int ND = DP / 8;  // 8-element chunks per padded row
  const int nd = (a.D + 7) / 8;
  const uint32_t rows = (uint32_t)a.B * a.H * a.Lq;
  const uint32_t n8 = rows * (uint32_t)nd;
  const bool hfast = a.q_sh < a.q_sl;
  (void)ND;
  const uint64_t pol = l2_policy_evict_first();
  for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n8; idx += gridDim.x * blockDim.x) {
    uint32_t r = fdiv(idx, a.fd_nd), r2;
    const uint32_t d0 = (idx - r * (uint32_t)nd) * 8;
    uint32_t h, q;
    if (hfast) {
      r2 = fdiv(r, a.fd_H); h = r - r2 * (uint32_t)a.H; r = r2;
      r2 = fdiv(r, a.fd_Lq); q = r - r2 * (uint32_t)a.Lq; r = r2;
    } else {
      r2 = fdiv(r, a.fd_Lq); q = r - r2 * (uint32_t)a.Lq; r = r2;
      r2 = fdiv(r, a.fd_H); h = r - r2 * (uint32_t)a.H; r = r2;
    }
    const int64_t b = r;
    // last read of the fp32 accumulator / parts: evict_first, so these lines (left at
    // evict_last by bwd_pre's zero-fill and the reduce-adds) do not crowd the next kernels out
    const float* src = a.acc + b * a.p_sb + (int64_t)h * a.p_sh + (int64_t)q * a.p_sl + d0;
    float4 x = ldg_f4_hint(src, pol);
    float4 y = ldg_f4_hint(src + 4, pol);
    for (int p = 1; p < a.nparts; ++p) {  // parts summed in key-tile order (deterministic)
      const float4 x2 = ldg_f4_hint(src + p * a.part_stride, pol);
      const float4 y2 = ldg_f4_hint(src + p * a.part_stride + 4, pol);
      x.x += x2.x; x.y += x2.y; x.z += x2.z; x.w += x2.w;
      y.x += y2.x; y.y += y2.y; y.z += y2.z; y.w += y2.w;
    }
    uint4 st;
    st.x = pack_bf16(x.x * a.scale, x.y * a.scale);
    st.y = pack_bf16(x.z * a.scale, x.w * a.scale);
    st.z = pack_bf16(y.x * a.scale, y.y * a.scale);
    st.w = pack_bf16(y.z * a.scale, y.w * a.scale);
    *reinterpret_cast<uint4*>(a.dq + b * a.q_sb + (int64_t)h * a.q_sh + (int64_t)q * a.q_sl + d0) = st;
  }
}

cudaError_t launch_dq_convert(const ConvertArgs& a, cudaStream_t st) {
  const int64_t n8 = (int64_t)a.B * a.H * a.Lq * ((a.D + 7) / 8);
  if (n8 == 0) return cudaSuccess;
  if (n8 >= (int64_t)1 << 31) return cudaErrorInvalidValue;
  const int64_t blocks = (n8 + 255) / 256;
  const unsigned g = (unsigned)(blocks < 148 * 16 ? blocks : 148 * 16);
  ConvertArgs v = a;
  v.fd_nd = make_fastdiv((uint32_t)((a.D + 7) / 8));
  v.fd_H = make_fastdiv((uint32_t)a.H);
  v.fd_Lq = make_fastdiv((uint32_t)a.Lq);
  if (a.D <= 16) dq_convert_kernel<16><<<g, 256, 0, st>>>(v);
  else if (a.D <= 32) dq_convert_kernel<32><<<g, 256, 0, st>>>(v);
  else dq_convert_kernel<64><<<g, 256, 0, st>>>(v);
  return cudaGetLastError();
}

}  // namespace evo
