// evo_fwd.cu — bf16 forward of Evoformer gated attention with pair bias on sm_100a.
//
// PAPER.md L294 (§3.3.1 MHA): pair bias added to the logits before the softmax, all of MHA
// fused, "based on FlashAttention".  One CTA computes one (b, h, 128-query tile):
//   TMA  Q tile, K/V tiles (2-stage ring), bias tile (SW128)            -> shared memory
//   tcgen05.mma  S = Q·Kᵀ  (M=128, N=128, K=DP)                          -> TMEM cols [0,128)
//   8 warps: tcgen05.ld S, s·scale·log2e + bias·log2e, hard mask, online softmax (exp2),
//            O rescale in TMEM, P (bf16) -> SW128 shared memory
//   tcgen05.mma  O += P·V  (M=128, N=DP, K=128)                          -> TMEM cols [128,128+DP)
//   epilogue: O / l · sigmoid(g) -> o (bf16), lse = (m + log2 l)·ln2 (fp32)
// Warp w owns TMEM lane quadrant (w % 4) (query rows 32(w%4)..+31) and key-column half (w / 4).
#include "evo_kernels.cuh"

namespace evo {

template <int DP, int BIAS>
__global__ void __launch_bounds__(256, 2) fwd_bf16_kernel(const __grid_constant__ CUtensorMap tm_q,
                                                           const __grid_constant__ CUtensorMap tm_k,
                                                           const __grid_constant__ CUtensorMap tm_v,
                                                           const __grid_constant__ CUtensorMap tm_b,
                                                           const FwdArgs a) {
  constexpr uint32_t kRowBytes = DP * 2;
  constexpr uint32_t kTileBytes = 128 * kRowBytes;  // one 128-row Q/K/V tile
  constexpr uint32_t kSw = DP == 64 ? kSw128 : (DP == 32 ? kSw64 : kSw32);
  constexpr uint32_t kHalfCols = DP / 2;            // O columns per warp half

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;  // dynamic smem base is 1024-aligned (no static smem); checked:
  if (smem_u32(smem) & 1023u) __trap();
  const uint32_t sQ = smem_u32(smem);
  const uint32_t sK = sQ + kTileBytes;              // 2 stages
  const uint32_t sV = sK + 2 * kTileBytes;          // 2 stages
  const uint32_t sB = sV + 2 * kTileBytes;          // bias tile, 2 x 16 KB regions
  const uint32_t sP = sB + 32768;                   // P tile, 2 x 16 KB regions
  uint32_t* maskw = reinterpret_cast<uint32_t*>(smem + 5 * kTileBytes + 65536);  // kMaxMaskWords
  float* red_m = reinterpret_cast<float*>(maskw + kMaxMaskWords);  // [2][128]
  float* red_l = red_m + 256;                                       // [2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(red_l + 256);        // 8 barriers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);
  const uint32_t bar_q = smem_u32(&bars[0]);
  const uint32_t bar_kv0 = smem_u32(&bars[1]);  // +8 for stage 1
  const uint32_t bar_bias = smem_u32(&bars[3]);
  const uint32_t bar_s = smem_u32(&bars[4]);
  const uint32_t bar_o = smem_u32(&bars[5]);

  const uint32_t tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const uint32_t qd = w & 3, hh = w >> 2, row = qd * 32 + lane;
  const int nq = (a.Lq + 127) >> 7, nk = (a.Lk + 127) >> 7;
  const int unit = blockIdx.x;
  const int qt = unit % nq;
  const int bh = unit / nq;
  const int h = bh % a.H;
  const int b = bh / a.H;
  const int q0 = qt * 128;

  if (w == 0) tmem_alloc<256>(smem_u32(tmem_slot));
  if (tid == 0) {
    mbar_init(bar_q, 1);
    mbar_init(bar_kv0, 1);
    mbar_init(bar_kv0 + 8, 1);
    mbar_init(bar_bias, 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_o, 1);
    fence_barrier_init();
  }
  // key-validity words: bit k%32 of word k/32 = (k < Lk) && mask[b,k] != 0
  for (int kb = (int)w * 32; kb < nk * 128; kb += 256) {
    const int k = kb + (int)lane;
    bool keep = k < a.Lk;
    if (keep && a.mask) keep = a.mask[(int64_t)b * a.mask_s0 + (int64_t)k * a.mask_s1] != 0;
    const uint32_t word = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) maskw[kb >> 5] = word;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + 128;
  const uint32_t lane_base = (qd * 32) << 16;
  const int bcoord = a.bias_batched ? b : 0;

  constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, 0, 0);
  constexpr uint32_t idesc_o = make_idesc_bf16(128, DP, 0, 1);

  if (tid == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    if (BIAS) tma_prefetch_desc(&tm_b);
    mbar_arrive_expect_tx(bar_q, kTileBytes);
    tma_load_4d(sQ, &tm_q, bar_q, 0, q0, h, b);
    for (int s = 0; s < 2 && s < nk; ++s) {
      mbar_arrive_expect_tx(bar_kv0 + 8 * s, 2 * kTileBytes);
      tma_load_4d(sK + s * kTileBytes, &tm_k, bar_kv0 + 8 * s, 0, s * 128, h, b);
      tma_load_4d(sV + s * kTileBytes, &tm_v, bar_kv0 + 8 * s, 0, s * 128, h, b);
    }
    if (BIAS) {
      mbar_arrive_expect_tx(bar_bias, 32768);
      for (int r = 0; r < 2; ++r) {
        if (BIAS == 1) tma_load_4d(sB + r * 16384, &tm_b, bar_bias, r * 64, q0, h, bcoord);
        else tma_load_4d(sB + r * 16384, &tm_b, bar_bias, q0 + r * 64, 0, h, bcoord);
      }
    }
    mbar_wait(bar_q, 0);
    mbar_wait(bar_kv0, 0);
    tc_fence_after();
#pragma unroll
    for (int t = 0; t < DP / 16; ++t)
      umma_bf16(tS, make_sdesc(sQ + t * 32, 16, 8 * kRowBytes, kSw),
                make_sdesc(sK + t * 32, 16, 8 * kRowBytes, kSw), idesc_s, t > 0);
    umma_commit(bar_s);
  }

  float m_run = -INFINITY, l_run = 0.f;
  for (int j = 0; j < nk; ++j) {
    // ---- scores for keys [128j, 128j+128): this thread's row, columns [64hh, 64hh+64)
    mbar_wait(bar_s, j & 1);
    tc_fence_after();
    float s2[64];
    {
      uint32_t r[32];
      tmem_ld32(tS + lane_base + hh * 64, r);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 32; ++c) s2[c] = __uint_as_float(r[c]) * a.scale_log2;
      tmem_ld32(tS + lane_base + hh * 64 + 32, r);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 32; ++c) s2[32 + c] = __uint_as_float(r[c]) * a.scale_log2;
    }
    if (BIAS) {
      mbar_wait(bar_bias, j & 1);
      if (BIAS == 1) {  // bias[q, k] with k contiguous: this row, region hh
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 v = ld_shared_v4(sB + hh * 16384 + swz_offset(row, c, 128));
          const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            s2[c * 8 + 2 * e] = fmaf(bf16_lo(u[e]), kLog2e, s2[c * 8 + 2 * e]);
            s2[c * 8 + 2 * e + 1] = fmaf(bf16_hi(u[e]), kLog2e, s2[c * 8 + 2 * e + 1]);
          }
        }
      } else {  // bias stored [k][q] (q contiguous): column `row` of rows k
        const uint32_t base = sB + (row >> 6) * 16384 + (row & 7) * 2;
        const uint32_t qc = (row & 63) >> 3;
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          const uint32_t k = hh * 64 + c;
          const float bv = bf16_to_f(ld_shared_u16(base + k * 128 + ((qc ^ (k & 7)) << 4)));
          s2[c] = fmaf(bv, kLog2e, s2[c]);
        }
      }
    }
    // hard mask (also kills padded keys k >= Lk)
    float mx = -INFINITY;
    {
      const uint32_t w0 = maskw[(j * 128 + hh * 64) >> 5];
      const uint32_t w1 = maskw[((j * 128 + hh * 64) >> 5) + 1];
#pragma unroll
      for (int c = 0; c < 64; ++c) {
        const uint32_t bit = (c < 32 ? (w0 >> c) : (w1 >> (c - 32))) & 1u;
        s2[c] = bit ? s2[c] : -INFINITY;
        mx = fmaxf(mx, s2[c]);
      }
    }
    red_m[hh * 128 + row] = mx;
    tc_fence_before();
    __syncthreads();  // S_j and bias tile j fully consumed; row maxima exchanged
    mx = fmaxf(red_m[row], red_m[128 + row]);
    if (BIAS && tid == 0 && j + 1 < nk) {
      mbar_arrive_expect_tx(bar_bias, 32768);
      for (int r = 0; r < 2; ++r) {
        if (BIAS == 1)
          tma_load_4d(sB + r * 16384, &tm_b, bar_bias, (j + 1) * 128 + r * 64, q0, h, bcoord);
        else
          tma_load_4d(sB + r * 16384, &tm_b, bar_bias, q0 + r * 64, (j + 1) * 128, h, bcoord);
      }
    }
    const float m_new = fmaxf(m_run, mx);
    const float m_use = m_new == -INFINITY ? 0.f : m_new;
    const float alpha = fast_exp2(m_run - m_use);  // m_run = -inf -> 0
    float lsum = 0.f;
#pragma unroll
    for (int c = 0; c < 64; ++c) {
      s2[c] = fast_exp2(s2[c] - m_use);
      lsum += s2[c];
    }
    l_run = l_run * alpha + lsum;
    m_run = m_new;
    if (j > 0) {
      // PV_{j-1} must be done before P is overwritten and O is rescaled
      mbar_wait(bar_o, (j - 1) & 1);
      tc_fence_after();
      if (tid == 0 && j + 1 < nk && j + 1 >= 2) {
        const int s = (j + 1) & 1;
        mbar_arrive_expect_tx(bar_kv0 + 8 * s, 2 * kTileBytes);
        tma_load_4d(sK + s * kTileBytes, &tm_k, bar_kv0 + 8 * s, 0, (j + 1) * 128, h, b);
        tma_load_4d(sV + s * kTileBytes, &tm_v, bar_kv0 + 8 * s, 0, (j + 1) * 128, h, b);
      }
      // (tcgen05.ld/st are warp-collective: the rescale is done by every lane, even at alpha=1)
#pragma unroll
      for (int c0 = 0; c0 < (int)kHalfCols; c0 += 8) {
        uint32_t r[8];
        tmem_ld8(tO + lane_base + hh * kHalfCols + c0, r);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 8; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
        tmem_st8(tO + lane_base + hh * kHalfCols + c0, r);
      }
      tmem_wait_st();
    }
    // P (bf16) -> shared memory, K-major SW128: region hh, row `row`
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      st_shared_v4(sP + hh * 16384 + swz_offset(row, c, 128), pack_bf16(s2[8 * c], s2[8 * c + 1]),
                   pack_bf16(s2[8 * c + 2], s2[8 * c + 3]), pack_bf16(s2[8 * c + 4], s2[8 * c + 5]),
                   pack_bf16(s2[8 * c + 6], s2[8 * c + 7]));
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t vbase = sV + (j & 1) * kTileBytes;
#pragma unroll
      for (int t = 0; t < 8; ++t)
        umma_bf16(tO, make_sdesc(sP + (t >> 2) * 16384 + (t & 3) * 32, 16, 1024, kSw128),
                  make_sdesc(vbase + t * 16 * kRowBytes, 16384, 8 * kRowBytes, kSw), idesc_o,
                  (j > 0 || t > 0) ? 1u : 0u);
      umma_commit(bar_o);
      if (j + 1 < nk) {
        const int s = (j + 1) & 1;
        mbar_wait(bar_kv0 + 8 * s, ((j + 1) >> 1) & 1);
        tc_fence_after();
        const uint32_t kbase = sK + s * kTileBytes;
#pragma unroll
        for (int t = 0; t < DP / 16; ++t)
          umma_bf16(tS, make_sdesc(sQ + t * 32, 16, 8 * kRowBytes, kSw),
                    make_sdesc(kbase + t * 32, 16, 8 * kRowBytes, kSw), idesc_s, t > 0);
        umma_commit(bar_s);
      }
    }
  }

  // ---- epilogue
  red_l[hh * 128 + row] = l_run;
  mbar_wait(bar_o, (nk - 1) & 1);  // nk >= 1 (Lk == 0 never launches this kernel)
  tc_fence_after();
  __syncthreads();
  const float l_tot = red_l[row] + red_l[128 + row];
  const float inv = l_tot > 0.f ? 1.f / l_tot : 0.f;
  const int q = q0 + (int)row;
  const bool qvalid = q < a.Lq;
  const int64_t orow = (int64_t)b * a.o_sb + (int64_t)h * a.o_sh + (int64_t)q * a.o_sl;
  const int64_t grow = (int64_t)b * a.g_sb + (int64_t)h * a.g_sh + (int64_t)q * a.g_sl;
#pragma unroll
  for (int c0 = 0; c0 < (int)kHalfCols; c0 += 8) {
    const int d0 = hh * kHalfCols + c0;
    uint32_t r[8];
    tmem_ld8(tO + lane_base + d0, r);  // warp-collective
    tmem_wait_ld();
    if (qvalid && d0 < a.D) {
      float gv[8];
      if (a.g) {
        const uint4 gg = *reinterpret_cast<const uint4*>(a.g + grow + d0);
        const uint32_t u[4] = {gg.x, gg.y, gg.z, gg.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          gv[2 * e] = 1.f / (1.f + __expf(-bf16_lo(u[e])));
          gv[2 * e + 1] = 1.f / (1.f + __expf(-bf16_hi(u[e])));
        }
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) gv[e] = 1.f;
      }
      float ov[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) ov[e] = __uint_as_float(r[e]) * inv * gv[e];
      uint4 st;
      st.x = pack_bf16(ov[0], ov[1]);
      st.y = pack_bf16(ov[2], ov[3]);
      st.z = pack_bf16(ov[4], ov[5]);
      st.w = pack_bf16(ov[6], ov[7]);
      *reinterpret_cast<uint4*>(a.o + orow + d0) = st;
    }
  }
  if (qvalid && hh == 0) {
    const float m_use = m_run == -INFINITY ? 0.f : m_run;
    a.lse[((int64_t)b * a.H + h) * a.Lq + q] =
        l_tot > 0.f ? (m_use + __log2f(l_tot)) * kLn2 : -INFINITY;
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<256>(tmem);
}

template <int DP, int BIAS>
static cudaError_t launch_fwd_t(const FwdLaunch& L, cudaStream_t st) {
  auto kern = fwd_bf16_kernel<DP, BIAS>;
  const size_t smem = fwd_smem_bytes(DP);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int nq = (L.args.Lq + 127) / 128;
  const long long grid = (long long)L.args.B * L.args.H * nq;
  if (grid == 0) return cudaSuccess;
  kern<<<(unsigned)grid, 256, smem, st>>>(L.tm_q, L.tm_k, L.tm_v, L.tm_b, L.args);
  return cudaGetLastError();
}

cudaError_t launch_fwd_bf16(const FwdLaunch& L, int DP, int bias_mode, cudaStream_t st) {
#define EVO_FWD_CASE(dp, bm) \
  if (DP == dp && bias_mode == bm) return launch_fwd_t<dp, bm>(L, st);
  EVO_FWD_CASE(16, 0) EVO_FWD_CASE(16, 1) EVO_FWD_CASE(16, 2)
  EVO_FWD_CASE(32, 0) EVO_FWD_CASE(32, 1) EVO_FWD_CASE(32, 2)
  EVO_FWD_CASE(64, 0) EVO_FWD_CASE(64, 1) EVO_FWD_CASE(64, 2)
#undef EVO_FWD_CASE
  return cudaErrorInvalidValue;
}

}  // namespace evo
