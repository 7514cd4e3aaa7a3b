// evo_fwd_pp.cu — ping-pong persistent bf16 forward (sm_100a): two softmax warpgroups, each
// walking its own sequence of (b, h, 128-query tile) units, with per-group MMA-issuer and TMA
// warps, so that the Sᵀ MMA of chunk c+1 runs while the group does the softmax of chunk c and
// neither group's hand-offs stall the other.
//
// Same operation as evo_fwd_occ.cu (the pair bias added to the logits before
// the softmax, all of MHA fused, FlashAttention-style online softmax; gate epilogue, AF2 Alg. 7
// l.4/6).  Per group g, unit u, 64-key chunk c:
//   TMA:      Q, G tiles of u (once per unit, 2 buffers);  K_c, V_c, bias_c (ring)
//   MMA:      S[c%2] = Q·K_cᵀ (SS, M = 128 queries, N = 64 keys)         -> TMEM slot c%2
//   softmax:  x = S·scale + bias (fp32), hard mask, chunk max, lazy rescale of O (threshold 8
//             in log2 units; PV(c-1) is waited first), p = exp2(x·log2e − m), P (bf16) over the
//             consumed S columns
//   MMA:      O += P·V_c (TS form, A = P from TMEM)
//   epilogue: o = O/l ⊙ σ(g) (bf16), lse = m + log l (fp32)
// TMEM (512 cols): group g at 256·g: S slot 0 [0,64), slot 1 [64,128), O [128, 128+DP)
#include "evo_kernels.cuh"

namespace evo {

template <int DP, int BIAS>
struct PpCfg {
  static constexpr uint32_t kRowBytes = DP * 2;
  static constexpr uint32_t kQT = 128 * kRowBytes;           // Q or G tile
  static constexpr uint32_t kKV = 64 * kRowBytes;            // K or V chunk
  static constexpr uint32_t kBias = BIAS ? 16384u : 0u;      // 128 x 64 bf16
  static constexpr uint32_t kStage = 2 * kKV + kBias;
  static constexpr int kNSt = BIAS ? 2 : 4;
  // per group: Q/G x 2 buffers | ring
  static constexpr uint32_t kGroup = 4 * kQT + kNSt * kStage;
  static constexpr uint32_t oMask = 2 * kGroup + 512;          // per group: 2 x kMaxMaskWords
  static constexpr uint32_t kSmem = oMask + 2 * 2 * kMaxMaskWords * 4;
};

template <int DP, int BIAS>
__global__ void __launch_bounds__(384, 1)
    fwd_pp_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_g,
                  const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                  const __grid_constant__ CUtensorMap tm_b, const FwdArgs a) {
  using C = PpCfg<DP, BIAS>;
  constexpr uint32_t kSw = DP == 64 ? kSw128 : (DP == 32 ? kSw64 : kSw32);
  constexpr int NST = C::kNSt;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t s0 = smem_u32(smem);
  if (s0 & 1023u) __trap();
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  // roles: warps 0-3 group 0, 4-7 group 1 (softmax); 8/10 MMA issuer g0/g1; 9/11 TMA g0/g1
  const int g = w < 8 ? (w >> 2) : ((w - 8) >> 1);
  const uint32_t gs = s0 + g * C::kGroup;                    // this group's smem
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * C::kGroup) + g * 24;
  auto bar = [&](int i) { return smem_u32(&bars[i]); };
  // per-group barrier indices
  const uint32_t b_q = bar(0);        // +8·ub: Q/G of a unit landed (tx)
  const uint32_t b_qfree = bar(2);    // +8·ub: the unit's epilogue read G (4 warps)
  const uint32_t b_kv = bar(4);       // +8·st: K/V/bias chunk landed (tx), NST <= 4
  const uint32_t b_kvfree = bar(8);   // +8·st: PV of the chunk done (commit)
  const uint32_t b_s = bar(12);       // +8·slot: Sᵀ of a chunk in TMEM (commit)
  const uint32_t b_p = bar(14);       // P of a chunk in TMEM (4 warps)
  const uint32_t b_pv = bar(15);      // PV of a chunk done (commit)
  const uint32_t b_oempty = bar(16);  // the unit's epilogue pulled O (4 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + 2 * C::kGroup + 2 * 24 * 8);

  const int nq = (a.Lq + 127) >> 7, nc = (a.Lk + 63) >> 6;
  const int64_t U = (int64_t)a.B * a.H * nq;
  const int64_t u_first = 2 * (int64_t)blockIdx.x + g, u_step = 2 * (int64_t)gridDim.x;

  if (w == 0) tmem_alloc<512>(smem_u32(tmem_slot));
  if (tid == 0) {
    for (int gg = 0; gg < 2; ++gg) {
      uint64_t* bb = reinterpret_cast<uint64_t*>(smem + 2 * C::kGroup) + gg * 24;
      for (int i = 0; i < 2; ++i) { mbar_init(smem_u32(&bb[0 + i]), 1); mbar_init(smem_u32(&bb[2 + i]), 4); }
      for (int i = 0; i < 4; ++i) { mbar_init(smem_u32(&bb[4 + i]), 1); mbar_init(smem_u32(&bb[8 + i]), 1); }
      for (int i = 0; i < 2; ++i) mbar_init(smem_u32(&bb[12 + i]), 1);
      mbar_init(smem_u32(&bb[14]), 4);
      mbar_init(smem_u32(&bb[15]), 1);
      mbar_init(smem_u32(&bb[16]), 4);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot + (uint32_t)g * 256;
  const uint32_t tO = tmem + 128;

  auto unit_coords = [&](int64_t u, int& b, int& h, int& qt) {
    qt = (int)(u % nq);
    const int64_t bh = u / nq;
    h = (int)(bh % a.H);
    b = (int)(bh / a.H);
  };

  if (w == 9 || w == 11) {
    // ------------------------------------------------------------------ TMA producer (group g)
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      if (a.g) tma_prefetch_desc(&tm_g);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      if (BIAS) tma_prefetch_desc(&tm_b);
      int64_t ci = 0;  // global chunk counter of this group
      int k = 0;       // unit counter
      for (int64_t u = u_first; u < U; u += u_step, ++k) {
        int b, h, qt;
        unit_coords(u, b, h, qt);
        const int ub = k & 1;
        if (k >= 2) mbar_wait(b_qfree + 8 * ub, ((k - 2) >> 1) & 1);
        const uint32_t qb = gs + ub * 2 * C::kQT;
        mbar_arrive_expect_tx(b_q + 8 * ub, (a.g ? 2 : 1) * C::kQT);
        tma_load_4d(qb, &tm_q, b_q + 8 * ub, 0, qt * 128, h, b);
        if (a.g) tma_load_4d(qb + C::kQT, &tm_g, b_q + 8 * ub, 0, qt * 128, h, b);
        const int bc = a.bias_batched ? b : 0;
        for (int c = 0; c < nc; ++c, ++ci) {
          const int st = (int)(ci % NST);
          if (ci >= NST) mbar_wait(b_kvfree + 8 * st, ((ci - NST) / NST) & 1);
          const uint32_t sb = gs + 4 * C::kQT + st * C::kStage;
          const uint32_t bb = b_kv + 8 * st;
          mbar_arrive_expect_tx(bb, C::kStage);
          tma_load_4d(sb, &tm_k, bb, 0, c * 64, h, b);
          tma_load_4d(sb + C::kKV, &tm_v, bb, 0, c * 64, h, b);
          if (BIAS == 1) tma_load_4d(sb + 2 * C::kKV, &tm_b, bb, c * 64, qt * 128, h, bc);
          if (BIAS == 2) {
            tma_load_4d(sb + 2 * C::kKV, &tm_b, bb, qt * 128, c * 64, h, bc);
            tma_load_4d(sb + 2 * C::kKV + 8192, &tm_b, bb, qt * 128 + 64, c * 64, h, bc);
          }
        }
      }
    }
  } else if (w == 8 || w == 10) {
    // ------------------------------------------------------------------ MMA issuer (group g)
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, 0, 0);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, DP, 0, 1);
      int64_t ci = 0;  // global chunk counter
      int k = 0;
      for (int64_t u = u_first; u < U; u += u_step, ++k) {
        const int ub = k & 1;
        mbar_wait(b_q + 8 * ub, (k >> 1) & 1);
        const uint32_t qb = gs + ub * 2 * C::kQT;
        for (int c = 0; c <= nc; ++c) {
          if (c < nc) {  // Sᵀ(c) into slot (ci + c) % 2
            const int64_t cc = ci + c;
            const int st = (int)(cc % NST), slot = (int)(cc & 1);
            mbar_wait(b_kv + 8 * st, (cc / NST) & 1);
            tc_fence_after();
            const uint32_t kb = gs + 4 * C::kQT + st * C::kStage;
#pragma unroll
            for (int kk = 0; kk < DP / 16; ++kk)
              umma_bf16(tmem + slot * 64, make_sdesc(qb + kk * 32, 16, 8 * C::kRowBytes, kSw),
                        make_sdesc(kb + kk * 32, 16, 8 * C::kRowBytes, kSw), idesc_s, kk > 0);
            umma_commit(b_s + 8 * slot);
          }
          if (c > 0) {  // PV(c-1): O += P·V
            const int64_t cc = ci + c - 1;
            const int st = (int)(cc % NST), slot = (int)(cc & 1);
            mbar_wait(b_p, cc & 1);
            if (c == 1 && k > 0) mbar_wait(b_oempty, (k - 1) & 1);  // previous unit drained O
            tc_fence_after();
            const uint32_t vb = gs + 4 * C::kQT + st * C::kStage + C::kKV;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              umma_bf16_ts(tO, tmem + slot * 64 + kk * 8,
                           make_sdesc(vb + kk * 16 * C::kRowBytes, 16384, 8 * C::kRowBytes, kSw),
                           idesc_o, (c > 1 || kk > 0) ? 1u : 0u);
            umma_commit(b_pv);
            umma_commit(b_kvfree + 8 * st);
          }
        }
        ci += nc;
      }
    }
  } else {
    // ------------------------------------------------------------------ softmax group g
    const int qd = w & 3;
    const int row = qd * 32 + lane;  // query row within the tile = TMEM lane
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    const uint64_t scale2 = f2_pack(a.scale, a.scale);
    const uint64_t log2e2 = f2_pack(kLog2e, kLog2e);
    int64_t ci = 0;
    int k = 0;
    for (int64_t u = u_first; u < U; u += u_step, ++k) {
      int b, h, qt;
      unit_coords(u, b, h, qt);
      const int ub = k & 1;
      const int q = qt * 128 + row;
      const bool all_kept = a.mask == nullptr && (a.Lk & 63) == 0;
      // hard-mask bits of this unit's batch row, once per unit: one coalesced pass over the mask
      // row into 32-key words in shared memory (double-buffered by unit parity), instead of a
      // dependent global load per chunk
      uint32_t* smask = reinterpret_cast<uint32_t*>(smem + C::oMask) + (g * 2 + ub) * kMaxMaskWords;
      if (!all_kept) {
        const int nwords = nc * 2;
        for (int wd = qd; wd < nwords; wd += 4) {
          const int kk = wd * 32 + lane;
          const uint32_t keep = kk < a.Lk ? (a.mask ? (uint32_t)a.mask[(int64_t)b * a.mask_s0 + (int64_t)kk * a.mask_s1] : 1u) : 0u;
          const uint32_t word = __ballot_sync(0xffffffffu, keep != 0);
          if (lane == 0) smask[wd] = word;
        }
        named_bar_sync(1 + g, 128);
      }
      float m_ref = -INFINITY, l_run = 0.f;
      for (int c = 0; c < nc; ++c) {
        const int64_t cc = ci + c;
        const int st = (int)(cc % NST), slot = (int)(cc & 1);
        const uint32_t sb = gs + 4 * C::kQT + st * C::kStage;
        uint32_t mw0 = ~0u, mw1 = ~0u;
        if (!all_kept) { mw0 = smask[2 * c]; mw1 = smask[2 * c + 1]; }
        mbar_wait(b_s + 8 * slot, (cc >> 1) & 1);
        tc_fence_after();
        const uint32_t tS = tmem + slot * 64;
        float x[64];
        {
          uint32_t r0[32], r1[32];
          tmem_ld32(tS + lane_base, r0);
          tmem_ld32(tS + lane_base + 32, r1);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            x[i] = __uint_as_float(r0[i]);
            x[32 + i] = __uint_as_float(r1[i]);
          }
        }
        if (BIAS) mbar_wait(b_kv + 8 * st, (cc / NST) & 1);  // bias chunk visible
        const uint32_t bb = sb + 2 * C::kKV;
        if (BIAS == 1) {
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) {
            const uint4 v = ld_shared_v4(bb + swz_offset(row, c8, 128));
            const uint32_t u4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int kx = c8 * 8 + 2 * i;
              f2_unpack(f2_fma(f2_pack(x[kx], x[kx + 1]), scale2, bf16x2_to_f2(u4[i])), x[kx], x[kx + 1]);
            }
          }
        } else if (BIAS == 2) {
          const uint32_t base = bb + (row >> 6) * 8192 + (row & 7) * 2;
          const uint32_t qc = (row & 63) >> 3;
#pragma unroll
          for (int kx = 0; kx < 64; ++kx) {
            const float bv = bf16_to_f(ld_shared_u16(base + kx * 128 + ((qc ^ (kx & 7)) << 4)));
            x[kx] = fmaf(x[kx], a.scale, bv);
          }
        } else {
#pragma unroll
          for (int kx = 0; kx < 64; kx += 2) f2_unpack(f2_mul(f2_pack(x[kx], x[kx + 1]), scale2), x[kx], x[kx + 1]);
        }
        if ((mw0 & mw1) != ~0u) {
#pragma unroll
          for (int kx = 0; kx < 64; ++kx)
            x[kx] = (((kx < 32 ? mw0 : mw1) >> (kx & 31)) & 1u) ? x[kx] : -INFINITY;
        }
        float m4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) m4[i] = fmaxf(x[i], x[4 + i]);
#pragma unroll
        for (int kx = 8; kx < 64; kx += 8)
#pragma unroll
          for (int i = 0; i < 4; ++i) m4[i] = fmax3(m4[i], x[kx + i], x[kx + 4 + i]);
        const float mx = fmax3(fmaxf(m4[0], m4[1]), m4[2], m4[3]);
        const float m_new = fmaxf(m_ref, mx);
        if (c == 0) {
          m_ref = m_new;
        } else {
          // PV(c-1) must be complete before O is touched (waited every chunk, in order)
          mbar_wait(b_pv, (cc - 1) & 1);
          const bool need = (m_new - m_ref) * kLog2e > 8.f;
          if (__any_sync(0xffffffffu, need)) {
            tc_fence_after();
            const float alpha = need ? fast_exp2((m_ref - m_new) * kLog2e) : 1.f;
#pragma unroll
            for (int c0 = 0; c0 < DP; c0 += 8) {
              uint32_t r[8];
              tmem_ld8(tO + lane_base + c0, r);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 8; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
              tmem_st8(tO + lane_base + c0, r);
            }
            tmem_wait_st();
            l_run *= alpha;
            if (need) m_ref = m_new;
          }
        }
        const float negm = m_ref == -INFINITY ? 0.f : -m_ref * kLog2e;
        const uint64_t negm2 = f2_pack(negm, negm);
        uint64_t ls[4] = {0, 0, 0, 0};
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          float y0, y1;
          f2_unpack(f2_fma(f2_pack(x[2 * i], x[2 * i + 1]), log2e2, negm2), y0, y1);
          const float p0 = fast_exp2(y0), p1 = fast_exp2(y1);
          ls[i & 3] = f2_add(ls[i & 3], f2_pack(p0, p1));
          pk[i] = pack_bf16(p0, p1);
        }
        {
          float l0, l1;
          f2_unpack(f2_add(f2_add(ls[0], ls[1]), f2_add(ls[2], ls[3])), l0, l1);
          l_run += l0 + l1;
        }
        tmem_st32(tS + lane_base, pk);  // P over the consumed S columns [0, 32)
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(b_p);
      }
      // ---- epilogue: the unit's last PV, then o = O/l ⊙ σ(g), lse
      mbar_wait(b_pv, (ci + nc - 1) & 1);
      tc_fence_after();
      uint32_t ov[DP];
      if constexpr (DP == 16) {
        tmem_ld16(tO + lane_base, *reinterpret_cast<uint32_t(*)[16]>(ov));
      } else {
#pragma unroll
        for (int c0 = 0; c0 < DP; c0 += 32)
          tmem_ld32(tO + lane_base + c0, *reinterpret_cast<uint32_t(*)[32]>(ov + c0));
      }
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(b_oempty);
      const uint32_t gb = gs + ub * 2 * C::kQT + C::kQT;  // G tile (same swizzle as Q)
      if (a.g) mbar_wait(b_q + 8 * ub, (k >> 1) & 1);     // G visible to this thread
      if (q < a.Lq) {
        const float inv = l_run > 0.f ? fast_rcp(l_run) : 0.f;
        __nv_bfloat16* op = a.o + (int64_t)b * a.o_sb + (int64_t)h * a.o_sh + (int64_t)q * a.o_sl;
#pragma unroll
        for (int d0 = 0; d0 < DP; d0 += 8) {
          if (d0 >= a.D) break;
          float gv[8];
          if (a.g) {
            const uint4 gu = ld_shared_v4(gb + swz_offset(row, d0 / 8, C::kRowBytes));
            const uint32_t u4[4] = {gu.x, gu.y, gu.z, gu.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              gv[2 * i] = inv * fast_sigmoid(bf16_lo(u4[i]));
              gv[2 * i + 1] = inv * fast_sigmoid(bf16_hi(u4[i]));
            }
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) gv[i] = inv;
          }
          uint4 o4;
          o4.x = pack_bf16(__uint_as_float(ov[d0]) * gv[0], __uint_as_float(ov[d0 + 1]) * gv[1]);
          o4.y = pack_bf16(__uint_as_float(ov[d0 + 2]) * gv[2], __uint_as_float(ov[d0 + 3]) * gv[3]);
          o4.z = pack_bf16(__uint_as_float(ov[d0 + 4]) * gv[4], __uint_as_float(ov[d0 + 5]) * gv[5]);
          o4.w = pack_bf16(__uint_as_float(ov[d0 + 6]) * gv[6], __uint_as_float(ov[d0 + 7]) * gv[7]);
          *reinterpret_cast<uint4*>(op + d0) = o4;
        }
        a.lse[((int64_t)b * a.H + h) * a.Lq + q] =
            l_run > 0.f ? (m_ref == -INFINITY ? 0.f : m_ref) + __logf(l_run) : -INFINITY;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(b_qfree + 8 * ub);  // Q/G buffer ub may be reloaded
      ci += nc;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(*tmem_slot);
}

template <int DP, int BIAS>
static cudaError_t launch_fwd_pp_t(const FwdPpLaunch& L, cudaStream_t st) {
  auto kern = fwd_pp_kernel<DP, BIAS>;
  const size_t smem = PpCfg<DP, BIAS>::kSmem;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int nq = (L.args.Lq + 127) / 128;
  const long long U = (long long)L.args.B * L.args.H * nq;
  if (U == 0) return cudaSuccess;
  long long grid = (U + 1) / 2;
  if (grid > 148) grid = 148;
  kern<<<(unsigned)grid, 384, smem, st>>>(L.tm_q, L.tm_g, L.tm_k, L.tm_v, L.tm_b, L.args);
  return cudaGetLastError();
}

cudaError_t launch_fwd_pp_bf16(const FwdPpLaunch& L, int DP, int bias_mode, cudaStream_t st) {
#define EVO_PP_CASE(dp, bm) \
  if (DP == dp && bias_mode == bm) return launch_fwd_pp_t<dp, bm>(L, st);
  EVO_PP_CASE(16, 0) EVO_PP_CASE(16, 1) EVO_PP_CASE(16, 2)
  EVO_PP_CASE(32, 0) EVO_PP_CASE(32, 1) EVO_PP_CASE(32, 2)
#undef EVO_PP_CASE
  return cudaErrorInvalidValue;
}

}  // namespace evo
