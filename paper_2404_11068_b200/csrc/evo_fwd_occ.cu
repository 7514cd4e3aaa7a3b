// evo_fwd_occ.cu — occupancy-based bf16 forward (sm_100a): one (b, h, 128-query tile) unit per
// 128-thread CTA, four CTAs per SM.
//
// Same operation as the oracle's forward (pair bias added to the logits before the softmax,
// all of MHA fused, FlashAttention-style online softmax).  At head dim 32 the exp (MUFU) pipe
// binds, so the design goal is simply "always have a warp with exps ready": each SM runs four
// independent units whose softmax warps the hardware scheduler interleaves, instead of a
// hand-scheduled warp-specialised pipeline whose cross-warp hand-offs sit on the critical path.
//
// Per CTA (thread = query row = TMEM lane; thread 0 also issues TMA and tcgen05.mma):
//   TMEM (128 cols for D <= 32):  S|P [0,64)  O [64, 64+DP)  Q [96, 96+DP/2)  (G [.., +DP/2)
//   only with two key chunks or fewer: the gate row is otherwise prefetched to L2 and read in
//   the epilogue)
//   Q row -> TMEM once (tcgen05.st), then per 64-key chunk c (K/V/bias double-buffered by TMA):
//     S  = Q·K_cᵀ            tcgen05.mma, A = Q from TMEM (TS form), N = 64
//     x  = S·scale + bias    f32x2 FMA; hard mask; chunk max (3-input max)
//     lazy online-softmax rescale (threshold 8 in log2 units), p = exp2(x·log2e - m)
//     P (bf16x2) -> TMEM over the consumed S columns
//     O += P·V_c             tcgen05.mma, A = P from TMEM (TS form)
//   epilogue: o = O / l · sigmoid(g) (bf16), lse = m + log l (fp32)
#include <cstdio>

#include "evo_kernels.cuh"

namespace evo {

#ifdef EVO_TIMELINE
// Debug builds only (tools/fwd_timeline.py): per CTA (first 4096) its SM id and clock64 stamps:
// [0] start, [1] Q row in TMEM, [2 + 2c] S_c landed, [3 + 2c] P_c written (c < 8), [18] end.
__device__ unsigned long long g_ftl[4096][20];
#define FTL(i)                                                                   \
  do {                                                                           \
    if (threadIdx.x == 0 && blockIdx.x < 4096) g_ftl[blockIdx.x][i] = clock64(); \
  } while (0)
extern "C" int evo_debug_fwd_timeline_copy(void* dst, size_t bytes) {
  if (bytes > sizeof(g_ftl)) bytes = sizeof(g_ftl);
  return (int)cudaMemcpyFromSymbol(dst, g_ftl, bytes);
}
#else
#define FTL(i) do { } while (0)
#endif

template <int DP, int BIAS>
struct OccCfg {
  static constexpr uint32_t kRowBytes = DP * 2;
  static constexpr uint32_t kKV = 64 * kRowBytes;            // one 64-key K (or V) chunk
  static constexpr uint32_t kBias = BIAS ? 16384u : 0u;      // 128 x 64 bf16
  static constexpr uint32_t kStage = 2 * kKV + kBias;
  // K/V(/bias) ring depth: 2 stages with a bias tile (smem-bound at 4 CTAs/SM), 4 without (long
  // key sequences otherwise expose the TMA latency)
  static constexpr int kNSt = BIAS ? 2 : 4;
  static constexpr uint32_t oMask = kNSt * kStage + 128;     // 32-key hard-mask words
  static constexpr uint32_t kSmem = oMask + kMaxMaskWords * 4;
  static constexpr uint32_t kTmemCols = DP <= 32 ? 128 : 256;
  static constexpr uint32_t cS = 0, cO = 64, cQ = DP <= 32 ? 96 : 128;
};

template <int DP, int BIAS>
__global__ void __launch_bounds__(128, 4)
    fwd_occ_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                   const __grid_constant__ CUtensorMap tm_b, const FwdArgs a,
                   const __nv_bfloat16* __restrict__ qptr, int64_t q_sb, int64_t q_sh,
                   int64_t q_sl) {
  using C = OccCfg<DP, BIAS>;
  constexpr uint32_t kSw = DP == 64 ? kSw128 : (DP == 32 ? kSw64 : kSw32);
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t s0 = smem_u32(smem);
  if (s0 & 1023u) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kNSt * C::kStage);
  const uint32_t bar_kv0 = smem_u32(&bars[0]);  // +8·s: stage s
  const uint32_t bar_s = smem_u32(&bars[C::kNSt]);
  const uint32_t bar_o = smem_u32(&bars[C::kNSt + 1]);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(&bars[C::kNSt + 2]);

  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int nq = (a.Lq + 127) >> 7;
  const int nc = (a.Lk + 63) >> 6;
  const int qt = blockIdx.x % nq;
  const int bh = blockIdx.x / nq;
  const int h = bh % a.H, b = bh / a.H;
  const int q0 = qt * 128, q = q0 + tid;
  const bool qv = q < a.Lq;
#ifdef EVO_TIMELINE
  if (threadIdx.x == 0 && blockIdx.x < 4096) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_ftl[blockIdx.x][19] = smid;
  }
#endif
  FTL(0);

  if (w == 0) tmem_alloc<C::kTmemCols>(smem_u32(tmem_slot));
  if (tid == 32) {
    for (int i = 0; i < C::kNSt; ++i) mbar_init(bar_kv0 + 8 * i, 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_o, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();  // barriers initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = (uint32_t)(w * 32) << 16;
  const uint32_t tS = tmem + C::cS, tO = tmem + C::cO, tQ = tmem + C::cQ, tG = tQ + DP / 2;
  const int bc = a.bias_batched ? b : 0;
  auto load_chunk = [&](int c) {  // thread 0 only
    const int st = c % C::kNSt;
    const uint32_t sb = s0 + st * C::kStage;
    const uint32_t bar = bar_kv0 + 8 * st;
    mbar_arrive_expect_tx(bar, C::kStage);
    tma_load_4d(sb, &tm_k, bar, 0, c * 64, h, b);
    tma_load_4d(sb + C::kKV, &tm_v, bar, 0, c * 64, h, b);
    if (BIAS == 1) tma_load_4d(sb + 2 * C::kKV, &tm_b, bar, c * 64, q0, h, bc);  // rows q, cols k
    if (BIAS == 2) {                                                            // rows k, cols q
      tma_load_4d(sb + 2 * C::kKV, &tm_b, bar, q0, c * 64, h, bc);
      tma_load_4d(sb + 2 * C::kKV + 8192, &tm_b, bar, q0 + 64, c * 64, h, bc);
    }
  };
  constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, 0, 0);
  constexpr uint32_t idesc_o = make_idesc_bf16(128, DP, 0, 1);
  auto issue_S = [&](int c) {  // thread 0 only
    const uint32_t kb = s0 + (c % C::kNSt) * C::kStage;
    tc_fence_after();
#pragma unroll
    for (int kk = 0; kk < DP / 16; ++kk)
      umma_bf16_ts(tS, tQ + kk * 8, make_sdesc(kb + kk * 32, 16, 8 * C::kRowBytes, kSw), idesc_s,
                   kk > 0);
    umma_commit(bar_s);
  };
  // The first K/V/bias chunks (TMA), this thread's Q row and its gate row are all in flight
  // together (the gate's latency is otherwise exposed at the end of every unit).
  if (tid == 0) {
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    if (BIAS) tma_prefetch_desc(&tm_b);
    for (int c = 0; c < C::kNSt && c < nc; ++c) load_chunk(c);
  }
  uint32_t* smask = reinterpret_cast<uint32_t*>(smem + C::oMask);
  const bool all_kept = a.mask == nullptr && (a.Lk & 63) == 0;
  uint32_t keep_pre[4] = {0, 0, 0, 0};  // mask bytes of words w, w+4, w+8, w+12 (in flight)
  if (!all_kept) {
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int kk = (w + 4 * x) * 32 + lane;
      if (kk < a.Lk) keep_pre[x] = a.mask ? (uint32_t)a.mask[(int64_t)b * a.mask_s0 + (int64_t)kk * a.mask_s1] : 1u;
    }
  }
  // With more than two key chunks the gate row is read in the epilogue (an L2 prefetch issued
  // here hides its latency behind the key loop) instead of with the Q row into TMEM: L = 256
  // forward 54.2 / 55.3 / 63.5 -> 51.2 / 51.3 / 57.3 us (row / start / end).  Two chunks are
  // too short to hide it (MSA column, L = 128: 36.9 early vs 38.9 late), so the gate rides with
  // Q there.
  const bool late_g = nc > 2;
  {
    uint32_t qrow[DP / 2], gpk[DP / 2];
    const __nv_bfloat16* qp = qptr + (int64_t)b * q_sb + (int64_t)h * q_sh + (int64_t)q * q_sl;
    const __nv_bfloat16* gp = a.g + (int64_t)b * a.g_sb + (int64_t)h * a.g_sh + (int64_t)q * a.g_sl;
    if (late_g && a.g && qv) prefetch_l2(gp);  // loaded in the epilogue
#pragma unroll
    for (int d0 = 0; d0 < DP; d0 += 8) {
      uint4 v = make_uint4(0, 0, 0, 0), gv = make_uint4(0, 0, 0, 0);
      if (qv && d0 < a.D) {
        v = *reinterpret_cast<const uint4*>(qp + d0);
        if (a.g && !late_g) gv = *reinterpret_cast<const uint4*>(gp + d0);
      }
      qrow[d0 / 2] = v.x; qrow[d0 / 2 + 1] = v.y; qrow[d0 / 2 + 2] = v.z; qrow[d0 / 2 + 3] = v.w;
      gpk[d0 / 2] = gv.x; gpk[d0 / 2 + 1] = gv.y; gpk[d0 / 2 + 2] = gv.z; gpk[d0 / 2 + 3] = gv.w;
    }
  // Q row and the gate row (packed bf16) go to this thread's TMEM lane: Q is the A operand of
  // Sᵀ's TS-form MMA, the gate waits there for the epilogue (no registers held across the loop)
  if (DP == 16) {
    tmem_st8(tQ + lane_base, *reinterpret_cast<uint32_t(*)[8]>(qrow));
    tmem_st8(tG + lane_base, *reinterpret_cast<uint32_t(*)[8]>(gpk));
  } else if (DP == 32) {
    tmem_st16(tQ + lane_base, *reinterpret_cast<uint32_t(*)[16]>(qrow));
    tmem_st16(tG + lane_base, *reinterpret_cast<uint32_t(*)[16]>(gpk));
  } else {
    tmem_st32(tQ + lane_base, *reinterpret_cast<uint32_t(*)[32]>(qrow));
    tmem_st32(tG + lane_base, *reinterpret_cast<uint32_t(*)[32]>(gpk));
  }
  }
  // hard-mask bits of this unit's batch row as 32-key words in smem (one pass instead of a
  // dependent global load per chunk); the first words' loads were issued with the Q/G loads
  if (!all_kept) {
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int wd = w + 4 * x;
      if (wd < nc * 2) {
        const uint32_t word = __ballot_sync(0xffffffffu, keep_pre[x] != 0);
        if (lane == 0) smask[wd] = word;
      }
    }
    for (int wd = w + 16; wd < nc * 2; wd += 4) {
      const int kk = wd * 32 + lane;
      const uint32_t keep = kk < a.Lk ? (a.mask ? (uint32_t)a.mask[(int64_t)b * a.mask_s0 + (int64_t)kk * a.mask_s1] : 1u) : 0u;
      const uint32_t word = __ballot_sync(0xffffffffu, keep != 0);
      if (lane == 0) smask[wd] = word;
    }
  }
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();  // Q in TMEM, mask words in smem
  FTL(1);
  if (tid == 0) {
    tc_fence_after();
    mbar_wait(bar_kv0, 0);
    issue_S(0);
  }

  const uint64_t scale2 = f2_pack(a.scale, a.scale);
  const uint64_t log2e2 = f2_pack(kLog2e, kLog2e);
  float m_ref = -INFINITY, l_run = 0.f;  // natural-log units
  for (int c = 0; c < nc; ++c) {
    const int st = c % C::kNSt;
    const uint32_t sb = s0 + st * C::kStage;
    uint32_t mw0 = ~0u, mw1 = ~0u;
    if (!all_kept) { mw0 = smask[2 * c]; mw1 = smask[2 * c + 1]; }
    mbar_wait(bar_s, c & 1);
    if (c < 8) FTL(2 + 2 * c);
    tc_fence_after();
    if (tid == 0 && c >= 1 && c - 1 + C::kNSt < nc) {
      // PV_{c-1} has landed (it precedes S_c in the MMA pipe): chunk c-1's stage is free
      mbar_wait(bar_o, (c - 1) & 1);
      load_chunk(c - 1 + C::kNSt);
    }
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
    // x = S·scale + bias
    const uint32_t bb = sb + 2 * C::kKV;
    if (BIAS == 1) {  // bias chunk rows q (this thread's row), cols k: one SW128 region
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        const uint4 v = ld_shared_v4(bb + swz_offset(tid, cc, 128));
        const uint32_t u4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int k = cc * 8 + 2 * i;
          f2_unpack(f2_fma(f2_pack(x[k], x[k + 1]), scale2, bf16x2_to_f2(u4[i])), x[k], x[k + 1]);
        }
      }
    } else if (BIAS == 2) {  // rows k, cols q: two 64-q regions
      const uint32_t base = bb + (tid >> 6) * 8192 + (tid & 7) * 2;
      const uint32_t qc = (tid & 63) >> 3;
#pragma unroll
      for (int k = 0; k < 64; ++k) {
        const float bv = bf16_to_f(ld_shared_u16(base + k * 128 + ((qc ^ (k & 7)) << 4)));
        x[k] = fmaf(x[k], a.scale, bv);
      }
    } else {
#pragma unroll
      for (int k = 0; k < 64; k += 2) f2_unpack(f2_mul(f2_pack(x[k], x[k + 1]), scale2), x[k], x[k + 1]);
    }
    if ((mw0 & mw1) != ~0u) {
#pragma unroll
      for (int k = 0; k < 64; ++k)
        x[k] = (((k < 32 ? mw0 : mw1) >> (k & 31)) & 1u) ? x[k] : -INFINITY;
    }
    float m4[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) m4[i] = fmaxf(x[i], x[4 + i]);
#pragma unroll
    for (int k = 8; k < 64; k += 8)
#pragma unroll
      for (int i = 0; i < 4; ++i) m4[i] = fmax3(m4[i], x[k + i], x[k + 4 + i]);
    const float mx = fmax3(fmaxf(m4[0], m4[1]), m4[2], m4[3]);
    // lazy online-softmax rescale (threshold 8 in log2 units); PV_{c-1} is complete here (S_c
    // was issued after it and the MMA pipe executes in order), so O may be touched directly
    const float m_new = fmaxf(m_ref, mx);
    if (c == 0) {
      m_ref = m_new;
    } else {
      const bool need = (m_new - m_ref) * kLog2e > 8.f;
      if (__any_sync(0xffffffffu, need)) {
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
    if (c < 8) FTL(3 + 2 * c);
    tc_fence_before();
    __syncthreads();  // all P written; S_c fully consumed; bias stage read
    if (tid == 0) {
      tc_fence_after();
      const uint32_t vb = sb + C::kKV;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        umma_bf16_ts(tO, tS + kk * 8, make_sdesc(vb + kk * 16 * C::kRowBytes, 16384, 8 * C::kRowBytes, kSw),
                     idesc_o, (c > 0 || kk > 0) ? 1u : 0u);
      umma_commit(bar_o);
      if (c + 1 < nc) {
        // S_{c+1} overwrites the P columns PV_c reads: tcgen05.mma executes in issue order, so
        // it is issued right behind PV_c (no wait for PV_c on the critical path)
        mbar_wait(bar_kv0 + 8 * ((c + 1) % C::kNSt), ((c + 1) / C::kNSt) & 1);
        issue_S(c + 1);
      }
    }
  }
  // ---- epilogue
  mbar_wait(bar_o, (nc - 1) & 1);
  tc_fence_after();
  uint32_t ov[DP];
  if (DP == 16) {
    uint32_t r[16];
    tmem_ld16(tO + lane_base, r);
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 16; ++i) ov[i] = r[i];
  } else {
#pragma unroll
    for (int c0 = 0; c0 < DP; c0 += 32) {
      uint32_t r[32];
      tmem_ld32(tO + lane_base + c0, r);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) ov[c0 + i] = r[i];
    }
  }
  uint32_t gpk[DP / 2];
  if (late_g) {
    if (a.g && qv) {
      const __nv_bfloat16* gp = a.g + (int64_t)b * a.g_sb + (int64_t)h * a.g_sh + (int64_t)q * a.g_sl;
#pragma unroll
      for (int d0 = 0; d0 < DP; d0 += 8) {
        uint4 gv = make_uint4(0, 0, 0, 0);
        if (d0 < a.D) gv = *reinterpret_cast<const uint4*>(gp + d0);
        gpk[d0 / 2] = gv.x; gpk[d0 / 2 + 1] = gv.y; gpk[d0 / 2 + 2] = gv.z; gpk[d0 / 2 + 3] = gv.w;
      }
    }
  } else {
    if (DP == 16) tmem_ld8(tG + lane_base, *reinterpret_cast<uint32_t(*)[8]>(gpk));
    else if (DP == 32) tmem_ld16(tG + lane_base, *reinterpret_cast<uint32_t(*)[16]>(gpk));
    else tmem_ld32(tG + lane_base, *reinterpret_cast<uint32_t(*)[32]>(gpk));
    tmem_wait_ld();
  }
  if (qv) {
    const float inv = l_run > 0.f ? fast_rcp(l_run) : 0.f;
    __nv_bfloat16* op = a.o + (int64_t)b * a.o_sb + (int64_t)h * a.o_sh + (int64_t)q * a.o_sl;
#pragma unroll
    for (int d0 = 0; d0 < DP; d0 += 8) {
      if (d0 >= a.D) break;
      float gv[8];
      if (a.g) {
        const uint32_t u[4] = {gpk[d0 / 2], gpk[d0 / 2 + 1], gpk[d0 / 2 + 2], gpk[d0 / 2 + 3]};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          gv[2 * i] = inv * fast_sigmoid(bf16_lo(u[i]));
          gv[2 * i + 1] = inv * fast_sigmoid(bf16_hi(u[i]));
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
  FTL(18);
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<C::kTmemCols>(tmem);
}

template <int DP, int BIAS>
static cudaError_t launch_fwd_occ_t(const FwdOccLaunch& L, cudaStream_t st) {
  auto kern = fwd_occ_kernel<DP, BIAS>;
  const size_t smem = OccCfg<DP, BIAS>::kSmem;
  cudaError_t e = set_smem_once(kern, smem);
  if (e != cudaSuccess) return e;
  const long long grid = (long long)L.args.B * L.args.H * ((L.args.Lq + 127) / 128);
  if (grid == 0) return cudaSuccess;
  kern<<<(unsigned)grid, 128, smem, st>>>(L.tm_k, L.tm_v, L.tm_b, L.args, L.q, L.q_sb, L.q_sh,
                                          L.q_sl);
  return cudaGetLastError();
}

cudaError_t launch_fwd_occ_bf16(const FwdOccLaunch& L, int DP, int bias_mode, cudaStream_t st) {
#define EVO_OCC_CASE(dp, bm) \
  if (DP == dp && bias_mode == bm) return launch_fwd_occ_t<dp, bm>(L, st);
  EVO_OCC_CASE(16, 0) EVO_OCC_CASE(16, 1) EVO_OCC_CASE(16, 2)
  EVO_OCC_CASE(32, 0) EVO_OCC_CASE(32, 1) EVO_OCC_CASE(32, 2)
  EVO_OCC_CASE(64, 0) EVO_OCC_CASE(64, 1) EVO_OCC_CASE(64, 2)
#undef EVO_OCC_CASE
  return cudaErrorInvalidValue;
}

}  // namespace evo
