// evo_bwd_fused.cu — single-pass bf16 backward on sm_100a: dK, dV, dQ and the pair-bias
// gradient of one (head, 128-key tile) for a chunk of batch rows, in one persistent CTA.
//
// Same arithmetic as evo_bwd.cu's bwd_main + bwd_bias (SPEC.md L168
// recompute backward; dbias = Σ_b dS over the broadcast axis, PAPER.md L294 / north star), but
// the probabilities are recomputed ONCE: the CTA loops over its batch rows and, for each, over
// 64-query sub-tiles, and accumulates Σ_b dSᵀ for its key tile in TMEM (fp32, read-modify-write
// by the owning thread), so the separate dbias pass and its second recompute disappear.
//
// Roles (320 threads): warps 0-7 compute (thread = key row k = TMEM lane, warp>>2 = which 32
// queries of the 64-query sub-tile), warp 8 lane 0 issues tcgen05.mma, warp 9 lane 0 issues TMA.
// Per sub-tile j (queries q0..q0+63 of batch row b):
//   MMA:      Sᵀ = K_b·Q_jᵀ, dPᵀ = V_b·dA_jᵀ      (M = 128 keys, N = 64 queries)  -> TMEM
//   compute:  Pᵀ = exp2(Sᵀ·scale·log2e + biasᵀ·log2e − lse2), dSᵀ = Pᵀ⊙(dPᵀ − D)
//             Σ_b dSᵀ += dSᵀ (TMEM RMW), Pᵀ, dSᵀ -> smem bf16 (SW128, K-major)
//   MMA:      dV_b += Pᵀ·dA_j, dK_b += dSᵀ·Q_j;  after both halves of a 128-query tile:
//             dQ_part = dS·K_b (A = the dSᵀ tile read MN-major)
// The next sub-tile's Sᵀ/dPᵀ MMAs are issued as soon as the compute warps have pulled the
// current ones into registers, so the tensor core runs under the exp/ALU work.
//
// TMEM (512 cols): [0, Lq_pad) Σ dSᵀ (with bias) | Sᵀ 64 | dPᵀ 64 | dV DP | dK DP | dQ DP
// SMEM: biasᵀ resident [128 k][Lq_pad] bf16 (16-B chunks XOR-swizzled by k&7) | K,V x2 stages |
//       Q,dA x2 stages | Pᵀ 16 KB | dSᵀ 32 KB (one 128-query tile) | lse2/D x2 | barriers
#include "evo_kernels.cuh"

namespace evo {

template <int DP, bool BIAS>
struct FusedCfg {
  static constexpr uint32_t kRowBytes = DP * 2;
  static constexpr uint32_t kTile = 128 * kRowBytes;  // one 128-row Q/K/V/dA tile
  // resident biasᵀ for Lq_pad <= 256 (<= 128 at DP = 64: bwd_fused_supported's TMEM rule)
  static constexpr uint32_t kBiasMax = BIAS ? 128u * (DP == 64 ? 128u : 256u) * 2u : 0u;
  static constexpr uint32_t oBias = 0;
  static constexpr uint32_t oKV = oBias + kBiasMax;      // stage s: K at +s*2*kTile, V +kTile
  static constexpr uint32_t oQA = oKV + 4 * kTile;       // stage s: Q at +s*2*kTile, dA +kTile
  static constexpr uint32_t oP = oQA + 4 * kTile;        // 16 KB
  static constexpr uint32_t oDS = oP + 16384;            // 32 KB (2 x 64-query halves)
  static constexpr uint32_t oVec = oDS + 32768;          // 2 x (lse2[128], D[128]) fp32
  static constexpr uint32_t oBar = oVec + 2048;
  static constexpr uint32_t kSmem = oBar + 256;
};

template <int DP, bool BIAS>
__global__ void __launch_bounds__(320, 1)
    bwd_fused_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_da,
                     const BwdFusedArgs a) {
  using C = FusedCfg<DP, BIAS>;
  constexpr uint32_t kSw = DP == 64 ? kSw128 : (DP == 32 ? kSw64 : kSw32);
  constexpr uint32_t kHalf = DP / 2;  // d columns per compute-warp half in the drains
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t s0 = smem_u32(smem);
  if (s0 & 1023u) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::oBar);
  const uint32_t bar_kv = smem_u32(&bars[0]);       // +8: stage 1   (TMA K,V landed)
  const uint32_t bar_in = smem_u32(&bars[2]);       // +8: stage 1   (TMA Q,dA,vec landed)
  const uint32_t bar_kvfree = smem_u32(&bars[4]);   // +8            (MMA done with K,V stage)
  const uint32_t bar_infree = smem_u32(&bars[6]);   // +8            (MMA done with Q,dA stage)
  const uint32_t bar_sp = smem_u32(&bars[8]);       // Sᵀ, dPᵀ in TMEM
  const uint32_t bar_sfree = smem_u32(&bars[9]);    // compute pulled Sᵀ, dPᵀ (8 warps)
  const uint32_t bar_ps = smem_u32(&bars[10]);      // Pᵀ, dSᵀ in smem (8 warps)
  const uint32_t bar_mm = smem_u32(&bars[11]);      // dV/dK MMAs of a sub-tile done
  const uint32_t bar_dq = smem_u32(&bars[12]);      // dQ MMA of a query tile done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(&bars[14]);

  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int nq = (a.Lq + 127) >> 7, nk = (a.Lk + 127) >> 7;
  const int Lq_pad = nq * 128, Lk_pad = nk * 128;
  const int c = blockIdx.x % a.nchunks;
  const int grp = blockIdx.x / a.nchunks;
  const int kt = grp % nk, h = grp / nk;
  const int k0 = kt * 128;
  const int b0 = c * a.chunk;
  const int nb = min(a.B - b0, a.chunk);
  if (nb <= 0) return;
  const int J = nb * nq * 2;  // sub-tiles

  if (w == 0) tmem_alloc<512>(smem_u32(tmem_slot));
  if (tid == 32) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_kv + 8 * i, 1);
      mbar_init(bar_in + 8 * i, 1);
      mbar_init(bar_kvfree + 8 * i, 1);
      mbar_init(bar_infree + 8 * i, 1);
    }
    mbar_init(bar_sp, 1);
    mbar_init(bar_sfree, 8);
    mbar_init(bar_ps, 8);
    mbar_init(bar_mm, 1);
    mbar_init(bar_dq, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t cb = BIAS ? (uint32_t)Lq_pad : 0u;
  const uint32_t tDB = tmem, tSt = tmem + cb, tdPt = tSt + 64, tdV = tSt + 128, tdK = tdV + DP,
                 tdQ = tdK + DP;

  if (w == 9) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      tma_prefetch_desc(&tm_da);
      for (int bi = 0; bi < nb; ++bi) {
        const int b = b0 + bi, kvs = bi & 1;
        if (bi >= 2) mbar_wait(bar_kvfree + 8 * kvs, ((bi - 2) >> 1) & 1);
        const uint32_t kb = s0 + C::oKV + kvs * 2 * C::kTile;
        mbar_arrive_expect_tx(bar_kv + 8 * kvs, 2 * C::kTile);
        tma_load_4d(kb, &tm_k, bar_kv + 8 * kvs, 0, k0, h, b);
        tma_load_4d(kb + C::kTile, &tm_v, bar_kv + 8 * kvs, 0, k0, h, b);
        for (int t = 0; t < nq; ++t) {
          const int T = bi * nq + t, st = T & 1;
          if (T >= 2) mbar_wait(bar_infree + 8 * st, ((T - 2) >> 1) & 1);
          const uint32_t qb = s0 + C::oQA + st * 2 * C::kTile;
          const uint32_t bar = bar_in + 8 * st;
          mbar_arrive_expect_tx(bar, 2 * C::kTile + 1024);
          tma_load_4d(qb, &tm_q, bar, 0, t * 128, h, b);
          tma_load_4d(qb + C::kTile, &tm_da, bar, 0, t * 128, h, b);
          const int64_t vrow = ((int64_t)b * a.H + h) * Lq_pad + t * 128;
          bulk_load(s0 + C::oVec + st * 1024, a.lse2 + vrow, 512, bar);
          bulk_load(s0 + C::oVec + st * 1024 + 512, a.Dvec + vrow, 512, bar);
        }
      }
    }
  } else if (w == 8) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, 0, 0);   // Sᵀ, dPᵀ
      constexpr uint32_t idesc_kv = make_idesc_bf16(128, DP, 0, 1);  // dV, dK (B MN-major)
      constexpr uint32_t idesc_q = make_idesc_bf16(128, DP, 1, 1);   // dQ (A, B MN-major)
      for (int j = 0; j <= J; ++j) {
        if (j < J) {
          const int bi = j / (2 * nq), t = (j >> 1) % nq, sub = j & 1, T = j >> 1;
          const int st = T & 1, kvs = bi & 1;
          if (sub == 0) mbar_wait(bar_in + 8 * st, (T >> 1) & 1);
          if (sub == 0 && t == 0) mbar_wait(bar_kv + 8 * kvs, (bi >> 1) & 1);
          if (j > 0) mbar_wait(bar_sfree, (j - 1) & 1);
          tc_fence_after();
          const uint32_t kb = s0 + C::oKV + kvs * 2 * C::kTile;
          const uint32_t qb = s0 + C::oQA + st * 2 * C::kTile + sub * 64 * C::kRowBytes;
#pragma unroll
          for (int kk = 0; kk < DP / 16; ++kk)
            umma_bf16(tSt, make_sdesc(kb + kk * 32, 16, 8 * C::kRowBytes, kSw),
                      make_sdesc(qb + kk * 32, 16, 8 * C::kRowBytes, kSw), idesc_s, kk > 0);
#pragma unroll
          for (int kk = 0; kk < DP / 16; ++kk)
            umma_bf16(tdPt, make_sdesc(kb + C::kTile + kk * 32, 16, 8 * C::kRowBytes, kSw),
                      make_sdesc(qb + C::kTile + kk * 32, 16, 8 * C::kRowBytes, kSw), idesc_s,
                      kk > 0);
          umma_commit(bar_sp);
        }
        if (j > 0) {
          const int i = j - 1;
          const int bi = i / (2 * nq), t = (i >> 1) % nq, sub = i & 1, T = i >> 1;
          const int st = T & 1, kvs = bi & 1;
          mbar_wait(bar_ps, i & 1);
          tc_fence_after();
          const uint32_t qb = s0 + C::oQA + st * 2 * C::kTile + sub * 64 * C::kRowBytes;
          const uint32_t ab = qb + C::kTile;
          const uint32_t pb = s0 + C::oP, db = s0 + C::oDS + sub * 16384;
          const uint32_t acc0 = (t > 0 || sub > 0) ? 1u : 0u;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // dV += Pᵀ·dA (K = 64 queries)
            umma_bf16(tdV, make_sdesc(pb + kk * 32, 16, 1024, kSw128),
                      make_sdesc(ab + kk * 16 * C::kRowBytes, 16384, 8 * C::kRowBytes, kSw),
                      idesc_kv, (acc0 | (uint32_t)kk) ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // dK += dSᵀ·Q
            umma_bf16(tdK, make_sdesc(db + kk * 32, 16, 1024, kSw128),
                      make_sdesc(qb + kk * 16 * C::kRowBytes, 16384, 8 * C::kRowBytes, kSw),
                      idesc_kv, (acc0 | (uint32_t)kk) ? 1u : 0u);
          umma_commit(bar_mm);
          if (sub == 1) {  // both halves of the query tile are in the dSᵀ buffer: dQ part
            const uint32_t kb = s0 + C::oKV + kvs * 2 * C::kTile;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              umma_bf16(tdQ, make_sdesc(s0 + C::oDS + kk * 2048, 16384, 1024, kSw128),
                        make_sdesc(kb + kk * 16 * C::kRowBytes, 16384, 8 * C::kRowBytes, kSw),
                        idesc_q, kk > 0 ? 1u : 0u);
            umma_commit(bar_dq);
            umma_commit(bar_infree + 8 * st);
            if (t == nq - 1) umma_commit(bar_kvfree + 8 * kvs);
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------------ compute warps 0-7
    const int qd = w & 3, hh = w >> 2;
    const int row = qd * 32 + lane;  // key row within the tile = TMEM lane
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    const uint32_t RB = (uint32_t)Lq_pad * 2;  // resident biasᵀ row bytes
    const uint32_t sBias = s0 + C::oBias;
    if (BIAS) {
      // biasᵀ[k][q] = bias[h, q, k0 + k] for q < Lq, k0 + k < Lk; 0 elsewhere (padding must be
      // finite: it meets zero P/dA rows in the MMAs)
      const __nv_bfloat16* bp = a.bias + (int64_t)h * a.b_sh;
      if (a.b_sk == 1) {  // k-contiguous rows: lanes along k, 4 keys each
        for (int q = tid >> 5; q < Lq_pad; q += 8) {
          const int kl = lane * 4;
          uint16_t v4[4] = {0, 0, 0, 0};
          if (q < a.Lq) {
            const __nv_bfloat16* src = bp + (int64_t)q * a.b_sq + k0 + kl;
            if (k0 + kl + 3 < a.Lk) {
              const uint2 u = *reinterpret_cast<const uint2*>(src);
              v4[0] = u.x & 0xffff; v4[1] = u.x >> 16; v4[2] = u.y & 0xffff; v4[3] = u.y >> 16;
            } else {
              for (int e = 0; e < 4; ++e)
                if (k0 + kl + e < a.Lk) v4[e] = __bfloat16_as_ushort(src[e]);
            }
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t r = kl + e;
            const uint32_t addr = sBias + r * RB + ((((uint32_t)q >> 3) ^ (r & 7)) << 4) + (q & 7) * 2;
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v4[e]) : "memory");
          }
        }
      } else {  // q-contiguous rows: thread per key row, 8 queries per 16-B load
        for (int r = tid; r < 128; r += 256) {
          const __nv_bfloat16* src = bp + (int64_t)(k0 + r) * a.b_sk;
          const bool kv = k0 + r < a.Lk;
          for (int q8 = 0; q8 < Lq_pad / 8; ++q8) {
            uint4 u = make_uint4(0, 0, 0, 0);
            if (kv && q8 * 8 < a.Lq) {
              if (q8 * 8 + 7 < a.Lq) {
                u = *reinterpret_cast<const uint4*>(src + q8 * 8);
              } else {
                uint16_t e8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                for (int e = 0; e < 8; ++e)
                  if (q8 * 8 + e < a.Lq) e8[e] = __bfloat16_as_ushort(src[q8 * 8 + e]);
                u = make_uint4(e8[0] | (e8[1] << 16), e8[2] | (e8[3] << 16), e8[4] | (e8[5] << 16),
                               e8[6] | (e8[7] << 16));
              }
            }
            st_shared_v4(sBias + r * RB + (((uint32_t)q8 ^ (r & 7)) << 4), u.x, u.y, u.z, u.w);
          }
        }
      }
      named_bar_sync(1, 256);
    }

    const uint64_t sl2 = f2_pack(a.scale_log2, a.scale_log2);
    const uint64_t l2e2 = f2_pack(kLog2e, kLog2e);
    bool keep = false;
    const int kglob = k0 + row;
    for (int j = 0; j < J; ++j) {
      const int bi = j / (2 * nq), t = (j >> 1) % nq, sub = j & 1, T = j >> 1;
      const int st = T & 1;
      const int b = b0 + bi;
      if (sub == 0 && t == 0) {
        keep = kglob < a.Lk;
        if (keep && a.mask) keep = a.mask[(int64_t)b * a.mask_s0 + (int64_t)kglob * a.mask_s1] != 0;
      }
      mbar_wait(bar_sp, j & 1);
      tc_fence_after();
      uint32_t rs[32], rd[32];
      tmem_ld32(tSt + lane_base + hh * 32, rs);
      tmem_ld32(tdPt + lane_base + hh * 32, rd);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_sfree);
      mbar_wait(bar_in + 8 * st, (T >> 1) & 1);  // lse2 / D of this query tile visible
      const uint32_t vbase = s0 + C::oVec + st * 1024 + (sub * 64 + hh * 32) * 4;
      const int qcol = t * 128 + sub * 64 + hh * 32;  // first query of this thread's 32
      uint32_t pk[16], dk2[16];
      float ds[32];
#pragma unroll
      for (int g = 0; g < 4; ++g) {  // 8 queries per group
        const uint4 l0 = ld_shared_v4(vbase + g * 32), l1 = ld_shared_v4(vbase + g * 32 + 16);
        const uint4 d0 = ld_shared_v4(vbase + 512 + g * 32), d1 = ld_shared_v4(vbase + 512 + g * 32 + 16);
        const uint32_t nl[8] = {l0.x ^ 0x80000000u, l0.y ^ 0x80000000u, l0.z ^ 0x80000000u,
                                l0.w ^ 0x80000000u, l1.x ^ 0x80000000u, l1.y ^ 0x80000000u,
                                l1.z ^ 0x80000000u, l1.w ^ 0x80000000u};
        const uint32_t nd[8] = {d0.x ^ 0x80000000u, d0.y ^ 0x80000000u, d0.z ^ 0x80000000u,
                                d0.w ^ 0x80000000u, d1.x ^ 0x80000000u, d1.y ^ 0x80000000u,
                                d1.z ^ 0x80000000u, d1.w ^ 0x80000000u};
        uint32_t bu[4] = {0, 0, 0, 0};
        if (BIAS) {
          const uint4 bv = ld_shared_v4(sBias + row * RB + (((uint32_t)(qcol >> 3) + g) ^ (row & 7)) * 16);
          bu[0] = bv.x; bu[1] = bv.y; bu[2] = bv.z; bu[3] = bv.w;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int i = g * 8 + 2 * e;
          const uint64_t nl2 = ((uint64_t)nl[2 * e + 1] << 32) | nl[2 * e];
          const uint64_t nd2 = ((uint64_t)nd[2 * e + 1] << 32) | nd[2 * e];
          uint64_t x = BIAS ? f2_fma(bf16x2_to_f2(bu[e]), l2e2, nl2) : nl2;
          x = f2_fma(((uint64_t)rs[i + 1] << 32) | rs[i], sl2, x);
          float x0, x1;
          f2_unpack(x, x0, x1);
          float p0 = fast_exp2(x0), p1 = fast_exp2(x1);
          if (!keep) { p0 = 0.f; p1 = 0.f; }
          const uint64_t p2 = f2_pack(p0, p1);
          const uint64_t dd = f2_mul(p2, f2_add(((uint64_t)rd[i + 1] << 32) | rd[i], nd2));
          f2_unpack(dd, ds[i], ds[i + 1]);
          pk[i / 2] = pack_bf16(p0, p1);
          dk2[i / 2] = pack_bf16(ds[i], ds[i + 1]);
        }
      }
      if (BIAS) {  // Σ_b dSᵀ in TMEM (this thread's lane, its 32 query columns)
        uint32_t acc[32];
        if (bi == 0) {  // first batch row of the chunk initialises the (uninitialised) TMEM
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[i] = __float_as_uint(ds[i]);
        } else {
          tmem_ld32(tDB + lane_base + qcol, acc);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const uint64_t s2 = f2_add(((uint64_t)acc[i + 1] << 32) | acc[i], f2_pack(ds[i], ds[i + 1]));
            float lo, hi;
            f2_unpack(s2, lo, hi);
            acc[i] = __float_as_uint(lo);
            acc[i + 1] = __float_as_uint(hi);
          }
        }
        tmem_st32(tDB + lane_base + qcol, acc);
      }
      // previous sub-tile's dV/dK MMAs have consumed Pᵀ / dSᵀ (and, at a new batch row, the
      // dK/dV accumulators are final; at a new query tile, dQ of the previous one is issued)
      if (j > 0) {
        mbar_wait(bar_mm, (j - 1) & 1);
        tc_fence_after();
        if (sub == 0) {  // dQ part of query tile T-1 (TMEM lane = query row)
          mbar_wait(bar_dq, (T - 1) & 1);
          tc_fence_after();
          const int tp = (T - 1) % nq, bp = b0 + (T - 1) / nq;
          const int q = tp * 128 + row;
          uint32_t r[kHalf];
          if constexpr (kHalf == 8) tmem_ld8(tdQ + lane_base + hh * kHalf, *reinterpret_cast<uint32_t(*)[8]>(r));
          else if constexpr (kHalf == 16) tmem_ld16(tdQ + lane_base + hh * kHalf, *reinterpret_cast<uint32_t(*)[16]>(r));
          else tmem_ld32(tdQ + lane_base + hh * kHalf, *reinterpret_cast<uint32_t(*)[32]>(r));
          tmem_wait_ld();
          if (q < a.Lq) {
#pragma unroll
            for (int e = 0; e < (int)kHalf; e += 8) {
              const int d0 = hh * kHalf + e;
              if (d0 >= a.D) break;
              if (nk == 1) {
                uint4 o;
                o.x = pack_bf16(__uint_as_float(r[e]) * a.scale, __uint_as_float(r[e + 1]) * a.scale);
                o.y = pack_bf16(__uint_as_float(r[e + 2]) * a.scale, __uint_as_float(r[e + 3]) * a.scale);
                o.z = pack_bf16(__uint_as_float(r[e + 4]) * a.scale, __uint_as_float(r[e + 5]) * a.scale);
                o.w = pack_bf16(__uint_as_float(r[e + 6]) * a.scale, __uint_as_float(r[e + 7]) * a.scale);
                *reinterpret_cast<uint4*>(a.dq + (int64_t)bp * a.q_sb + (int64_t)h * a.q_sh +
                                          (int64_t)q * a.q_sl + d0) = o;
              } else {
                float4* dst = reinterpret_cast<float4*>(a.dq_acc + (((int64_t)bp * a.H + h) * a.Lq + q) * a.D + d0);
                atomicAdd(dst, make_float4(__uint_as_float(r[e]), __uint_as_float(r[e + 1]),
                                           __uint_as_float(r[e + 2]), __uint_as_float(r[e + 3])));
                atomicAdd(dst + 1, make_float4(__uint_as_float(r[e + 4]), __uint_as_float(r[e + 5]),
                                               __uint_as_float(r[e + 6]), __uint_as_float(r[e + 7])));
              }
            }
          }
          if (t == 0) {  // dK, dV of the previous batch row are complete
            const int bprev = b - 1;
            uint32_t rk[kHalf], rv[kHalf];
            if constexpr (kHalf == 8) {
              tmem_ld8(tdK + lane_base + hh * kHalf, *reinterpret_cast<uint32_t(*)[8]>(rk));
              tmem_ld8(tdV + lane_base + hh * kHalf, *reinterpret_cast<uint32_t(*)[8]>(rv));
            } else if constexpr (kHalf == 16) {
              tmem_ld16(tdK + lane_base + hh * kHalf, *reinterpret_cast<uint32_t(*)[16]>(rk));
              tmem_ld16(tdV + lane_base + hh * kHalf, *reinterpret_cast<uint32_t(*)[16]>(rv));
            } else {
              tmem_ld32(tdK + lane_base + hh * kHalf, *reinterpret_cast<uint32_t(*)[32]>(rk));
              tmem_ld32(tdV + lane_base + hh * kHalf, *reinterpret_cast<uint32_t(*)[32]>(rv));
            }
            tmem_wait_ld();
            if (kglob < a.Lk) {
#pragma unroll
              for (int e = 0; e < (int)kHalf; e += 8) {
                const int d0 = hh * kHalf + e;
                if (d0 >= a.D) break;
                uint4 x, y;
                x.x = pack_bf16(__uint_as_float(rk[e]) * a.scale, __uint_as_float(rk[e + 1]) * a.scale);
                x.y = pack_bf16(__uint_as_float(rk[e + 2]) * a.scale, __uint_as_float(rk[e + 3]) * a.scale);
                x.z = pack_bf16(__uint_as_float(rk[e + 4]) * a.scale, __uint_as_float(rk[e + 5]) * a.scale);
                x.w = pack_bf16(__uint_as_float(rk[e + 6]) * a.scale, __uint_as_float(rk[e + 7]) * a.scale);
                y.x = pack_bf16(__uint_as_float(rv[e]), __uint_as_float(rv[e + 1]));
                y.y = pack_bf16(__uint_as_float(rv[e + 2]), __uint_as_float(rv[e + 3]));
                y.z = pack_bf16(__uint_as_float(rv[e + 4]), __uint_as_float(rv[e + 5]));
                y.w = pack_bf16(__uint_as_float(rv[e + 6]), __uint_as_float(rv[e + 7]));
                *reinterpret_cast<uint4*>(a.dk + (int64_t)bprev * a.k_sb + (int64_t)h * a.k_sh +
                                          (int64_t)kglob * a.k_sl + d0) = x;
                *reinterpret_cast<uint4*>(a.dv + (int64_t)bprev * a.v_sb + (int64_t)h * a.v_sh +
                                          (int64_t)kglob * a.v_sl + d0) = y;
              }
            }
          }
        }
      }
      // Pᵀ and dSᵀ rows (this thread's key row, its 32 queries = 4 x 16-B chunks, SW128)
      {
        const uint32_t pb = s0 + C::oP, db = s0 + C::oDS + sub * 16384;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t off = swz_offset(row, hh * 4 + e, 128);
          st_shared_v4(pb + off, pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]);
          st_shared_v4(db + off, dk2[4 * e], dk2[4 * e + 1], dk2[4 * e + 2], dk2[4 * e + 3]);
        }
      }
      if (BIAS) tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_ps);
    }
    // ---- tail: last dQ part, last dK/dV, then this chunk's Σ_b dSᵀ
    mbar_wait(bar_mm, (J - 1) & 1);
    mbar_wait(bar_dq, ((J >> 1) - 1) & 1);
    tc_fence_after();
    {
      const int Tl = (J >> 1) - 1;
      const int tp = Tl % nq, bp = b0 + Tl / nq;
      const int q = tp * 128 + row;
      uint32_t r[kHalf], rk[kHalf], rv[kHalf];
      if constexpr (kHalf == 8) {
        tmem_ld8(tdQ + lane_base + hh * kHalf, *reinterpret_cast<uint32_t(*)[8]>(r));
        tmem_ld8(tdK + lane_base + hh * kHalf, *reinterpret_cast<uint32_t(*)[8]>(rk));
        tmem_ld8(tdV + lane_base + hh * kHalf, *reinterpret_cast<uint32_t(*)[8]>(rv));
      } else if constexpr (kHalf == 16) {
        tmem_ld16(tdQ + lane_base + hh * kHalf, *reinterpret_cast<uint32_t(*)[16]>(r));
        tmem_ld16(tdK + lane_base + hh * kHalf, *reinterpret_cast<uint32_t(*)[16]>(rk));
        tmem_ld16(tdV + lane_base + hh * kHalf, *reinterpret_cast<uint32_t(*)[16]>(rv));
      } else {
        tmem_ld32(tdQ + lane_base + hh * kHalf, *reinterpret_cast<uint32_t(*)[32]>(r));
        tmem_ld32(tdK + lane_base + hh * kHalf, *reinterpret_cast<uint32_t(*)[32]>(rk));
        tmem_ld32(tdV + lane_base + hh * kHalf, *reinterpret_cast<uint32_t(*)[32]>(rv));
      }
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < (int)kHalf; e += 8) {
        const int d0 = hh * kHalf + e;
        if (d0 >= a.D) break;
        if (q < a.Lq) {
          if (nk == 1) {
            uint4 o;
            o.x = pack_bf16(__uint_as_float(r[e]) * a.scale, __uint_as_float(r[e + 1]) * a.scale);
            o.y = pack_bf16(__uint_as_float(r[e + 2]) * a.scale, __uint_as_float(r[e + 3]) * a.scale);
            o.z = pack_bf16(__uint_as_float(r[e + 4]) * a.scale, __uint_as_float(r[e + 5]) * a.scale);
            o.w = pack_bf16(__uint_as_float(r[e + 6]) * a.scale, __uint_as_float(r[e + 7]) * a.scale);
            *reinterpret_cast<uint4*>(a.dq + (int64_t)bp * a.q_sb + (int64_t)h * a.q_sh +
                                      (int64_t)q * a.q_sl + d0) = o;
          } else {
            float4* dst = reinterpret_cast<float4*>(a.dq_acc + (((int64_t)bp * a.H + h) * a.Lq + q) * a.D + d0);
            atomicAdd(dst, make_float4(__uint_as_float(r[e]), __uint_as_float(r[e + 1]),
                                       __uint_as_float(r[e + 2]), __uint_as_float(r[e + 3])));
            atomicAdd(dst + 1, make_float4(__uint_as_float(r[e + 4]), __uint_as_float(r[e + 5]),
                                           __uint_as_float(r[e + 6]), __uint_as_float(r[e + 7])));
          }
        }
        if (kglob < a.Lk) {
          const int bl = b0 + nb - 1;
          uint4 x, y;
          x.x = pack_bf16(__uint_as_float(rk[e]) * a.scale, __uint_as_float(rk[e + 1]) * a.scale);
          x.y = pack_bf16(__uint_as_float(rk[e + 2]) * a.scale, __uint_as_float(rk[e + 3]) * a.scale);
          x.z = pack_bf16(__uint_as_float(rk[e + 4]) * a.scale, __uint_as_float(rk[e + 5]) * a.scale);
          x.w = pack_bf16(__uint_as_float(rk[e + 6]) * a.scale, __uint_as_float(rk[e + 7]) * a.scale);
          y.x = pack_bf16(__uint_as_float(rv[e]), __uint_as_float(rv[e + 1]));
          y.y = pack_bf16(__uint_as_float(rv[e + 2]), __uint_as_float(rv[e + 3]));
          y.z = pack_bf16(__uint_as_float(rv[e + 4]), __uint_as_float(rv[e + 5]));
          y.w = pack_bf16(__uint_as_float(rv[e + 6]), __uint_as_float(rv[e + 7]));
          *reinterpret_cast<uint4*>(a.dk + (int64_t)bl * a.k_sb + (int64_t)h * a.k_sh +
                                    (int64_t)kglob * a.k_sl + d0) = x;
          *reinterpret_cast<uint4*>(a.dv + (int64_t)bl * a.v_sb + (int64_t)h * a.v_sh +
                                    (int64_t)kglob * a.v_sl + d0) = y;
        }
      }
    }
    if (BIAS) {  // partial[c][h][q][k0 + row] for all padded q (32-column blocks alternate by hh)
      float* dst = a.partial + ((int64_t)c * a.H + h) * Lq_pad * (int64_t)Lk_pad + k0 + row;
      for (int cbk = hh; cbk < Lq_pad / 32; cbk += 2) {
        uint32_t acc[32];
        tmem_ld32(tDB + lane_base + cbk * 32, acc);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) dst[(int64_t)(cbk * 32 + i) * Lk_pad] = __uint_as_float(acc[i]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tmem);
}

template <int DP, bool BIAS>
static cudaError_t launch_bwd_fused_t(const BwdFusedLaunch& L, cudaStream_t st) {
  auto kern = bwd_fused_kernel<DP, BIAS>;
  const size_t smem = FusedCfg<DP, BIAS>::kSmem;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int nk = (L.args.Lk + 127) / 128;
  const long long grid = (long long)L.args.H * nk * L.args.nchunks;
  if (grid == 0) return cudaSuccess;
  kern<<<(unsigned)grid, 320, smem, st>>>(L.tm_q, L.tm_k, L.tm_v, L.tm_da, L.args);
  return cudaGetLastError();
}

cudaError_t launch_bwd_fused_bf16(const BwdFusedLaunch& L, int DP, int has_bias, cudaStream_t st) {
#define EVO_FUSED_CASE(dp, bb) \
  if (DP == dp && (has_bias != 0) == bb) return launch_bwd_fused_t<dp, bb>(L, st);
  EVO_FUSED_CASE(16, false) EVO_FUSED_CASE(16, true)
  EVO_FUSED_CASE(32, false) EVO_FUSED_CASE(32, true)
  EVO_FUSED_CASE(64, false) EVO_FUSED_CASE(64, true)
#undef EVO_FUSED_CASE
  return cudaErrorInvalidValue;
}

}  // namespace evo
