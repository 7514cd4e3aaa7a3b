// evo_bwd_nb.cu — single-pass bf16 backward WITHOUT a pair bias (MSA column attention, BASELINE
// cfg 4 extra-MSA column attention, the no-bias calls of cfg 5) on sm_100a: dK, dV and dQ of one
// (head, 128-key tile) for a chunk of batch rows, in one persistent CTA, one 128 x 128 (key x
// query) block per hand-off.
//
// Same arithmetic as evo_bwd_pb.cu (P recomputed once from lse,
// dS = P ⊙ (dP − D), dV = Pᵀ dA, dK = scale dSᵀ Q, dQ = scale dS K), but without
// the Σ_b dSᵀ accumulator the tensor memory has room for a whole query tile: Sᵀ and dPᵀ are
// single N = 128 MMAs (one per K step) and the compute warps hand a full 128-query tile to the
// gradient MMAs at once — a quarter of the per-32-query hand-offs of the bias kernel, whose
// mbarrier round trips under-feed the tensor pipe.
//
// Roles (512 threads): warps 0-7 compute (warp w: TMEM lane quarter w & 3 = its 32 key rows,
// query half w >> 2 of every tile, processed as two 32-query batches); warp 8 lane 0 issues
// Sᵀ/dPᵀ, warp 10 lane 0 dV/dK/dQ, warp 9 lane 0 the TMA loads, warp 11 idles; warps 12-15
// drain dQ per tile and dK/dV per batch row (staging + per-warp TMA stores).
// Per tile T (queries t·128.., batch row b):
//   Sᵀ = K_b·Q_tᵀ, dPᵀ = V_b·dA_tᵀ                    (M = 128 keys, N = 128 queries) -> TMEM
//   Pᵀ = exp2(Sᵀ·scale·log2e − lse2), dSᵀ = Pᵀ(dPᵀ − D) -> Pᵀ (bf16) to TMEM, dSᵀ to smem
//   dV_b += Pᵀ·dA_t (TS), dK_b += dSᵀ·Q_t, dQ_t = dS·K_b   (K = 128 in 8 steps each)
// TMEM (512 cols): Sᵀ [0,128) | dPᵀ [128,256) | Pᵀ [256,320) | dV | dK | dQ  (DP each)
// SMEM: K,V x2 | Q,dA x2 | dSᵀ 2 x [128 k][128 q] (tile T in buffer T & 1) | lse2/D x2 | staging
#include <cstdio>
#include <cstdlib>

#include "evo_kernels.cuh"

namespace evo {

#ifdef EVO_TIMELINE
// Debug builds only (tools/nb_timeline.py compiles a separate library with -DEVO_TIMELINE):
// clock64 stamps of CTAs 0 and 1, 14 event kinds x 512 tiles each.
__device__ unsigned long long g_tlnb[2][14][512];
#define NTL(ev, i)                                                               \
  do {                                                                           \
    if (blockIdx.x < 2 && (i) < 512) g_tlnb[blockIdx.x][ev][i] = clock64();      \
  } while (0)
#else
#define NTL(ev, i) do { } while (0)
#endif

template <int DP>
struct NbCfg {
  static constexpr uint32_t kRowBytes = DP * 2;
  static constexpr uint32_t kTile = 128 * kRowBytes;  // one 128-row Q/K/V/dA tile
  // K/V and Q/dA ring depth: a batch row with one query tile (L <= 128) is a single hand-off,
  // so the loads of the rows ahead must already be in flight
  static constexpr int kSt = DP == 16 ? 4 : 3;
  static constexpr uint32_t oKV = 0;                        // stage s: K at +s*2*kTile, V +kTile
  static constexpr uint32_t oQA = oKV + kSt * 2 * kTile;    // stage s: Q at +s*2*kTile, dA +kTile
  static constexpr uint32_t oDS = oQA + kSt * 2 * kTile;    // 2 x 4 x [128 k][32 q] SW64 (8 KB)
  static constexpr uint32_t oVec = oDS + 65536;             // kSt x (lse2[128], D[128]) fp32
  static constexpr uint32_t oStK = oVec + kSt * 1024;  // staging: dK, dV bf16, dQ bf16|fp32
  static constexpr uint32_t oStV = oStK + kTile;
  static constexpr uint32_t oStQ = oStV + kTile;
  static constexpr uint32_t oBar = oStQ + 128 * DP * 4;
  static constexpr uint32_t kSmem = oBar + 256;
};

template <int DP>
EVO_DEV void nb_ld_cols(uint32_t taddr, uint32_t (&r)[DP]) {
  if constexpr (DP == 16) tmem_ld16(taddr, r);
  else tmem_ld32(taddr, r);
}

template <int DP>
__global__ void __launch_bounds__(512, 1)
    bwd_nb_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_da,
                  const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ CUtensorMap tm_dk,
                  const __grid_constant__ CUtensorMap tm_dv, const BwdFusedArgs a) {
  using C = NbCfg<DP>;
  static_assert(DP == 16 || DP == 32, "no-bias backward: head dim pad 16 or 32");
  constexpr uint32_t kSw = DP == 32 ? kSw64 : kSw32;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t s0 = smem_u32(smem);
  if (s0 & 1023u) __trap();
  constexpr int S = C::kSt;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::oBar);
  const uint32_t bar_kv = smem_u32(&bars[0]);           // +8 s: stage s   K,V landed (TMA)
  const uint32_t bar_in = smem_u32(&bars[S]);           // +8 s: Q,dA,vectors landed (TMA)
  const uint32_t bar_kvfree = smem_u32(&bars[2 * S]);   // +8 s: MMAs done with a K,V stage
  const uint32_t bar_infree = smem_u32(&bars[3 * S]);   // +8 s: MMAs done with a Q,dA stage
  const uint32_t bar_sp = smem_u32(&bars[4 * S]);       // Sᵀ/dPᵀ of a tile landed
  const uint32_t bar_sfree = smem_u32(&bars[4 * S + 1]);  // the 8 compute warps pulled Sᵀ/dPᵀ
  const uint32_t bar_ps = smem_u32(&bars[4 * S + 2]);     // the 8 compute warps handed Pᵀ/dSᵀ over
  const uint32_t bar_mm = smem_u32(&bars[4 * S + 3]);     // dV/dK of a tile done
  const uint32_t bar_dq = smem_u32(&bars[4 * S + 4]);     // +8: dSᵀ buffer 1   dQ MMA done
  const uint32_t bar_dqfree = smem_u32(&bars[4 * S + 6]); // the drain warps pulled a tile's dQ
  const uint32_t bar_kvdone = smem_u32(&bars[4 * S + 7]); // a batch row's last dV/dK MMA landed
  const uint32_t bar_dkvfree = smem_u32(&bars[4 * S + 8]);  // the drain warps pulled dK/dV
  const uint32_t bar_dqrow = smem_u32(&bars[4 * S + 9]);    // kloop: a batch row's dQ is final
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(&bars[4 * S + 10]);

  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int nq = (a.Lq + 127) >> 7, nk = (a.Lk + 127) >> 7;
  const int Lq_pad = nq * 128;
  const int c = (int)blockIdx.x % a.nchunks;
  const int grp = (int)blockIdx.x / a.nchunks;
  // a "group" is one (batch row, key tile) pair: its K/V stay resident while its nq query tiles
  // stream by.  kloop: the CTA walks key tiles 0..nk-1 of each of its batch rows (dQ accumulates
  // over them in TMEM); otherwise the CTA owns the single key tile ktf
  const bool kloop = a.kloop != 0;
  const int nkl = kloop ? nk : 1;
  const int ktf = kloop ? 0 : grp % nk, h = kloop ? grp : grp / nk;
  const int b0 = c * a.chunk;
  const int nb = min(a.B - b0, a.chunk);
  if (nb <= 0) return;
  const int NG = nb * nkl;  // groups
  const int NT = NG * nq;   // tiles

  if (w == 0) tmem_alloc<512>(smem_u32(tmem_slot));
  if (tid == 32) {
    for (int i = 0; i < S; ++i) {
      mbar_init(bar_kv + 8 * i, 1);
      mbar_init(bar_in + 8 * i, 1);
      mbar_init(bar_kvfree + 8 * i, 1);
      mbar_init(bar_infree + 8 * i, 1);
    }
    mbar_init(bar_dq, 1);
    mbar_init(bar_dq + 8, 1);
    mbar_init(bar_sp, 1);
    mbar_init(bar_sfree, 8);
    mbar_init(bar_ps, 8);
    mbar_init(bar_mm, 1);
    mbar_init(bar_dqfree, 4);
    mbar_init(bar_kvdone, 1);
    mbar_init(bar_dkvfree, 4);
    mbar_init(bar_dqrow, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tdP = tmem + 128, tP = tmem + 256;
  const uint32_t tdV = tmem + 320, tdK = tdV + DP, tdQ = tdK + DP;

  if (w >= 8) {
  setmaxnreg_dec<88>();
  if (w == 9) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      tma_prefetch_desc(&tm_da);
      for (int gi = 0; gi < NG; ++gi) {
        const int bi = gi / nkl, kt = kloop ? gi - bi * nkl : ktf;
        const int b = b0 + bi, kvs = gi % S;
        if (gi >= S) mbar_wait(bar_kvfree + 8 * kvs, ((gi - S) / S) & 1);
        const uint32_t kb = s0 + C::oKV + kvs * 2 * C::kTile;
        mbar_arrive_expect_tx(bar_kv + 8 * kvs, 2 * C::kTile);
        tma_load_4d(kb, &tm_k, bar_kv + 8 * kvs, 0, kt * 128, h, b);
        tma_load_4d(kb + C::kTile, &tm_v, bar_kv + 8 * kvs, 0, kt * 128, h, b);
        for (int t = 0; t < nq; ++t) {
          const int T = gi * nq + t, st = T % S;
          if (T >= S) mbar_wait(bar_infree + 8 * st, ((T - S) / S) & 1);
          NTL(11, T);  // Q/dA load issued
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
    // ------------------------------------------------------------------ Sᵀ/dPᵀ issuer (N = 128)
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, 0, 0);
      for (int T = 0; T < NT; ++T) {
        const int gi = T / nq, t = T - gi * nq, st = T % S, kvs = gi % S;
        if (T >= 1) mbar_wait(bar_sfree, (T - 1) & 1);  // the previous tile's Sᵀ/dPᵀ pulled
        mbar_wait(bar_in + 8 * st, (T / S) & 1);
        if (t == 0) mbar_wait(bar_kv + 8 * kvs, (gi / S) & 1);
        NTL(12, T);  // S issuer ready
        tc_fence_after();
        const uint32_t kb = s0 + C::oKV + kvs * 2 * C::kTile;
        const uint32_t qb = s0 + C::oQA + st * 2 * C::kTile;
#pragma unroll
        for (int kk = 0; kk < DP / 16; ++kk)
          umma_bf16(tS, make_sdesc(kb + kk * 32, 16, 8 * C::kRowBytes, kSw),
                    make_sdesc(qb + kk * 32, 16, 8 * C::kRowBytes, kSw), idesc_s, kk > 0);
#pragma unroll
        for (int kk = 0; kk < DP / 16; ++kk)
          umma_bf16(tdP, make_sdesc(kb + C::kTile + kk * 32, 16, 8 * C::kRowBytes, kSw),
                    make_sdesc(qb + C::kTile + kk * 32, 16, 8 * C::kRowBytes, kSw), idesc_s, kk > 0);
        umma_commit(bar_sp);
        NTL(0, T);  // Sᵀ/dPᵀ issued
      }
    }
  } else if (w == 10) {
    // ------------------------------------------------------------------ gradient-MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_kv = make_idesc_bf16(128, DP, 0, 1);  // dV, dK (B MN-major)
      constexpr uint32_t idesc_q = make_idesc_bf16(128, DP, 1, 1);   // dQ (A, B MN-major)
      for (int T = 0; T < NT; ++T) {
        const int gi = T / nq, t = T - gi * nq, st = T % S, kvs = gi % S, ds = T & 1;
        const int bi = gi / nkl, kt = kloop ? gi - bi * nkl : ktf;
        mbar_wait(bar_ps, T & 1);
        NTL(6, T);  // hand-off seen
        // a new group overwrites dK/dV: the drain warps must have pulled the previous ones
        if (t == 0 && gi > 0) mbar_wait(bar_dkvfree, (gi - 1) & 1);
        NTL(7, T);  // dK/dV free
        tc_fence_after();
        const uint32_t qb = s0 + C::oQA + st * 2 * C::kTile;
        const uint32_t ab = qb + C::kTile;
        const uint32_t db = s0 + C::oDS + ds * 32768;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dV += Pᵀ·dA (K = 128 queries; A = Pᵀ from TMEM)
          umma_bf16_ts(tdV, tP + kk * 8,
                       make_sdesc(ab + kk * 16 * C::kRowBytes, 16384, 8 * C::kRowBytes, kSw),
                       idesc_kv, (t > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dK += dSᵀ·Q
          umma_bf16(tdK, make_sdesc(db + (kk >> 1) * 8192 + (kk & 1) * 32, 16, 512, kSw64),
                    make_sdesc(qb + kk * 16 * C::kRowBytes, 16384, 8 * C::kRowBytes, kSw),
                    idesc_kv, (t > 0 || kk > 0) ? 1u : 0u);
        umma_commit(bar_mm);
        NTL(8, T);  // dV/dK issued
        if (t == nq - 1) umma_commit(bar_kvdone);  // the group's dK/dV are final
        // dQ = dS·K (A = the tile's dSᵀ blocks read MN-major).  kloop: accumulated over the key
        // tiles in the tile's own TMEM columns, which the drain warps must have pulled for the
        // previous batch row; otherwise one TMEM dQ the drain pulls after every tile
        if (kloop) {
          if (kt == 0 && t == 0 && bi > 0) mbar_wait(bar_dqfree, (bi - 1) & 1);
        } else if (T >= 1) {
          mbar_wait(bar_dqfree, (T - 1) & 1);
        }
        tc_fence_after();
        const uint32_t kb = s0 + C::oKV + kvs * 2 * C::kTile;
        const uint32_t tq = kloop ? tdQ + t * DP : tdQ;
        const uint32_t acc0 = kloop && kt > 0 ? 1u : 0u;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16(tq, make_sdesc(db + kk * 1024, 8192, 512, kSw64),
                    make_sdesc(kb + kk * 16 * C::kRowBytes, 16384, 8 * C::kRowBytes, kSw),
                    idesc_q, kk > 0 ? 1u : acc0);
        umma_commit(bar_dq + 8 * ds);
        NTL(9, T);  // dQ issued
        if (kloop && kt == nk - 1 && t == nq - 1) umma_commit(bar_dqrow);  // the row's dQ final
        // every reader of the Q/dA stage (Sᵀ/dPᵀ MMAs: pulled before the hand-off; dV/dK/dQ:
        // this thread) and, after a row's last tile, of the K/V stage is done once these land
        umma_commit(bar_infree + 8 * st);
        if (t == nq - 1) umma_commit(bar_kvfree + 8 * kvs);
      }
    }
  } else if (w >= 12) {
    // ------------------------------------------------------------------ drain warps
    const int qd = w & 3;
    const int row = qd * 32 + lane;  // TMEM lane: a key row (dK/dV) or a query row (dQ)
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    const uint32_t slice = (uint32_t)(qd * 32);
    constexpr uint32_t kRbB = DP * 2;
    // TMEM columns -> bf16 staging row (swizzled), 8 columns at a time (small register budget)
    auto stage_bf16 = [&](uint32_t base, uint32_t tcol, float mul) {
#pragma unroll
      for (int i = 0; i < DP / 8; ++i) {
        uint32_t r[8];
        tmem_ld8(tcol + 8 * i, r);
        tmem_wait_ld();
        st_shared_v4(base + swz_offset(row, i, kRbB),
                     pack_bf16(__uint_as_float(r[0]) * mul, __uint_as_float(r[1]) * mul),
                     pack_bf16(__uint_as_float(r[2]) * mul, __uint_as_float(r[3]) * mul),
                     pack_bf16(__uint_as_float(r[4]) * mul, __uint_as_float(r[5]) * mul),
                     pack_bf16(__uint_as_float(r[6]) * mul, __uint_as_float(r[7]) * mul));
      }
    };
    for (int T = 0; T < NT; ++T) {
      const int gi = T / nq, t = T - gi * nq;
      const int bi = gi / nkl, kt = kloop ? gi - bi * nkl : ktf;
      if (t == nq - 1) {  // the group's dK/dV, once its last dV/dK MMA landed
        mbar_wait(bar_kvdone, gi & 1);
        if (qd == 0 && lane == 0) NTL(10, T);  // dK/dV landed (drain)
        tc_fence_after();
        if (lane == 0) bulk_wait_group_read0();  // this warp's previous stores left its slices
        __syncwarp();
        stage_bf16(s0 + C::oStK, tdK + lane_base, a.scale);
        stage_bf16(s0 + C::oStV, tdV + lane_base, 1.f);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_dkvfree);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_4d(&tm_dk, s0 + C::oStK + slice * kRbB, 0, kt * 128 + (int)slice, h, b0 + bi);
          tma_store_4d(&tm_dv, s0 + C::oStV + slice * kRbB, 0, kt * 128 + (int)slice, h, b0 + bi);
          bulk_commit_group();
        }
      }
      if (kloop) {
        // the batch row's dQ of every query tile, once its last key tile's dQ MMA landed:
        // bf16 through two alternating staging halves
        if (kt == nk - 1 && t == nq - 1) {
          mbar_wait(bar_dqrow, bi & 1);
          tc_fence_after();
          for (int tq = 0; tq < nq; ++tq) {
            const uint32_t sb = s0 + C::oStQ + (tq & 1) * (128 * kRbB);
            if (lane == 0) bulk_wait_group_read<1>();  // the store from this half has left
            __syncwarp();
            stage_bf16(sb, tdQ + tq * DP + lane_base, a.scale);
            if (tq == nq - 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(bar_dqfree);  // the next row's dQ MMAs may overwrite
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_4d(&tm_dq, sb + slice * kRbB, 0, tq * 128 + (int)slice, h, b0 + bi);
              bulk_commit_group();
            }
          }
        }
        continue;
      }
      // dQ part of tile T: bf16 rows with one key tile, else this key tile's fp32 part
      // (reduce-add into the one accumulator at nk == 2, its own part otherwise)
      mbar_wait(bar_dq + 8 * (T & 1), (T >> 1) & 1);
      tc_fence_after();
      if (lane == 0) bulk_wait_group_read0();
      __syncwarp();
      if (nk == 1) {
        stage_bf16(s0 + C::oStQ, tdQ + lane_base, a.scale);
      } else {
#pragma unroll
        for (int i = 0; i < DP / 8; ++i) {
          uint32_t r[8];
          tmem_ld8(tdQ + lane_base + 8 * i, r);
          tmem_wait_ld();
          st_shared_v4(s0 + C::oStQ + swz_offset(row, 2 * i, DP * 4), r[0], r[1], r[2], r[3]);
          st_shared_v4(s0 + C::oStQ + swz_offset(row, 2 * i + 1, DP * 4), r[4], r[5], r[6], r[7]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_dqfree);  // the next tile's dQ MMA may overwrite TMEM
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        const int bq = b0 + bi;
        const uint32_t rb = nk == 1 ? kRbB : (uint32_t)(DP * 4);
        if (nk > 1 && a.dq_reduce)  // TMA .add at L2 into one fp32 accumulator (bwd_pre zeroed it)
          tma_reduce_add_4d_hint(&tm_dq, s0 + C::oStQ + slice * rb, 0, t * 128 + (int)slice, h, bq,
                                 l2_policy_evict_last());
        else
          tma_store_4d(&tm_dq, s0 + C::oStQ + slice * rb, 0, t * 128 + (int)slice, h,
                       nk == 1 ? bq : kt * a.B + bq);
        bulk_commit_group();
      }
    }
    if (lane == 0) bulk_wait_group0();
  }  // (warp 11 idles)
  } else {
    setmaxnreg_inc<168>();
    // ------------------------------------------------------------------ compute warps
    const int qd = w & 3, hq = w >> 2;  // lane quarter (key rows), query half of every tile
    const int row = qd * 32 + lane;      // key row within the tile = TMEM lane
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    const uint64_t sl2 = f2_pack(a.scale_log2, a.scale_log2);
    // hard-mask byte of this thread's key in group gi (raw: loaded a group ahead, tested late)
    auto load_keep = [&](int gi) -> uint32_t {
      if (gi >= NG) return 0u;
      const int bi = gi / nkl, kg = (kloop ? gi - bi * nkl : ktf) * 128 + row;
      if (kg >= a.Lk) return 0u;
      if (!a.mask) return 1u;
      return (uint32_t)__ldg(a.mask + (int64_t)(b0 + bi) * a.mask_s0 + (int64_t)kg * a.mask_s1);
    };
    uint32_t pd_off[4];  // this thread's row of a [128][32] bf16 SW64 dSᵀ block: 4 chunk offsets
#pragma unroll
    for (int e = 0; e < 4; ++e) pd_off[e] = swz_offset(row, e, 64);
    uint32_t keep_nx = load_keep(0);
    bool keep = false;
    for (int T = 0; T < NT; ++T) {
      const int gi = T / nq, t = T - gi * nq, st = T % S, ds = T & 1;
      if (t == 0) {
        keep = keep_nx != 0u;
        keep_nx = load_keep(gi + 1);
      }
      if (w == 0 && lane == 0) NTL(1, T);  // waits for Sᵀ/dPᵀ
      mbar_wait(bar_sp, T & 1);
      tc_fence_after();
      if (w == 0 && lane == 0) NTL(2, T);  // Sᵀ/dPᵀ landed
      mbar_wait(bar_in + 8 * st, (T / S) & 1);  // lse2 / D of this query tile visible
#pragma unroll 1
      for (int hb = 0; hb < 2; ++hb) {  // two 32-query batches of this warp's 64 queries
        const int qloc = hq * 64 + hb * 32;  // first query of the batch within the tile
        uint32_t rs[32], rd[32];
        tmem_ld32(tS + lane_base + qloc, rs);
        tmem_ld32(tdP + lane_base + qloc, rd);
        tmem_wait_ld();
        if (hb == 1) {  // this warp's Sᵀ/dPᵀ columns are in registers: the next tile may land
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_sfree);
        }
        const uint32_t vbase = s0 + C::oVec + st * 1024 + qloc * 4;
        uint32_t pk[16], dk2[16];
#pragma unroll
        for (int gq = 0; gq < 4; ++gq) {  // 8 queries per group
          // the vectors arrive negated: -lse·log2e (-inf for rows without a kept key), -D
          const uint4 l0 = ld_shared_v4(vbase + gq * 32), l1 = ld_shared_v4(vbase + gq * 32 + 16);
          const uint4 d0 = ld_shared_v4(vbase + 512 + gq * 32), d1 = ld_shared_v4(vbase + 512 + gq * 32 + 16);
          const uint32_t nl[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
          const uint32_t nd[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = gq * 8 + 2 * e;
            const uint64_t nl2 = ((uint64_t)nl[2 * e + 1] << 32) | nl[2 * e];
            const uint64_t nd2 = ((uint64_t)nd[2 * e + 1] << 32) | nd[2 * e];
            const uint64_t x = f2_fma(((uint64_t)rs[i + 1] << 32) | rs[i], sl2, nl2);
            float x0, x1;
            f2_unpack(x, x0, x1);
            const float p0 = fast_exp2(x0), p1 = fast_exp2(x1);
            const uint64_t dd = f2_mul(f2_pack(p0, p1), f2_add(((uint64_t)rd[i + 1] << 32) | rd[i], nd2));
            float ds0, ds1;
            f2_unpack(dd, ds0, ds1);
            pk[i / 2] = pack_bf16(p0, p1);
            dk2[i / 2] = pack_bf16(ds0, ds1);
          }
        }
        // hard mask (R5): a masked key row has P = dS = 0 (per thread; whole warps skip it)
        if (__any_sync(0xffffffffu, !keep) && !keep) {
#pragma unroll
          for (int i = 0; i < 16; ++i) { pk[i] = 0u; dk2[i] = 0u; }
        }
        if (hb == 0) {
          if (w == 0 && lane == 0) NTL(3, T);  // first batch's math done
          // before overwriting: Pᵀ is read by dV of the previous tile; this tile's dSᵀ buffer
          // (T & 1) by tile T-2's dQ MMA
          if (T >= 1) mbar_wait(bar_mm, (T - 1) & 1);
          if (T >= 2) mbar_wait(bar_dq + 8 * ds, ((T - 2) >> 1) & 1);
          tc_fence_after();
          if (w == 0 && lane == 0) NTL(4, T);  // Pᵀ slot / dSᵀ buffer free
        }
        // Pᵀ -> TMEM (16 packed columns for these 32 queries); dSᵀ rows -> smem block qloc / 32
        tmem_st16(tP + lane_base + qloc / 2, pk);
        {
          const uint32_t db = s0 + C::oDS + ds * 32768 + (qloc >> 5) * 8192;
#pragma unroll
          for (int e = 0; e < 4; ++e)
            st_shared_v4(db + pd_off[e], dk2[4 * e], dk2[4 * e + 1], dk2[4 * e + 2], dk2[4 * e + 3]);
        }
      }
      tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_ps);
      if (w == 0 && lane == 0) NTL(5, T);  // hand-off
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tmem);
}

#ifdef EVO_TIMELINE
extern "C" int evo_debug_nb_timeline_copy(void* dst, size_t bytes) {
  if (bytes > sizeof(g_tlnb)) bytes = sizeof(g_tlnb);
  return (int)cudaMemcpyFromSymbol(dst, g_tlnb, bytes);
}
#endif

template <int DP>
static cudaError_t launch_bwd_nb_t(const BwdFusedLaunch& L, cudaStream_t st) {
  auto kern = bwd_nb_kernel<DP>;
  const size_t smem = NbCfg<DP>::kSmem;
  cudaError_t e = set_smem_once(kern, smem);
  if (e != cudaSuccess) return e;
  const int nk = (L.args.Lk + 127) / 128;
  const long long grid = (long long)L.args.H * (L.args.kloop ? 1 : nk) * L.args.nchunks;
  if (grid == 0) return cudaSuccess;
  kern<<<(unsigned)grid, 512, smem, st>>>(L.tm_q, L.tm_k, L.tm_v, L.tm_da, L.tm_dq, L.tm_dk,
                                          L.tm_dv, L.args);
  return cudaGetLastError();
}

cudaError_t launch_bwd_nb_bf16(const BwdFusedLaunch& L, int DP, cudaStream_t st) {
  if (DP == 16) return launch_bwd_nb_t<16>(L, st);
  if (DP == 32) return launch_bwd_nb_t<32>(L, st);
  return cudaErrorInvalidValue;
}

}  // namespace evo
