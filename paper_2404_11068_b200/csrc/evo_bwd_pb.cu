// evo_bwd_pb.cu — single-pass bf16 backward WITH a shared pair bias, Lq <= 384 (MSA row
// attention with pair bias, triangle attention around the starting / ending node: BASELINE
// cfg 1-3 and 5 and the block's three bias modules) on sm_100a: dK, dV, dQ and Σ_b dSᵀ (the
// pair-bias gradient) of one (head, 128-key tile) for a chunk of batch rows, in one persistent
// CTA.
//
// The backward of the pair-bias attention (P recomputed once from lse,
// dS = P ⊙ (dP − D), dV = Pᵀ dA, dK = scale dSᵀ Q, dQ = scale dS K, dbias = Σ_b dS over the
// broadcast axis), with the hand-off structure of the no-bias kernel
// (evo_bwd_nb.cu): 64-query hand-offs (N = 64 Sᵀ/dPᵀ MMAs, two per 128-query tile) processed by
// all eight compute warps at once (round 2 replaced a design with two ping-pong warpgroups on
// 32-query sub-tiles, whose mbarrier round trips under-fed the tensor pipe).  Σ_b dSᵀ of the key tile stays in
// TMEM (fp32, read-modify-write by the owning thread), 256 columns; that leaves room for exactly
// one 64-query Sᵀ/dPᵀ slot, one Pᵀ slot and dV/dK/dQ.
//
// Roles (512 threads): warps 0-7 compute (warp w: TMEM lane quarter w & 3 = its 32 key rows,
// query half w >> 2 = 32 of the 64 queries of every hand-off); warp 8 lane 0 issues Sᵀ/dPᵀ,
// warp 10 lane 0 dV/dK/dQ, warp 9 lane 0 the TMA loads, warp 11 idles; warps 12-15 drain dQ per
// tile and dK/dV per batch row (staging + per-warp TMA stores).
// Per hand-off j (queries 64 s.. of tile T = j / 2, s = j & 1, batch row b):
//   Sᵀ = K_b·Q_jᵀ, dPᵀ = V_b·dA_jᵀ                    (M = 128 keys, N = 64 queries) -> TMEM
//   Pᵀ = exp2(Sᵀ·scale·log2e + biasᵀ·log2e − lse2), dSᵀ = Pᵀ(dPᵀ − D), Σ_b dSᵀ += dSᵀ (TMEM)
//   -> Pᵀ (bf16) to TMEM, dSᵀ to smem blocks 2s, 2s+1 of the tile's buffer
//   dV_b += Pᵀ·dA_j (TS), dK_b += dSᵀ·Q_j  (K = 64 in 4 steps each); after s = 1: dQ_T = dS·K_b
// TMEM (512 cols): Σ_b dSᵀ [0,256) | Sᵀ [256,320) | dPᵀ [320,384) | Pᵀ [384,416) | dV | dK | dQ
// SMEM: biasᵀ resident [128 k][256 q] | K,V x2 | Q,dA x2 | dSᵀ 2 x [128 k][128 q] | lse2/D x2 |
//       staging | barriers
#include <cstdio>
#include <cstdlib>

#include "evo_kernels.cuh"

namespace evo {

#ifdef EVO_TIMELINE
// Debug builds only (tools/pb_timeline.py compiles a separate library with -DEVO_TIMELINE):
// clock64 stamps of CTAs 0 and 1, 16 event kinds x 512 hand-offs each.
__device__ unsigned long long g_tlpb[2][16][512];
#define PTL(ev, i)                                                               \
  do {                                                                           \
    if (blockIdx.x < 2 && (i) < 512) g_tlpb[blockIdx.x][ev][i] = clock64();      \
  } while (0)
#else
#define PTL(ev, i) do { } while (0)
#endif

// BIG: a shared bias with 256 < Lq <= 384 (BASELINE cfg 5, N_res = 384): the resident biasᵀ grows
// to [128 k][384 q] and the dSᵀ tile buffer is single (smem 226 KB); Σ_b dSᵀ stays in TMEM for the
// first 256 queries and the last query tile's Σ comes from a second, Σ-only launch of this kernel
// (sigma_only, first query tile t0 = 2: Sᵀ/dPᵀ MMAs and the compute warps only)
template <int DP, bool BIG = false>
struct PbCfg {
  static constexpr uint32_t kRowBytes = DP * 2;
  static constexpr uint32_t kTile = 128 * kRowBytes;  // one 128-row Q/K/V/dA tile
  static constexpr uint32_t oBias = 0;  // [128 k][256 | 384 q] bf16, 4 | 6 x [128][64] SW128
  static constexpr uint32_t oKV = oBias + (BIG ? 98304 : 65536);  // stage s: K +s*2*kTile, V +kTile
  static constexpr uint32_t oQA = oKV + 4 * kTile;     // stage s: Q at +s*2*kTile, dA +kTile
  static constexpr uint32_t oDS = oQA + 4 * kTile;     // (2 | 1) x 4 x [128 k][32 q] SW64 (8 KB)
  static constexpr uint32_t oVec = oDS + (BIG ? 32768 : 65536);  // 2 x (lse2[128], D[128]) fp32
  static constexpr uint32_t oStK = oVec + 2048;        // staging: dK, dV bf16, dQ bf16|fp32
  static constexpr uint32_t oStV = oStK + kTile;
  static constexpr uint32_t oStQ = oStV + kTile;
  static constexpr uint32_t oBar = oStQ + 128 * DP * 4;
  static constexpr uint32_t kSmem = oBar + 256;
};

template <int DP, bool BIG>
__global__ void __launch_bounds__(512, 1)
    bwd_pb_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_da,
                  const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ CUtensorMap tm_dk,
                  const __grid_constant__ CUtensorMap tm_dv, const __grid_constant__ CUtensorMap tm_b,
                  const BwdFusedArgs a) {
  using C = PbCfg<DP, BIG>;
  static_assert(DP == 16 || DP == 32, "pair-bias backward: head dim pad 16 or 32");
  static_assert(C::kSmem <= 232448, "pair-bias backward: shared memory");
  constexpr uint32_t kSw = DP == 32 ? kSw64 : kSw32;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t s0 = smem_u32(smem);
  if (s0 & 1023u) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::oBar);
  const uint32_t bar_kv = smem_u32(&bars[0]);        // +8: stage 1   K,V landed (TMA)
  const uint32_t bar_in = smem_u32(&bars[2]);        // +8: stage 1   Q,dA,vectors landed (TMA)
  const uint32_t bar_kvfree = smem_u32(&bars[4]);    // +8            MMAs done with a K,V stage
  const uint32_t bar_infree = smem_u32(&bars[6]);    // +8            MMAs done with a Q,dA stage
  const uint32_t bar_sp = smem_u32(&bars[8]);        // Sᵀ/dPᵀ of a hand-off landed
  const uint32_t bar_sfree = smem_u32(&bars[9]);     // the 8 compute warps pulled Sᵀ/dPᵀ
  const uint32_t bar_ps = smem_u32(&bars[10]);       // the 8 compute warps handed Pᵀ/dSᵀ over
  // the dV MMAs reading the Pᵀ columns of query half 0 / 1 of a hand-off are done
  const uint32_t bar_mm0 = smem_u32(&bars[11]);
  const uint32_t bar_mm1 = smem_u32(&bars[12]);
  const uint32_t bar_dq = smem_u32(&bars[13]);       // +8: dSᵀ buffer 1   dQ MMA of a tile done
  const uint32_t bar_dqfree = smem_u32(&bars[15]);   // the drain warps pulled a tile's dQ
  const uint32_t bar_kvdone = smem_u32(&bars[16]);   // a batch row's last dV/dK MMA landed
  const uint32_t bar_dkvfree = smem_u32(&bars[17]);  // the drain warps pulled a row's dK/dV
  const uint32_t bar_bias = smem_u32(&bars[18]);     // the bias tiles of the prologue landed
  // dq_pair (+8: buffer 1): the peer's half of a dQ tile landed in this CTA's receive buffer
  // (the 2 keeping warps' expect-tx arrivals + the peer's st.async bytes) / the peer released its
  // receive buffer (2 remote arrivals)
  const uint32_t bar_recv = smem_u32(&bars[19]);
  const uint32_t bar_recvfree = smem_u32(&bars[21]);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(&bars[23]);

  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int nq_all = (a.Lq + 127) >> 7, nk = (a.Lk + 127) >> 7;
  const int Lq_pad = nq_all * 128, Lk_pad = nk * 128;
  // query tiles t0 .. nq_all-1 (t0 = 2 in the Σ-only pass of a BIG call: Σ_b dSᵀ of the last
  // query tile, no gradients); every loop runs t over [0, nq) with query tile t0 + t
  const int t0 = a.t0, nq = nq_all - t0;
  const bool sig_only = a.sigma_only != 0;
  // dq_pair: the cluster's two CTAs are key tiles 0 and 1 of one (h, chunk); otherwise the grid
  // is (h, key tile, chunk) with the chunk fastest
  const bool pair = a.dq_pair != 0;
  const int rank = pair ? (int)cluster_ctarank() : 0;
  const int cid = pair ? (int)blockIdx.x >> 1 : (int)blockIdx.x;
  const int c = cid % a.nchunks;
  const int grp = cid / a.nchunks;
  const int kt = pair ? rank : grp % nk, h = pair ? grp : grp / nk;
  const int k0 = kt * 128;
  const int b0 = c * a.chunk;
  const int nb = min(a.B - b0, a.chunk);
  if (nb <= 0) return;
  const int NT = nb * nq;  // 128-query tiles
  const int J = NT * 2;    // 64-query hand-offs

  if (w == 0) tmem_alloc<512>(smem_u32(tmem_slot));
  if (tid == 32) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_kv + 8 * i, 1);
      mbar_init(bar_in + 8 * i, 1);
      mbar_init(bar_kvfree + 8 * i, 1);
      // the Σ-only pass frees a Q/dA/vector stage when the 8 compute warps are done with the
      // tile's lse2/D vectors (the gradient issuer's dQ commit does it otherwise)
      mbar_init(bar_infree + 8 * i, sig_only ? 8 : 1);
      mbar_init(bar_dq + 8 * i, 1);
    }
    mbar_init(bar_sp, 1);
    mbar_init(bar_sfree, 8);
    mbar_init(bar_ps, 8);
    mbar_init(bar_mm0, 1);
    mbar_init(bar_mm1, 1);
    mbar_init(bar_dqfree, 4);
    mbar_init(bar_kvdone, 1);
    mbar_init(bar_dkvfree, 4);
    mbar_init(bar_bias, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_recv + 8 * i, 2);
      mbar_init(bar_recvfree + 8 * i, 2);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  if (pair) cluster_sync_all();  // both CTAs' barriers initialised before any remote arrival
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tSig = tmem, tS = tmem + 256, tdP = tmem + 320, tP = tmem + 384;
  const uint32_t tdV = tmem + 416, tdK = tdV + DP, tdQ = tdK + DP;

  if (w >= 8) {
  setmaxnreg_dec<88>();
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
          PTL(11, 2 * T);  // Q/dA load issued
          const uint32_t qb = s0 + C::oQA + st * 2 * C::kTile;
          const uint32_t bar = bar_in + 8 * st;
          mbar_arrive_expect_tx(bar, 2 * C::kTile + 1024);
          tma_load_4d(qb, &tm_q, bar, 0, (t0 + t) * 128, h, b);
          tma_load_4d(qb + C::kTile, &tm_da, bar, 0, (t0 + t) * 128, h, b);
          const int64_t vrow = ((int64_t)b * a.H + h) * Lq_pad + (t0 + t) * 128;
          bulk_load(s0 + C::oVec + st * 1024, a.lse2 + vrow, 512, bar);
          bulk_load(s0 + C::oVec + st * 1024 + 512, a.Dvec + vrow, 512, bar);
        }
      }
    }
  } else if (w == 8) {
    // ------------------------------------------------------------------ Sᵀ/dPᵀ issuer (N = 64)
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, 0, 0);
      for (int j = 0; j < J; ++j) {
        const int T = j >> 1, s = j & 1, bi = T / nq, t = T - bi * nq, st = T & 1, kvs = bi & 1;
        if (j >= 1) mbar_wait(bar_sfree, (j - 1) & 1);  // the previous hand-off's Sᵀ/dPᵀ pulled
        if (s == 0) mbar_wait(bar_in + 8 * st, (T >> 1) & 1);
        if (s == 0 && t == 0) mbar_wait(bar_kv + 8 * kvs, (bi >> 1) & 1);
        PTL(12, j);  // S issuer ready
        tc_fence_after();
        const uint32_t kb = s0 + C::oKV + kvs * 2 * C::kTile;
        const uint32_t qb = s0 + C::oQA + st * 2 * C::kTile + s * 64 * C::kRowBytes;
#pragma unroll
        for (int kk = 0; kk < DP / 16; ++kk)
          umma_bf16(tS, make_sdesc(kb + kk * 32, 16, 8 * C::kRowBytes, kSw),
                    make_sdesc(qb + kk * 32, 16, 8 * C::kRowBytes, kSw), idesc_s, kk > 0);
#pragma unroll
        for (int kk = 0; kk < DP / 16; ++kk)
          umma_bf16(tdP, make_sdesc(kb + C::kTile + kk * 32, 16, 8 * C::kRowBytes, kSw),
                    make_sdesc(qb + C::kTile + kk * 32, 16, 8 * C::kRowBytes, kSw), idesc_s, kk > 0);
        umma_commit(bar_sp);
        PTL(0, j);  // Sᵀ/dPᵀ issued
        if (sig_only && s == 1 && t == nq - 1)  // no gradient MMAs in the Σ-only pass: the
          umma_commit(bar_kvfree + 8 * kvs);    // Sᵀ/dPᵀ MMAs are K/V's last readers
      }
    }
  } else if (w == 10) {
    // ------------------------------------------------------------------ gradient-MMA issuer
    if (lane == 0 && !sig_only) {
      constexpr uint32_t idesc_kv = make_idesc_bf16(128, DP, 0, 1);  // dV, dK (B MN-major)
      constexpr uint32_t idesc_q = make_idesc_bf16(128, DP, 1, 1);   // dQ (A, B MN-major)
      for (int j = 0; j < J; ++j) {
        const int T = j >> 1, s = j & 1, bi = T / nq, t = T - bi * nq, st = T & 1, kvs = bi & 1;
        const int ds = T & 1;
        mbar_wait(bar_ps, j & 1);
        PTL(6, j);  // hand-off seen
        // a new batch row overwrites dK/dV: the drain warps must have pulled the previous ones
        if (t == 0 && s == 0 && bi > 0) mbar_wait(bar_dkvfree, (bi - 1) & 1);
        PTL(7, j);  // dK/dV free
        tc_fence_after();
        const uint32_t qb = s0 + C::oQA + st * 2 * C::kTile;
        const uint32_t ab = qb + C::kTile;
        const uint32_t db = s0 + C::oDS + (BIG ? 0 : ds) * 32768;
        // dV += Pᵀ·dA (K = the hand-off's 64 queries; A = Pᵀ from TMEM): K steps 0,1 read the
        // Pᵀ columns of query half 0, steps 2,3 of half 1 — one commit each, so each half of the
        // next hand-off may overwrite its columns as soon as they are consumed
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const int q16 = s * 4 + kk;  // 16-query step within the tile
          umma_bf16_ts(tdV, tP + kk * 8,
                       make_sdesc(ab + q16 * 16 * C::kRowBytes, 16384, 8 * C::kRowBytes, kSw),
                       idesc_kv, (t > 0 || s > 0 || kk > 0) ? 1u : 0u);
          if (kk == 1) umma_commit(bar_mm0);
        }
        umma_commit(bar_mm1);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {  // dK += dSᵀ·Q
          const int q16 = s * 4 + kk;
          umma_bf16(tdK, make_sdesc(db + (q16 >> 1) * 8192 + (q16 & 1) * 32, 16, 512, kSw64),
                    make_sdesc(qb + q16 * 16 * C::kRowBytes, 16384, 8 * C::kRowBytes, kSw),
                    idesc_kv, (t > 0 || s > 0 || kk > 0) ? 1u : 0u);
        }
        PTL(8, j);  // dV/dK issued
        if (s == 0) continue;
        if (t == nq - 1) umma_commit(bar_kvdone);  // the row's dK/dV are final
        // dQ = dS·K over the whole tile (A = its 4 dSᵀ blocks read MN-major); the drain warps
        // must have pulled the previous tile's dQ out of TMEM
        if (T >= 1) mbar_wait(bar_dqfree, (T - 1) & 1);
        tc_fence_after();
        const uint32_t kb = s0 + C::oKV + kvs * 2 * C::kTile;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16(tdQ, make_sdesc(db + kk * 1024, 8192, 512, kSw64),
                    make_sdesc(kb + kk * 16 * C::kRowBytes, 16384, 8 * C::kRowBytes, kSw),
                    idesc_q, kk > 0 ? 1u : 0u);
        umma_commit(bar_dq + 8 * (BIG ? 0 : ds));
        PTL(9, j);  // dQ issued
        // every reader of the Q/dA stage (Sᵀ/dPᵀ MMAs: pulled before the hand-off; dV/dK/dQ:
        // this thread) and, after a row's last tile, of the K/V stage is done once these land
        umma_commit(bar_infree + 8 * st);
        if (t == nq - 1) umma_commit(bar_kvfree + 8 * kvs);
      }
    }
  } else if (w >= 12 && !sig_only) {
    // ------------------------------------------------------------------ drain warps
    const int qd = w & 3;
    const int row = qd * 32 + lane;  // TMEM lane: a key row (dK/dV) or a query row (dQ)
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    const uint32_t slice = (uint32_t)(qd * 32);
    constexpr uint32_t kRbB = DP * 2;
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
    constexpr uint32_t kHalfRows = 32 * DP * 4;  // bytes of one warp's 32 fp32 dQ rows
    if (pair && (qd >> 1) == rank && lane == 0) {  // the first two receive phases (tiles 0, 1)
      mbar_arrive_expect_tx(bar_recv, kHalfRows);
      mbar_arrive_expect_tx(bar_recv + 8, kHalfRows);
    }
    for (int T = 0; T < NT; ++T) {
      const int bi = T / nq, t = T - bi * nq;
      if (t == nq - 1) {  // the batch row's dK/dV, once its last dV/dK MMA landed
        mbar_wait(bar_kvdone, bi & 1);
        if (qd == 0 && lane == 0) PTL(10, 2 * T + 1);  // dK/dV landed (drain)
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
          tma_store_4d(&tm_dk, s0 + C::oStK + slice * kRbB, 0, k0 + (int)slice, h, b0 + bi);
          tma_store_4d(&tm_dv, s0 + C::oStV + slice * kRbB, 0, k0 + (int)slice, h, b0 + bi);
          bulk_commit_group();
        }
      }
      if (pair) {
        // dQ of tile T = dQ_0 + dQ_1 over the cluster, split by query halves: rank 0 stores
        // queries 0-63 of the tile, rank 1 queries 64-127.  The drain warps of the other half
        // send their fp32 rows into the peer's receive buffer (double-buffered by T & 1, 64 rows,
        // swizzled like the fp32 staging); the keeping warps add the peer's rows to their own in
        // the fixed order dQ_0 + dQ_1, scale, and store bf16 in place from the receive buffer.
        if (BIG) mbar_wait(bar_dq, T & 1);
        else mbar_wait(bar_dq + 8 * (T & 1), (T >> 1) & 1);
        tc_fence_after();
        uint32_t r[DP];
        if constexpr (DP == 16) tmem_ld16(tdQ + lane_base, r);
        else tmem_ld32(tdQ + lane_base, r);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_dqfree);  // the next tile's dQ MMA may overwrite TMEM
        if (lane == 0 && qd == 0) PTL(13, 2 * T + 1);  // drain: own dQ pulled (qd 0)
        if (lane == 0 && qd == 2) PTL(12, 2 * T + 1);  // drain: own dQ pulled (qd 2)
        const int buf = T & 1;
        const int hrow = (qd & 1) * 32 + lane;  // row within the 64-query half
        const uint32_t rbuf = s0 + C::oStQ + buf * (64 * DP * 4);
        if ((qd >> 1) != rank) {  // the peer keeps these rows: send them
          if (T >= 2) mbar_wait_cluster(bar_recvfree + 8 * buf, ((T - 2) >> 1) & 1);
          const uint32_t dst = mapa_shared(rbuf, (uint32_t)(rank ^ 1));
          const uint32_t rbar = mapa_shared(bar_recv + 8 * buf, (uint32_t)(rank ^ 1));
#pragma unroll
          for (int i = 0; i < DP / 4; ++i)
            st_async_v4(dst + swz_offset(hrow, i, DP * 4), r[4 * i], r[4 * i + 1], r[4 * i + 2],
                        r[4 * i + 3], rbar);
        } else {
          mbar_wait_cluster(bar_recv + 8 * buf, (T >> 1) & 1);
          uint32_t pk[DP / 2];
#pragma unroll
          for (int i = 0; i < DP / 4; ++i) {
            const uint4 o = ld_shared_v4(rbuf + swz_offset(hrow, i, DP * 4));
            const uint32_t ov[4] = {o.x, o.y, o.z, o.w};
            // own + peer in key-tile order (rank 0's dQ first)
#pragma unroll
            for (int e = 0; e < 4; e += 2) {
              const float m0 = __uint_as_float(r[4 * i + e]), p0 = __uint_as_float(ov[e]);
              const float m1 = __uint_as_float(r[4 * i + e + 1]), p1 = __uint_as_float(ov[e + 1]);
              const float s0f = (rank == 0 ? m0 + p0 : p0 + m0) * a.scale;
              const float s1f = (rank == 0 ? m1 + p1 : p1 + m1) * a.scale;
              pk[2 * i + e / 2] = pack_bf16(s0f, s1f);
            }
          }
          // the receive rows are in registers: arm the buffer's next phase (tile T + 2) and
          // release the buffer to the peer right away
          __syncwarp();
          if (lane == 0) {
            if (T + 2 < NT) mbar_arrive_expect_tx(bar_recv + 8 * buf, kHalfRows);
            mbar_arrive_remote(mapa_shared(bar_recvfree + 8 * buf, (uint32_t)(rank ^ 1)));
          }
          // this thread's query row of dq, bf16, straight to global memory (16-B stores)
          const int q = t * 128 + qd * 32 + lane;
          if (q < a.Lq) {
            __nv_bfloat16* dqr = a.dq + (int64_t)(b0 + bi) * a.q_sb + (int64_t)h * a.q_sh + (int64_t)q * a.q_sl;
#pragma unroll
            for (int i = 0; i < DP / 8; ++i)  // D % 8 == 0 and 16-B aligned rows (use_dq_pair)
              if (8 * i < a.D)
                *reinterpret_cast<uint4*>(dqr + 8 * i) = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
          }
        }
        if (lane == 0 && qd == 0) PTL(11, 2 * T + 1);  // drain: exchange done (qd 0)
        if (lane == 0 && qd == 2) PTL(10, 2 * T);      // drain: exchange done (qd 2)
        continue;
      }
      // dQ of tile T: bf16 rows with one key tile, else this key tile's fp32 part (reduce-add
      // into the one accumulator at nk == 2, its own part otherwise)
      if (BIG) mbar_wait(bar_dq, T & 1);
      else mbar_wait(bar_dq + 8 * (T & 1), (T >> 1) & 1);
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
    const int qd = w & 3, hq = w >> 2;  // lane quarter (key rows), query half of every hand-off
    const int row = qd * 32 + lane;      // key row within the tile = TMEM lane
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    const uint32_t sBias = s0 + C::oBias;
    // biasᵀ[k][q] = bias[h, q, k0 + k] for q < Lq, k0 + k < Lk; 0 elsewhere (TMA zero fill:
    // padding must be finite, it meets zero P/dA rows in the MMAs).  Resident layout: Lq_pad / 64
    // segments of [128 k][64 q] with 128-B rows, 16-B chunks XOR-swizzled by k & 7 (the TMA 128-B
    // swizzle), so a q-contiguous (end-node) bias lands there straight from TMA, and a
    // k-contiguous one is staged [q][64 k] x 2 in the (not yet used) dSᵀ buffers and transposed
    // 8 x 8 blocks at a time by ldmatrix + stmatrix.trans (conflict-free both ways).
    if (tid == 0) {
      if (a.bmode == 2) {
        mbar_arrive_expect_tx(bar_bias, (uint32_t)(Lq_pad / 64) * 16384u);
        for (int sg = 0; sg < Lq_pad / 64; ++sg)
          tma_load_4d(sBias + sg * 16384, &tm_b, bar_bias, sg * 64, k0, h, 0);
      } else if (!BIG) {
        mbar_arrive_expect_tx(bar_bias, 65536u);  // two [256 q][64 k] boxes (zero-filled past Lq)
        tma_load_4d(s0 + C::oDS, &tm_b, bar_bias, k0, 0, h, 0);
        tma_load_4d(s0 + C::oDS + 32768, &tm_b, bar_bias, k0 + 64, 0, h, 0);
      }
    }
    if (a.bmode == 2 || !BIG) mbar_wait(bar_bias, 0);
    // k-contiguous: one pass over all queries ([256 q][64 k] x 2 staged), or for BIG passes of
    // 128 queries ([128 q][64 k] x 2 = the single 32 KB dSᵀ buffer)
    const int npass = a.bmode != 2 ? (BIG ? Lq_pad / 128 : 1) : 0;
    for (int ps = 0; ps < npass; ++ps) {
      const int qb0 = BIG ? ps * 128 : 0;                // first query of the pass
      const int nq8 = BIG ? 16 : Lq_pad / 8;            // 8-query blocks in the pass
      const uint32_t kbox = BIG ? 16384u : 32768u;      // staged [q][64 k] box bytes
      if (BIG) {
        if (tid == 0) {
          mbar_arrive_expect_tx(bar_bias, 32768u);
          tma_load_4d(s0 + C::oDS, &tm_b, bar_bias, k0, qb0, h, 0);
          tma_load_4d(s0 + C::oDS + 16384, &tm_b, bar_bias, k0 + 64, qb0, h, 0);
        }
        mbar_wait(bar_bias, ps & 1);
      }
      const int mi = lane >> 3, ri = lane & 7;
      for (int gi = w; gi < nq8 * 4; gi += 8) {  // x4 group: q block q8, k blocks 4 kk..4 kk+3
        const int q8l = gi >> 2, k8 = (gi & 3) * 4 + mi;
        const int q8 = qb0 / 8 + q8l;
        const uint32_t ql = (uint32_t)(q8l * 8 + ri);
        const uint32_t src = s0 + C::oDS + (uint32_t)(k8 >> 3) * kbox + ql * 128u +
                             ((((uint32_t)k8 & 7u) ^ (ql & 7u)) << 4);
        uint32_t r0, r1, r2, r3;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                     : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                     : "r"(src));
        const uint32_t k = (uint32_t)(k8 * 8 + ri);
        const uint32_t dst = sBias + (uint32_t)(q8 >> 3) * 16384u + k * 128u +
                             ((((uint32_t)q8 & 7u) ^ (k & 7u)) << 4);
        asm volatile("stmatrix.sync.aligned.m8n8.x4.trans.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(dst),
                     "r"(r0), "r"(r1), "r"(r2), "r"(r3)
                     : "memory");
      }
      if (BIG) named_bar_sync(1, 256);  // the staging is reloaded by the next pass
    }
    named_bar_sync(1, 256);  // the staging (dSᵀ buffers) is free and the resident bias complete

    const uint64_t sl2 = f2_pack(a.scale_log2, a.scale_log2);
    const uint64_t l2e2 = f2_pack(kLog2e, kLog2e);
    const int kglob = k0 + row;
    // hard-mask bits of this thread's key for batch rows bi..bi+31: all 32 byte loads in flight
    // together, once per 32 rows (a load per row is consumed right behind its issue)
    auto load_keep_word = [&](int bi) -> uint32_t {
      if (kglob >= a.Lk) return 0u;
      if (!a.mask) return ~0u;
      uint32_t v[32];
#pragma unroll
      for (int x = 0; x < 32; ++x)
        v[x] = bi + x < nb ? (uint32_t)__ldg(a.mask + (int64_t)(b0 + bi + x) * a.mask_s0 + (int64_t)kglob * a.mask_s1) : 0u;
      uint32_t wd = 0u;
#pragma unroll
      for (int x = 0; x < 32; ++x) wd |= (v[x] != 0u ? 1u : 0u) << x;
      return wd;
    };
    uint32_t pd_off[4];  // this thread's row of a [128][32] bf16 SW64 dSᵀ block: 4 chunk offsets
#pragma unroll
    for (int e = 0; e < 4; ++e) pd_off[e] = swz_offset(row, e, 64);
    uint32_t keep_word = 0u;
    bool keep = false;
    int bi = 0, t = 0;  // coordinates of hand-off j (kept incrementally: no divisions in the loop)
    for (int j = 0; j < J; ++j) {
      const int T = j >> 1, s = j & 1, st = T & 1, ds = T & 1;
      if (t == 0 && s == 0) {
        if ((bi & 31) == 0) keep_word = load_keep_word(bi);
        keep = (keep_word >> (bi & 31)) & 1u;
      }
      const int qt = s * 64 + hq * 32;  // this warp's first query within the tile
      const int qcol = t * 128 + qt;    // its Σ column (query tiles relative to t0)
      const int qabs = (t0 + t) * 128 + qt;  // ... and its query in the padded range
      if (w == 0 && lane == 0) PTL(1, j);  // waits for Sᵀ/dPᵀ
      mbar_wait(bar_sp, j & 1);
      tc_fence_after();
      if (w == 0 && lane == 0) PTL(2, j);  // Sᵀ/dPᵀ landed
      uint32_t rs[32], rd[32], acc[32];
      tmem_ld32(tS + lane_base + hq * 32, rs);
      tmem_ld32(tdP + lane_base + hq * 32, rd);
      // Σ_b dSᵀ so far for these 32 columns (this thread's lane, last written a batch row ago)
      // BIG main pass: the last query tile's Σ is the Σ-only pass's
      const bool do_sig = !BIG || sig_only || t < 2;
      if (do_sig && bi > 0) tmem_ld32(tSig + lane_base + qcol, acc);
      tmem_wait_ld();
      if (w == 0 && lane == 0) PTL(14, j);  // Sᵀ/dPᵀ/Σ in registers
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_sfree);  // the next hand-off's Sᵀ/dPᵀ may land
      mbar_wait(bar_in + 8 * st, (T >> 1) & 1);  // lse2 / D of this query tile visible
      if (w == 0 && lane == 0) PTL(13, j);  // vectors visible
      const uint32_t vbase = s0 + C::oVec + st * 1024 + qt * 4;
      uint32_t pk[16], dk2[16];
#pragma unroll
      for (int gq = 0; gq < 4; ++gq) {  // 8 queries per group
        // the vectors arrive negated: -lse·log2e (-inf for rows without a kept key), -D
        const uint4 l0 = ld_shared_v4(vbase + gq * 32), l1 = ld_shared_v4(vbase + gq * 32 + 16);
        const uint4 d0 = ld_shared_v4(vbase + 512 + gq * 32), d1 = ld_shared_v4(vbase + 512 + gq * 32 + 16);
        const uint32_t nl[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
        const uint32_t nd[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
        const uint32_t cq = (uint32_t)(qabs >> 3) + gq;  // 8-query chunk of the resident biasᵀ
        const uint4 bv = ld_shared_v4(sBias + (cq >> 3) * 16384u + row * 128u + (((cq & 7u) ^ (row & 7u)) << 4));
        const uint32_t bu[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int i = gq * 8 + 2 * e;
          const uint64_t nl2 = ((uint64_t)nl[2 * e + 1] << 32) | nl[2 * e];
          const uint64_t nd2 = ((uint64_t)nd[2 * e + 1] << 32) | nd[2 * e];
          uint64_t x = f2_fma(bf16x2_to_f2(bu[e]), l2e2, nl2);
          x = f2_fma(((uint64_t)rs[i + 1] << 32) | rs[i], sl2, x);
          float x0, x1;
          f2_unpack(x, x0, x1);
          // hard mask (R5): a masked key row has P = dS = 0 (select, not multiply: the masked
          // exponent may overflow)
          const float p0 = keep ? fast_exp2(x0) : 0.f, p1 = keep ? fast_exp2(x1) : 0.f;
          const uint64_t dd = f2_mul(f2_pack(p0, p1), f2_add(((uint64_t)rd[i + 1] << 32) | rd[i], nd2));
          float ds0, ds1;
          f2_unpack(dd, ds0, ds1);
          pk[i / 2] = pack_bf16(p0, p1);
          dk2[i / 2] = pack_bf16(ds0, ds1);
          if (bi == 0) {  // the chunk's first batch row initialises the (uninitialised) TMEM
            acc[i] = __float_as_uint(ds0);
            acc[i + 1] = __float_as_uint(ds1);
          } else {
            const uint64_t s2 = f2_add(((uint64_t)acc[i + 1] << 32) | acc[i], dd);
            float lo, hi;
            f2_unpack(s2, lo, hi);
            acc[i] = __float_as_uint(lo);
            acc[i + 1] = __float_as_uint(hi);
          }
        }
      }
      if (w == 0 && lane == 0) PTL(15, j);  // math done
      if (do_sig) tmem_st32(tSig + lane_base + qcol, acc);
      if (sig_only) {  // Σ-only pass: no Pᵀ/dSᵀ hand-off, no gradient MMAs, no drains
        if (s == 1) {  // this warp's last read of the tile's lse2/D: the stage may be reloaded
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_infree + 8 * st);
        }
        if (s == 1 && ++t == nq) { t = 0; ++bi; }
        continue;
      }
      // before overwriting: this half's Pᵀ columns are read by dV of the previous hand-off; the
      // tile's dSᵀ buffer (T & 1) by tile T-2's dQ MMA
      if (w == 0 && lane == 0) PTL(3, j);  // math + Σ done
      if (j >= 1) mbar_wait(hq ? bar_mm1 : bar_mm0, (j - 1) & 1);
      if (BIG) {  // single dSᵀ buffer: tile T-1's dQ MMA must have read it
        if (s == 0 && T >= 1) mbar_wait(bar_dq, (T - 1) & 1);
      } else if (s == 0 && T >= 2) {
        mbar_wait(bar_dq + 8 * ds, ((T - 2) >> 1) & 1);
      }
      tc_fence_after();
      if (w == 0 && lane == 0) PTL(4, j);  // Pᵀ columns / dSᵀ buffer free
      // Pᵀ -> TMEM (16 packed columns for these 32 queries); dSᵀ rows -> smem block qt / 32
      tmem_st16(tP + lane_base + hq * 16, pk);
      {
        const uint32_t db = s0 + C::oDS + (BIG ? 0 : ds) * 32768 + (qt >> 5) * 8192;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          st_shared_v4(db + pd_off[e], dk2[4 * e], dk2[4 * e + 1], dk2[4 * e + 2], dk2[4 * e + 3]);
      }
      tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_ps);
      if (w == 0 && lane == 0) PTL(5, j);  // hand-off
      if (s == 1 && ++t == nq) { t = 0; ++bi; }
    }
    // ---- Σ_b dSᵀ of the chunk -> partial[c][h][q][k0 + row]: warp half hq writes the 32-query
    // column blocks hq, hq + 2, ...
    float* dst = a.partial + ((int64_t)c * a.H + h) * Lq_pad * (int64_t)Lk_pad + k0 + row +
                 (int64_t)t0 * 128 * Lk_pad;
    const int sig_tiles = (BIG && !sig_only) ? 2 : nq;
    for (int cbk = hq; cbk < sig_tiles * 4; cbk += 2) {
      uint32_t acc[32];
      tmem_ld32(tSig + lane_base + cbk * 32, acc);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) dst[(int64_t)(cbk * 32 + i) * Lk_pad] = __uint_as_float(acc[i]);
    }
  }
  tc_fence_before();
  if (pair) cluster_sync_all();  // no CTA exits while its peer may still store / arrive into it
  else __syncthreads();
  if (w == 0) tmem_dealloc<512>(tmem);
}

#ifdef EVO_TIMELINE
extern "C" int evo_debug_pb_timeline_copy(void* dst, size_t bytes) {
  if (bytes > sizeof(g_tlpb)) bytes = sizeof(g_tlpb);
  return (int)cudaMemcpyFromSymbol(dst, g_tlpb, bytes);
}
#endif

template <int DP, bool BIG>
static cudaError_t launch_bwd_pb_t(const BwdFusedLaunch& L, cudaStream_t st) {
  auto kern = bwd_pb_kernel<DP, BIG>;
  const size_t smem = PbCfg<DP, BIG>::kSmem;
  cudaError_t e = set_smem_once(kern, smem);
  if (e != cudaSuccess) return e;
  const int nk = (L.args.Lk + 127) / 128;
  const long long grid = (long long)L.args.H * nk * L.args.nchunks;
  if (grid == 0) return cudaSuccess;
  if (L.args.dq_pair && nk != 2) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = L.args.dq_pair ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, L.tm_q, L.tm_k, L.tm_v, L.tm_da, L.tm_dq, L.tm_dk, L.tm_dv,
                         L.tm_b, L.args);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_bwd_pb_bf16(const BwdFusedLaunch& L, int DP, cudaStream_t st) {
  const bool big = ((L.args.Lq + 127) / 128) * 128 > 256;
  if (big && L.args.dq_pair) return cudaErrorInvalidValue;
  if (DP == 16) return big ? launch_bwd_pb_t<16, true>(L, st) : launch_bwd_pb_t<16, false>(L, st);
  if (DP == 32) return big ? launch_bwd_pb_t<32, true>(L, st) : launch_bwd_pb_t<32, false>(L, st);
  return cudaErrorInvalidValue;
}

}  // namespace evo
