// evo_bwd_fused.cu — single-pass bf16 backward on sm_100a: dK, dV, dQ and the pair-bias
// gradient of one (head, 128-key tile) for a chunk of batch rows, in one persistent CTA.
// Shipped only as the Σ-only pass (sigma_only, first query tile 2) of a shared bias with
// 256 < Lq <= 384 (BASELINE cfg 5): the gradients and the first 256 queries' Σ run on
// evo_bwd_pb.cu (BIG), no bias on evo_bwd_nb.cu.
//
// Same arithmetic as evo_bwd.cu's bwd_main + bwd_bias (SPEC.md L168
// recompute backward; dbias = Σ_b dS over the broadcast axis, PAPER.md L294 / north star), but
// the probabilities are recomputed ONCE: the CTA loops over its batch rows and, for each, over
// 32-query sub-tiles, and accumulates Σ_b dSᵀ for its key tile in TMEM (fp32, read-modify-write
// by the owning thread), so the separate dbias pass and its second recompute disappear.
//
// Roles (384 threads): two compute warpgroups (warps 0-3, 4-7) take alternate sub-tiles
// (ping-pong: one group's exp/ALU work covers the other's hand-offs and drains); warp 8 (lane 0)
// issues the Sᵀ/dPᵀ MMAs of a sub-tile pair (one per group) as N = 64 MMAs, warp 10 lane 0 the
// dV/dK/dQ MMAs, warp 9 lane 0 the TMA loads, warp 11 idles.  Thread = key row k = TMEM lane.
// Per sub-tile j (queries q0..q0+31 of batch row b), group g = j & 1:
//   MMA:      Sᵀ = K_b·Q_jᵀ, dPᵀ = V_b·dA_jᵀ      (M = 128 keys, N = 32 queries of the pair) -> TMEM
//   compute:  Pᵀ = exp2(Sᵀ·scale·log2e + biasᵀ·log2e − lse2), dSᵀ = Pᵀ⊙(dPᵀ − D)
//             Σ_b dSᵀ += dSᵀ (TMEM RMW), Pᵀ -> TMEM slot g, dSᵀ -> smem block (j & 3) of the tile
//   MMA:      dV_b += Pᵀ·dA_j (A = Pᵀ from TMEM), dK_b += dSᵀ·Q_j;  after the 4 sub-tiles of a tile:
//             dQ_part = dS·K_b (A = the tile's dSᵀ blocks read MN-major)
// Drains: group 1 the previous tile's dQ part after its first sub-tile of a tile, group 0 dK/dV
// at a new batch row, through swizzled staging tiles and per-warp TMA stores of 32-row slices
// (direct per-thread global stores of the rows measured ~10% slower).
// The issuer runs Sᵀ/dPᵀ ahead (one sub-tile pair), so before overwriting its Pᵀ slot a group
// waits for dV/dK(j-2) (bar_mm).  The dSᵀ blocks are double-buffered per 128-query tile (buffer
// T & 1): a group starting tile T waits only for tile T-2's dQ MMA, long done, instead of the
// previous tile's.
//
// TMEM (512 cols): [0, Lq_pad) Σ dSᵀ (with bias) | Sᵀ 2x32 | dPᵀ 2x32 | dV DP | dK DP | dQ DP |
//                  Pᵀ 2 x 16 (bf16 pairs)
// SMEM: biasᵀ resident [128 k][Lq_pad] bf16 (16-B chunks XOR-swizzled by k&7) | K,V x2 |
//       Q,dA x2 | dSᵀ 2 x 4 x 8 KB | lse2/D x2 | dK/dV/dQ staging | barriers
#include <cstdio>
#include <cstdlib>

#include "evo_kernels.cuh"

namespace evo {

#ifdef EVO_TIMELINE
// Debug builds only (tools/timeline.py compiles a separate library with -DEVO_TIMELINE):
// clock64 stamps of CTAs 0 and 1, 12 event kinds x 512 sub-tiles each.
__device__ unsigned long long g_tl[2][12][512];
#define TL(ev, i)                                                                \
  do {                                                                           \
    if (blockIdx.x < 2 && (i) < 512) g_tl[blockIdx.x][ev][i] = clock64();        \
  } while (0)
#else
#define TL(ev, i) do { } while (0)
#endif

// BIG: a shared bias with 256 < Lq <= 384 (BASELINE cfg 5, N_res = 384): the resident biasᵀ
// grows to [128 k][384 q] and the dSᵀ blocks are single-buffered to stay inside 227 KB of smem;
// Σ_b dSᵀ stays in TMEM for the first 256 queries (the main pass) and the remaining query tile
// gets its own Σ-only pass (a.sigma_only, first tile a.t0 = 2).
template <int DP, bool BIAS, bool BIG = false>
struct FusedCfg {
  static constexpr uint32_t kRowBytes = DP * 2;
  static constexpr uint32_t kTile = 128 * kRowBytes;  // one 128-row Q/K/V/dA tile
  static constexpr uint32_t kBiasMax = BIAS ? 128u * (BIG ? 384u : 256u) * 2u : 0u;
  static constexpr uint32_t kDS = BIG ? 32768u : 65536u;  // dSᵀ: (1 or 2) x 4 x 8 KB
  static constexpr uint32_t oBias = 0;
  static constexpr uint32_t oKV = oBias + kBiasMax;      // stage s: K at +s*2*kTile, V +kTile
  static constexpr uint32_t oQA = oKV + 4 * kTile;       // stage s: Q at +s*2*kTile, dA +kTile
  static constexpr uint32_t oDS = oQA + 4 * kTile;       // tile T in buffer BIG ? 0 : T & 1
  static constexpr uint32_t oVec = oDS + kDS;            // 2 x (lse2[128], D[128]) fp32
  static constexpr uint32_t oStK = oVec + 2048;          // staging: dK, dV bf16, dQ bf16|fp32
  static constexpr uint32_t oStV = oStK + kTile;
  static constexpr uint32_t oStQ = oStV + kTile;         // dQ staging: bf16 | fp32 [128][DP]
  static constexpr uint32_t oBar = oStQ + 128 * DP * 4;
  static constexpr uint32_t kSmem = oBar + 256;
};

template <int N>
EVO_DEV void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[N]) {
  if constexpr (N == 16) tmem_ld16(taddr, r);
  else tmem_ld32(taddr, r);
}

template <int DP, bool BIAS, bool BIG>
__global__ void __launch_bounds__(384, 1)
    bwd_fused_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_da,
                     const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ CUtensorMap tm_dk,
                     const __grid_constant__ CUtensorMap tm_dv, const __grid_constant__ CUtensorMap tm_b,
                     const BwdFusedArgs a) {
  using C = FusedCfg<DP, BIAS, BIG>;
  static_assert(DP == 16 || DP == 32, "fused backward: head dim pad 16 or 32");
  constexpr uint32_t kSw = DP == 32 ? kSw64 : kSw32;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t s0 = smem_u32(smem);
  if (s0 & 1023u) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::oBar);
  const uint32_t bar_kv = smem_u32(&bars[0]);       // +8: stage 1   (TMA K,V landed)
  const uint32_t bar_in = smem_u32(&bars[2]);       // +8: stage 1   (TMA Q,dA,vec landed)
  const uint32_t bar_kvfree = smem_u32(&bars[4]);   // +8            (MMA done with K,V stage)
  const uint32_t bar_infree = smem_u32(&bars[6]);   // +8            (MMA done with Q,dA stage)
  const uint32_t bar_sp = smem_u32(&bars[8]);       // +8: group 1   Sᵀ, dPᵀ in TMEM slot
  const uint32_t bar_sfree = smem_u32(&bars[10]);   // +8            group pulled its slot (4 warps)
  const uint32_t bar_ps = smem_u32(&bars[12]);      // +8            Pᵀ, dSᵀ in smem (4 warps)
  const uint32_t bar_dq = smem_u32(&bars[18]);      // +8: dSᵀ buffer 1   dQ MMA of a tile done
  const uint32_t bar_dkvfree = smem_u32(&bars[15]); // group 0 pulled a finished dK/dV (4 warps)
  const uint32_t bar_bias = smem_u32(&bars[14]);    // the bias tiles of the prologue landed (TMA)
  const uint32_t bar_mm = smem_u32(&bars[16]);      // +8: group 1   dV/dK of its sub-tile done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(&bars[20]);

  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int nq_all = (a.Lq + 127) >> 7, nk = (a.Lk + 127) >> 7;
  const int Lq_pad = nq_all * 128, Lk_pad = nk * 128;
  // query tiles t0 .. nq_all-1 (t0 = 2 in the Σ-only pass of a BIG call); nq counts them and
  // every loop below runs t over [0, nq) with query tile tq = t0 + t
  const int t0 = a.t0, nq = nq_all - t0;
  const bool sig_only = a.sigma_only != 0;
  const int c = (int)blockIdx.x % a.nchunks;
  const int grp = (int)blockIdx.x / a.nchunks;
  const int kt = grp % nk, h = grp / nk;
  const int k0 = kt * 128;
  const int b0 = c * a.chunk;
  const int nb = min(a.B - b0, a.chunk);
  if (nb <= 0) return;
  const int J = nb * nq * 4;  // 32-query sub-tiles

  if (w == 0) tmem_alloc<512>(smem_u32(tmem_slot));
  if (tid == 32) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_kv + 8 * i, 1);
      mbar_init(bar_in + 8 * i, 1);
      mbar_init(bar_kvfree + 8 * i, 1);
      // the Σ-only pass frees a Q/dA/vector stage when the 8 compute warps are done with the
      // tile's lse2/D vectors (the gradient issuer's dQ commit does it otherwise)
      mbar_init(bar_infree + 8 * i, a.sigma_only ? 8 : 1);
      mbar_init(bar_sp + 8 * i, 1);
      mbar_init(bar_sfree + 8 * i, 4);
      mbar_init(bar_ps + 8 * i, 4);
      mbar_init(bar_mm + 8 * i, 1);
    }
    mbar_init(bar_dq, 1);
    mbar_init(bar_dq + 8, 1);
    mbar_init(bar_dkvfree, 4);
    mbar_init(bar_bias, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Σ_b dSᵀ columns: the query tiles t < sig_n (relative to t0) accumulate in TMEM
  const int sig_n = BIAS ? (nq < 2 ? nq : 2) : 0;
  const uint32_t cb = BIAS ? (BIG ? 256u : (uint32_t)Lq_pad) : 0u;
  const uint32_t tDB = tmem, tS0 = tmem + cb, tdV = tS0 + 128, tdK = tdV + DP, tdQ = tdK + DP;
  const uint32_t tP0 = tdQ + DP;  // Pᵀ slot g at +16 g (32 bf16 queries as 16 packed columns)

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
          tma_load_4d(qb, &tm_q, bar, 0, (t0 + t) * 128, h, b);
          tma_load_4d(qb + C::kTile, &tm_da, bar, 0, (t0 + t) * 128, h, b);
          const int64_t vrow = ((int64_t)b * a.H + h) * Lq_pad + (t0 + t) * 128;
          bulk_load(s0 + C::oVec + st * 1024, a.lse2 + vrow, 512, bar);
          bulk_load(s0 + C::oVec + st * 1024 + 512, a.Dvec + vrow, 512, bar);
        }
      }
    }
  } else if (w == 8) {
    // ------------------------------------------------------------------ Sᵀ/dPᵀ MMA issuer
    // One N = 64 MMA per K step covers the sub-tile pair (j, j+1) of the two groups (queries
    // 32s..32s+63 of one tile, s in {0, 2}): a K = 16 step costs the same ~46 cycles at N = 32 and
    // N = 64 (tools/micro/mma_bench.cu), so pairing halves the Sᵀ/dPᵀ tensor time.  TMEM slot
    // layout [Sᵀ_j | Sᵀ_j+1 | dPᵀ_j | dPᵀ_j+1]; the pair starts once both groups pulled the
    // previous pair (so it runs while they compute it).
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, 0, 0);
      int sbi = 0, stt = 0, sss = 0;
      for (int j = 0; j < J; j += 2) {
        if (j >= 2) {
          mbar_wait(bar_sfree, ((j - 2) >> 1) & 1);
          mbar_wait(bar_sfree + 8, ((j - 2) >> 1) & 1);
        }
        const int T = sbi * nq + stt, st = T & 1, kvs = sbi & 1;
        if (sss == 0) mbar_wait(bar_in + 8 * st, (T >> 1) & 1);
        if (sss == 0 && stt == 0) mbar_wait(bar_kv + 8 * kvs, (sbi >> 1) & 1);
        TL(0, j);  // S/dP pair issued
        tc_fence_after();
        const uint32_t kb = s0 + C::oKV + kvs * 2 * C::kTile;
        const uint32_t qb = s0 + C::oQA + st * 2 * C::kTile + sss * 32 * C::kRowBytes;
#pragma unroll
        for (int kk = 0; kk < DP / 16; ++kk)
          umma_bf16(tS0, make_sdesc(kb + kk * 32, 16, 8 * C::kRowBytes, kSw),
                    make_sdesc(qb + kk * 32, 16, 8 * C::kRowBytes, kSw), idesc_s, kk > 0);
#pragma unroll
        for (int kk = 0; kk < DP / 16; ++kk)
          umma_bf16(tS0 + 64, make_sdesc(kb + C::kTile + kk * 32, 16, 8 * C::kRowBytes, kSw),
                    make_sdesc(qb + C::kTile + kk * 32, 16, 8 * C::kRowBytes, kSw), idesc_s,
                    kk > 0);
        umma_commit(bar_sp);
        umma_commit(bar_sp + 8);
        if (sig_only && sss == 2 && stt == nq - 1)  // no gradient MMAs in the Σ-only pass:
          umma_commit(bar_kvfree + 8 * kvs);         // the Sᵀ/dPᵀ MMAs are K/V's last readers
        sss += 2;
        if (sss >= 4) {
          sss = 0;
          if (++stt == nq) { stt = 0; ++sbi; }
        }
      }
    }
  } else if (w == 10) {
    // ------------------------------------------------------------------ gradient-MMA issuer
    // dV/dK of sub-tile i once its Pᵀ/dSᵀ are in smem; the dQ part after a tile's 4th.  A
    // separate thread from the Sᵀ issuer, so neither stream waits on the other's events.
    if (lane == 0 && !sig_only) {
      constexpr uint32_t idesc_kv = make_idesc_bf16(128, DP, 0, 1);  // dV, dK (B MN-major)
      constexpr uint32_t idesc_q = make_idesc_bf16(128, DP, 1, 1);   // dQ (A, B MN-major)
      int dbi = 0, dtt = 0, dss = 0;  // coordinates of sub-tile i
      for (int i = 0; i < J; ++i) {
        const int g = i & 1;
        const int T = dbi * nq + dtt, st = T & 1, kvs = dbi & 1;
        mbar_wait(bar_ps + 8 * g, (i >> 1) & 1);
        TL(4, i);  // hand-off seen by the grad issuer
        // the first sub-tile of a new batch row overwrites dK/dV: group 0 must have pulled them
        if (dtt == 0 && dss == 0 && dbi > 0) mbar_wait(bar_dkvfree, (dbi - 1) & 1);
        TL(5, i);  // dV/dK issued
        tc_fence_after();
        const uint32_t qb = s0 + C::oQA + st * 2 * C::kTile + dss * 32 * C::kRowBytes;
        const uint32_t ab = qb + C::kTile;
        const uint32_t db = s0 + C::oDS + (BIG ? 0 : st) * 32768 + dss * 8192;
        const uint32_t acc0 = (dtt > 0 || dss > 0) ? 1u : 0u;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk)  // dV += Pᵀ·dA (K = 32 queries; A = Pᵀ from TMEM)
          umma_bf16_ts(tdV, tP0 + g * 16 + kk * 8,
                       make_sdesc(ab + kk * 16 * C::kRowBytes, 16384, 8 * C::kRowBytes, kSw),
                       idesc_kv, (acc0 | (uint32_t)kk) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk)  // dK += dSᵀ·Q
          umma_bf16(tdK, make_sdesc(db + kk * 32, 16, 512, kSw64),
                    make_sdesc(qb + kk * 16 * C::kRowBytes, 16384, 8 * C::kRowBytes, kSw),
                    idesc_kv, (acc0 | (uint32_t)kk) ? 1u : 0u);
        umma_commit(bar_mm + 8 * g);
        TL(8, i);  // dV/dK issue finished
        if (dss == 3) {  // the tile's 4 dSᵀ blocks are complete: dQ part = dS·K
          const uint32_t kb = s0 + C::oKV + kvs * 2 * C::kTile;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16(tdQ, make_sdesc(s0 + C::oDS + (BIG ? 0 : st) * 32768 + kk * 1024, 8192, 512, kSw64),
                      make_sdesc(kb + kk * 16 * C::kRowBytes, 16384, 8 * C::kRowBytes, kSw),
                      idesc_q, kk > 0 ? 1u : 0u);
          umma_commit(bar_dq + 8 * (BIG ? 0 : st));
          TL(6, T);  // dQ issued
          // every reader of the Q/dA stage (Sᵀ/dPᵀ MMAs: pulled before the groups' hand-offs;
          // dV/dK/dQ: this thread) is done once these commits land
          umma_commit(bar_infree + 8 * st);
          if (dtt == nq - 1) umma_commit(bar_kvfree + 8 * kvs);
        }
        if (++dss == 4) {
          dss = 0;
          if (++dtt == nq) { dtt = 0; ++dbi; }
        }
      }
    }
  } else if (w < 8) {  // (warp 11 idles)
    // ------------------------------------------------------------------ compute warpgroups
    const int g = w >> 2, qd = w & 3;
    const int row = qd * 32 + lane;  // key row within the tile = TMEM lane
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    const uint32_t sBias = s0 + C::oBias;
    if (BIAS) {
      // biasᵀ[k][q] = bias[h, q, k0 + k] for q < Lq, k0 + k < Lk; 0 elsewhere (TMA zero fill:
      // padding must be finite, it meets zero P/dA rows in the MMAs).  Resident layout: Lq_pad / 64
      // segments of [128 k][64 q] with 128-B rows, 16-B chunks XOR-swizzled by k & 7 (the TMA
      // 128-B swizzle), so a q-contiguous (end-node) bias lands there straight from TMA, and a
      // k-contiguous one is staged [q][64 k] x 2 in the (not yet used) dSᵀ buffers and transposed
      // 8 x 8 blocks at a time by ldmatrix + stmatrix.trans (conflict-free both ways).
      if (tid == 0) {
        if (a.bmode == 2) {
          mbar_arrive_expect_tx(bar_bias, (uint32_t)(Lq_pad / 64) * 16384u);
          for (int sg = 0; sg < Lq_pad / 64; ++sg)
            tma_load_4d(sBias + sg * 16384, &tm_b, bar_bias, sg * 64, k0, h, 0);
        } else if (!BIG) {
          mbar_arrive_expect_tx(bar_bias, 65536u);
          tma_load_4d(s0 + C::oDS, &tm_b, bar_bias, k0, 0, h, 0);
          tma_load_4d(s0 + C::oDS + 32768, &tm_b, bar_bias, k0 + 64, 0, h, 0);
        }
      }
      if (a.bmode == 2 || !BIG) mbar_wait(bar_bias, 0);
      // k-contiguous: one pass over all queries ([256 q][64 k] x 2 staged), or for BIG passes of
      // 128 queries ([128 q][64 k] x 2 = the single 32 KB dSᵀ buffer)
      const int npass = (a.bmode != 2 && BIG) ? Lq_pad / 128 : (a.bmode != 2 ? 1 : 0);
      for (int ps = 0; ps < npass; ++ps) {
        const int qb0 = BIG ? ps * 128 : 0;                  // first query of the pass
        const int nq8 = BIG ? 16 : Lq_pad / 8;              // 8-query blocks in the pass
        const uint32_t kbox = BIG ? 16384u : 32768u;        // staged [q][64 k] box bytes
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
      named_bar_sync(1, 256);
    }

    const uint64_t sl2 = f2_pack(a.scale_log2, a.scale_log2);
    const uint64_t l2e2 = f2_pack(kLog2e, kLog2e);
    const int kglob = k0 + row;
    // ---- drains (group 0): TMEM rows -> swizzled staging tiles -> one thread's TMA stores
    constexpr uint32_t kRbB = DP * 2;  // bf16 staging row bytes (= the x-map swizzle span)
    auto stage_bf16 = [&](uint32_t base, const uint32_t (&r)[DP], float mul) {
#pragma unroll
      for (int i = 0; i < DP / 8; ++i)
        st_shared_v4(base + swz_offset(row, i, kRbB),
                     pack_bf16(__uint_as_float(r[8 * i]) * mul, __uint_as_float(r[8 * i + 1]) * mul),
                     pack_bf16(__uint_as_float(r[8 * i + 2]) * mul, __uint_as_float(r[8 * i + 3]) * mul),
                     pack_bf16(__uint_as_float(r[8 * i + 4]) * mul, __uint_as_float(r[8 * i + 5]) * mul),
                     pack_bf16(__uint_as_float(r[8 * i + 6]) * mul, __uint_as_float(r[8 * i + 7]) * mul));
    };
    // Drains: group 0 drains dK/dV at a new batch row (staging + TMA stores), group 1 the dQ part
    // of the previous query tile (straight from TMEM to global memory, each thread its own row),
    // so the two groups share the drain work and group 0's dK/dV release (which gates the
    // gradient issuer) is not queued behind the dQ store.
    // Each warp drains its own 32 rows (its TMEM lane quarter) into its slice of the staging tile
    // and issues that slice's TMA store itself (32-row boxes): no group-wide barrier, no single
    // issuing thread.
    const uint32_t slice = (uint32_t)(qd * 32);
    auto drain_kv = [&](int bk, bool release_kv) {  // group 0
      if (lane == 0) bulk_wait_group_read0();  // this warp's previous stores left its slices
      __syncwarp();
      uint32_t r[DP];
      tmem_ld_cols(tdK + lane_base, r);
      tmem_wait_ld();
      stage_bf16(s0 + C::oStK, r, a.scale);
      tmem_ld_cols(tdV + lane_base, r);
      tmem_wait_ld();
      if (release_kv) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_dkvfree);
      }
      stage_bf16(s0 + C::oStV, r, 1.f);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_4d(&tm_dk, s0 + C::oStK + slice * kRbB, 0, k0 + (int)slice, h, bk);
        tma_store_4d(&tm_dv, s0 + C::oStV + slice * kRbB, 0, k0 + (int)slice, h, bk);
        bulk_commit_group();
      }
    };
    // dQ part of tile Tq (group 1), once its dQ MMA has landed: bf16 rows when there is one key
    // tile, else this key tile's fp32 part (dq_convert sums the parts); swizzled staging + TMA store
    auto drain_q = [&](int Tq) {
      if (BIG) mbar_wait(bar_dq, Tq & 1);
      else mbar_wait(bar_dq + 8 * (Tq & 1), (Tq >> 1) & 1);
      if (qd == 0 && lane == 0) TL(7, Tq);  // dQ landed (drain)
      tc_fence_after();
      if (lane == 0) bulk_wait_group_read0();
      __syncwarp();
      uint32_t r[DP];
      tmem_ld_cols(tdQ + lane_base, r);
      tmem_wait_ld();
      if (nk == 1) {
        stage_bf16(s0 + C::oStQ, r, a.scale);
      } else {
#pragma unroll
        for (int i = 0; i < DP / 4; ++i)
          st_shared_v4(s0 + C::oStQ + swz_offset(row, i, DP * 4), r[4 * i], r[4 * i + 1], r[4 * i + 2],
                       r[4 * i + 3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        const int bq = b0 + Tq / nq;
        const uint32_t rb = nk == 1 ? kRbB : (uint32_t)(DP * 4);
        if (nk > 1 && a.dq_reduce)  // TMA .add at L2 into one fp32 accumulator (bwd_pre zeroed it),
          // evict_last so the lines stay in L2 for the other key tiles' adds and for dq_convert
          tma_reduce_add_4d_hint(&tm_dq, s0 + C::oStQ + slice * rb, 0, (t0 + Tq % nq) * 128 + (int)slice, h, bq,
                                 l2_policy_evict_last());
        else
          tma_store_4d(&tm_dq, s0 + C::oStQ + slice * rb, 0, (t0 + Tq % nq) * 128 + (int)slice, h,
                       nk == 1 ? bq : kt * a.B + bq);
        bulk_commit_group();
      }
    };
    // hard-mask bits of this thread's key for 32 batch rows from b: all 32 byte loads in flight
    // together, once per 32 rows (a per-row load was consumed right behind its issue)
    auto load_keep_word = [&](int b) -> uint32_t {
      if (kglob >= a.Lk) return 0u;
      if (!a.mask) return ~0u;
      uint32_t v[32];
#pragma unroll
      for (int x = 0; x < 32; ++x)
        v[x] = b + x < b0 + nb ? (uint32_t)__ldg(a.mask + (int64_t)(b + x) * a.mask_s0 + (int64_t)kglob * a.mask_s1) : 0u;
      uint32_t wd = 0u;
#pragma unroll
      for (int x = 0; x < 32; ++x) wd |= (v[x] != 0u ? 1u : 0u) << x;
      return wd;
    };
    uint32_t pd_off[4];  // this thread's row of a [128][32] bf16 SW64 tile: 4 chunk offsets
#pragma unroll
    for (int e = 0; e < 4; ++e) pd_off[e] = swz_offset(row, e, 64);
    uint32_t keep_word = 0u;
    bool keep = false;
    int bi = 0, t = 0, s = g;  // this group's sub-tiles: j = g, g+2, ...; j = ((bi*nq)+t)*4 + s
    for (int j = g; j < J; j += 2) {
      const int T = bi * nq + t;
      const int st = T & 1;
      const int b = b0 + bi;
      if (s == g && t == 0) {
        if ((bi & 31) == 0) keep_word = load_keep_word(b);
        keep = (keep_word >> (bi & 31)) & 1u;
      }
      if (qd == 0 && lane == 0) TL(1, j);  // group starts waiting for S
      mbar_wait(bar_sp + 8 * g, (j >> 1) & 1);
      if (qd == 0 && lane == 0) TL(2, j);  // S landed
      tc_fence_after();
      uint32_t rs[32], rd[32];
      const int qcol = (t0 + t) * 128 + s * 32;  // first query of this sub-tile
      const int scol = t * 128 + s * 32;         // its Σ column (query tiles t < sig_n)
      const bool do_sig = BIAS && t < sig_n;
      // Σ_b dSᵀ so far for these 32 columns (this thread's own lane and columns, last written
      // one batch row ago): loaded with Sᵀ/dPᵀ so one wait covers all three
      uint32_t acc[32];
      {
        tmem_ld32(tS0 + 32 * g + lane_base, rs);
        tmem_ld32(tS0 + 64 + 32 * g + lane_base, rd);
        if (do_sig && bi > 0) tmem_ld32(tDB + lane_base + scol, acc);
      }
      tmem_wait_ld();
      if (qd == 0 && lane == 0) TL(11, j);  // Sᵀ/dPᵀ/Σ in registers
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_sfree + 8 * g);
      mbar_wait(bar_in + 8 * st, (T >> 1) & 1);  // lse2 / D of this query tile visible
      const uint32_t vbase = s0 + C::oVec + st * 1024 + s * 32 * 4;
      uint32_t pk[16], dk2[16];
      float ds[32];
#pragma unroll
      for (int gq = 0; gq < 4; ++gq) {  // 8 queries per group
        // the vectors arrive negated: -lse·log2e (-inf for rows without a kept key), -D
        const uint4 l0 = ld_shared_v4(vbase + gq * 32), l1 = ld_shared_v4(vbase + gq * 32 + 16);
        const uint4 d0 = ld_shared_v4(vbase + 512 + gq * 32), d1 = ld_shared_v4(vbase + 512 + gq * 32 + 16);
        const uint32_t nl[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
        const uint32_t nd[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
        uint32_t bu[4] = {0, 0, 0, 0};
        if (BIAS) {
          const uint32_t cq = (uint32_t)(qcol >> 3) + gq;  // 8-query chunk
          const uint4 bv = ld_shared_v4(sBias + (cq >> 3) * 16384u + row * 128u + (((cq & 7u) ^ (row & 7u)) << 4));
          bu[0] = bv.x; bu[1] = bv.y; bu[2] = bv.z; bu[3] = bv.w;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int i = gq * 8 + 2 * e;
          const uint64_t nl2 = ((uint64_t)nl[2 * e + 1] << 32) | nl[2 * e];
          const uint64_t nd2 = ((uint64_t)nd[2 * e + 1] << 32) | nd[2 * e];
          uint64_t x = BIAS ? f2_fma(bf16x2_to_f2(bu[e]), l2e2, nl2) : nl2;
          x = f2_fma(((uint64_t)rs[i + 1] << 32) | rs[i], sl2, x);
          float x0, x1;
          f2_unpack(x, x0, x1);
          const float p0 = fast_exp2(x0), p1 = fast_exp2(x1);
          const uint64_t p2 = f2_pack(p0, p1);
          const uint64_t dd = f2_mul(p2, f2_add(((uint64_t)rd[i + 1] << 32) | rd[i], nd2));
          f2_unpack(dd, ds[i], ds[i + 1]);
          pk[i / 2] = pack_bf16(p0, p1);
          dk2[i / 2] = pack_bf16(ds[i], ds[i + 1]);
        }
      }
      // hard mask (R5): a masked key row has P = dS = 0.  The key is this thread's row, so the
      // fix-up is per thread and skipped by whole warps in the common all-kept case
      if (__any_sync(0xffffffffu, !keep) && !keep) {
#pragma unroll
        for (int i = 0; i < 16; ++i) { pk[i] = 0u; dk2[i] = 0u; }
#pragma unroll
        for (int i = 0; i < 32; ++i) ds[i] = 0.f;
      }
      if (do_sig) {  // Σ_b dSᵀ in TMEM (this thread's lane, this sub-tile's 32 query columns)
        if (bi == 0) {  // first batch row of the chunk initialises the (uninitialised) TMEM
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[i] = __float_as_uint(ds[i]);
        } else {
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const uint64_t s2 = f2_add(((uint64_t)acc[i + 1] << 32) | acc[i], f2_pack(ds[i], ds[i + 1]));
            float lo, hi;
            f2_unpack(s2, lo, hi);
            acc[i] = __float_as_uint(lo);
            acc[i + 1] = __float_as_uint(hi);
          }
        }
        tmem_st32(tDB + lane_base + scol, acc);
      }
      if (sig_only) {  // Σ-only pass: no Pᵀ/dSᵀ hand-off, no gradient MMAs, no drains
        if (s >= 2) {  // this warp's last sub-tile of the tile: its lse2/D stage may be reloaded
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_infree + 8 * st);
        }
        s += 2;
        if (s >= 4) {
          s -= 4;
          if (++t == nq) { t = 0; ++bi; }
        }
        continue;
      }
      // before overwriting: Pᵀ slot g is read by dV(j-2); this tile's dSᵀ buffer (T & 1) by tile
      // T-2's dQ MMA, long done (checked at the group's first sub-tile of a tile)
      if (qd == 0 && lane == 0) TL(9, j);  // math + Σ store done
      if (j >= 2) mbar_wait(bar_mm + 8 * g, ((j - 2) >> 1) & 1);
      if (BIG) {  // single dSᵀ buffer: tile T-1's dQ MMA must have read it
        if (s == g && T >= 1) mbar_wait(bar_dq, (T - 1) & 1);
      } else if (s == g && T >= 2) {
        mbar_wait(bar_dq + 8 * st, ((T - 2) >> 1) & 1);
      }
      if (qd == 0 && lane == 0) TL(10, j);  // Pᵀ slot / dSᵀ buffer free
      tc_fence_after();
      // Pᵀ -> TMEM slot g (the A operand of the TS-form dV MMA); dSᵀ (block s) rows to smem:
      // this thread's key row, 32 queries = 4 x 16 B, SW64
      tmem_st16(tP0 + g * 16 + lane_base, pk);
      {
        const uint32_t db = s0 + C::oDS + (BIG ? 0 : st) * 32768 + s * 8192;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          st_shared_v4(db + pd_off[e], dk2[4 * e], dk2[4 * e + 1], dk2[4 * e + 2], dk2[4 * e + 3]);
      }
      tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_ps + 8 * g);
      if (qd == 0 && lane == 0) TL(3, j);  // hand-off
      if (g == 0 && s == 0 && t == 0 && bi > 0) {
        // the previous row's last dV/dK MMAs were group 1's sub-tile j - 1 (bar_mm slot 1)
        mbar_wait(bar_mm + 8, ((j - 1) >> 1) & 1);
        tc_fence_after();
        drain_kv(b - 1, true);
      }
      // the previous tile's dQ part; the next dQ MMA (which overwrites it) waits for this
      // group's hand-off of the tile's last sub-tile
      if (g == 1 && s == 1 && T > 0) drain_q(T - 1);
      s += 2;
      if (s >= 4) {
        s -= 4;
        if (++t == nq) { t = 0; ++bi; }
      }
    }
    // ---- tail: last dQ part (group 1) and last dK/dV (group 0); then both write Σ_b dSᵀ
    const int Tl = (J >> 2) - 1;
    if (sig_only) {
    } else if (g == 0) {
      if (BIG) mbar_wait(bar_dq, Tl & 1);
      else mbar_wait(bar_dq + 8 * (Tl & 1), (Tl >> 1) & 1);
      tc_fence_after();
      drain_kv(b0 + nb - 1, false);
    } else {
      drain_q(Tl);
    }
    if (lane == 0) bulk_wait_group0();
    if (BIAS) {  // partial[c][h][q][k0 + row]: this group's 32-query column blocks
      float* dst = a.partial + ((int64_t)c * a.H + h) * Lq_pad * (int64_t)Lk_pad + k0 + row +
                   (int64_t)t0 * 128 * Lk_pad;
      for (int cbk = g; cbk < sig_n * 4; cbk += 2) {
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

template <int DP, bool BIAS, bool BIG>
static cudaError_t launch_bwd_fused_t(const BwdFusedLaunch& L, cudaStream_t st) {
  auto kern = bwd_fused_kernel<DP, BIAS, BIG>;
  const size_t smem = FusedCfg<DP, BIAS, BIG>::kSmem;
  cudaError_t e = set_smem_once(kern, smem);
  if (e != cudaSuccess) return e;
  const int nk = (L.args.Lk + 127) / 128;
  const long long grid = (long long)L.args.H * nk * L.args.nchunks;
  if (grid == 0) return cudaSuccess;
  kern<<<(unsigned)grid, 384, smem, st>>>(L.tm_q, L.tm_k, L.tm_v, L.tm_da, L.tm_dq, L.tm_dk, L.tm_dv,
                                          L.tm_b, L.args);
  return cudaGetLastError();
}

#ifdef EVO_TIMELINE
extern "C" int evo_debug_timeline_copy(void* dst, size_t bytes) {
  if (bytes > sizeof(g_tl)) bytes = sizeof(g_tl);
  return (int)cudaMemcpyFromSymbol(dst, g_tl, bytes);
}
#endif

// Only the BIG instantiation ships, as the Σ-only pass of 256 < Lq <= 384 with a bias (the main
// pass is evo_bwd_pb.cu's BIG variant; no bias runs on evo_bwd_nb.cu — DESIGN §7c)
cudaError_t launch_bwd_fused_bf16(const BwdFusedLaunch& L, int DP, int has_bias, cudaStream_t st) {
  const bool big = has_bias && ((L.args.Lq + 127) / 128) * 128 > 256;
  if (!big) return cudaErrorInvalidValue;
  if (DP == 16) return launch_bwd_fused_t<16, true, true>(L, st);
  if (DP == 32) return launch_bwd_fused_t<32, true, true>(L, st);
  return cudaErrorInvalidValue;
}

}  // namespace evo
