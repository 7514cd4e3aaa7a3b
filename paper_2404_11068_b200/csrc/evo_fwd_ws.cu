// evo_fwd_ws.cu — persistent, warp-specialised bf16 forward (sm_100a).
//
// Same operation as evo_fwd.cu ("a pair bias term is added to the logits matrix
// before the softmax operation", all of MHA fused, FlashAttention-style online softmax),
// re-organised so that the exp (MUFU) pipe — the binding unit at head dim 32 — never waits:
//
//   warp 0       producer: TMA for the Q tile of each unit (double-buffered per slot), the K/V
//                k-tiles (NKV-stage ring) and the bias tiles (NB-stage ring)
//   warp 2       mask packer: key-mask bytes -> 4 bit-words + "all kept" flag per ring entry
//   warp 1       tcgen05.mma issuer (one thread, non-blocking event loop):
//                   S  = Q·Kᵀ                      (SS, K = head dim)
//                   S += Ĩ·B   with Ĩ = bf16(1/scale)·I, B = the bias tile   (SS, K = 128)
//                   O += P·V   with P read from TMEM (TS form)
//                i.e. the pair bias is added by the otherwise idle tensor core, so S·scale is
//                exactly scale·q·k + bias·(scale·bf16(1/scale)) (reading R7b)
//   warps 4-7    softmax slot 0 } two units in flight; each thread owns one query row
//   warps 8-11   softmax slot 1 } (TMEM lane) of a 128x128 tile: tile max (3-input max),
//                lazy online-softmax rescale (threshold 8 in log2 units, as FlashAttention-4),
//                p = exp2(S·scale·log2e - m), row sum (f32x2), P (bf16x2) -> TMEM
//   warps 12-15  epilogue: O / l · sigmoid(g) -> o (bf16), lse = m + log l (fp32)
// TMEM (512 cols): slot s at 256·s: S [0,128), P [128,192), O [192,192+DP).
#include <cstdio>

#include "evo_kernels.cuh"

namespace evo {

namespace {
struct Unit {
  int b, h, qt;
};
EVO_DEV Unit decode_unit(int u, int nq, int H) {
  Unit r;
  r.qt = u % nq;
  const int bh = u / nq;
  r.h = bh % H;
  r.b = bh / H;
  return r;
}
}  // namespace

// ---- debug-only phase timestamps (EVO_DEBUG_TIMING=1): [cta][softmax warp][tile<32][8]
__device__ unsigned long long g_fwd_dbg[148 * 8 * 32 * 8 + 148 * 64 * 4];
unsigned long long* fwd_debug_ptr() {
  static unsigned long long* p = nullptr;
  if (!p) {
    void* q = nullptr;
    if (cudaGetSymbolAddress(&q, g_fwd_dbg) == cudaSuccess) p = (unsigned long long*)q;
  }
  return p;
}

template <int DP, int BIAS>
struct FwdCfg {
  static constexpr int NQ = DP == 64 ? 1 : 2;    // Q buffers per slot
  static constexpr int NKV = DP == 64 ? (BIAS ? 2 : 3) : (BIAS ? 3 : 4);  // K/V ring stages
  static constexpr int NB = DP == 64 ? 2 : 3;    // bias ring stages
  static constexpr uint32_t kTile = 128 * DP * 2;
  static constexpr uint32_t kIdent = BIAS ? 32768 : 0;  // Ĩ (128x128 bf16, SW128 K-major)
  static constexpr uint32_t kSmem = 2 * NQ * kTile + NKV * 2 * kTile + (BIAS ? NB * 32768 : 0) +
                                    kIdent + 2 * 2 * 2 * 128 * 4 + NKV * 32 + 64 * 8 + 16;
};

template <int DP, int BIAS>
__global__ void __launch_bounds__(512, 1)
    fwd_ws_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_b,
                  const FwdArgs a) {
  using C = FwdCfg<DP, BIAS>;
  constexpr int NQ = C::NQ, NKV = C::NKV, NB = C::NB;
  constexpr uint32_t kRowBytes = DP * 2;
  constexpr uint32_t kTile = C::kTile;
  constexpr uint32_t kSw = DP == 64 ? kSw128 : (DP == 32 ? kSw64 : kSw32);

  extern __shared__ __align__(1024) uint8_t smem[];
  if (smem_u32(smem) & 1023u) __trap();
  const uint32_t sQ = smem_u32(smem);              // [slot][NQ]
  const uint32_t sKV = sQ + 2 * NQ * kTile;         // NKV stages of K|V
  const uint32_t sBias = sKV + NKV * 2 * kTile;     // NB stages of 32 KB
  const uint32_t sI = sBias + (BIAS ? NB * 32768 : 0);  // Ĩ
  uint8_t* tail = smem + (sI - sQ) + C::kIdent;
  float* stat = reinterpret_cast<float*>(tail);                        // [slot][2][l|m][128]
  uint32_t* maskw = reinterpret_cast<uint32_t*>(stat + 2 * 2 * 2 * 128);  // [NKV][8]
  uint64_t* bars = reinterpret_cast<uint64_t*>(maskw + NKV * 8);
  const uint32_t b0 = smem_u32(bars);
  auto BAR = [&](int i) { return b0 + 8u * (uint32_t)i; };
  enum {
    Q_FULL = 0, Q_EMPTY = 4, S_FULL = 8, S_EMPTY = 10, P_FULL = 12, O_FULL = 14, O_EMPTY = 16,
    ST_FULL = 18, KV_FULL = 22
  };
  const int KV_EMPTY = KV_FULL + NKV, B_FULL = KV_FULL + 2 * NKV, B_EMPTY = B_FULL + NB,
            MW_FULL = B_EMPTY + NB, NBARS = MW_FULL + NKV;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NBARS);
  const bool all_keys_kept = a.mask == nullptr && (a.Lk & 127) == 0;

  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nq = (a.Lq + 127) >> 7, nk = (a.Lk + 127) >> 7;
  const int U = a.B * a.H * nq;
  const int G = gridDim.x;
  const int N = (U - (int)blockIdx.x + G - 1) / G;  // units of this CTA
  const int NA = (N + 1) >> 1, NBu = N >> 1;
  const int TA = NA * nk, TB = NBu * nk;
  // production / consumption index of tile t of slot s in the interleaved ring order
  auto ring_idx = [&](int s, int t) { return t < TB ? 2 * t + s : TB + t; };

  if (w == 0) tmem_alloc<512>(smem_u32(tmem_slot));
  if (threadIdx.x == 32) {
    for (int i = 0; i < 4; ++i) {
      mbar_init(BAR(Q_FULL + i), 1);
      mbar_init(BAR(Q_EMPTY + i), 1);
      mbar_init(BAR(ST_FULL + i), 4);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(BAR(S_FULL + s), 1);
      mbar_init(BAR(S_EMPTY + s), 4);
      mbar_init(BAR(P_FULL + s), 4);
      mbar_init(BAR(O_FULL + s), 1);
      mbar_init(BAR(O_EMPTY + s), 4);
    }
    for (int i = 0; i < NKV; ++i) {
      mbar_init(BAR(KV_FULL + i), 1);
      mbar_init(BAR(KV_EMPTY + i), 1);
      mbar_init(BAR(MW_FULL + i), 1);
    }
    for (int i = 0; i < NB; ++i) {
      mbar_init(BAR(B_FULL + i), 1);
      mbar_init(BAR(B_EMPTY + i), 1);
    }
    fence_barrier_init();
  }
  if (BIAS) {
    // Ĩ = bf16(1/scale)·I in the K-major SW128 layout (2 regions of 64 K-columns)
    const uint32_t cinv = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(1.f / a.scale));
    for (int idx = threadIdx.x; idx < 128 * 16; idx += blockDim.x) {
      const int r = idx >> 4, ch = idx & 15;  // row r, 16-B chunk ch (8 bf16 of K)
      uint32_t v[4] = {0, 0, 0, 0};
      const int k0 = ch * 8;
      if (r >= k0 && r < k0 + 8) {
        const int e = r - k0;
        v[e >> 1] = (e & 1) ? (cinv << 16) : cinv;
      }
      st_shared_v4(sI + (ch >> 3) * 16384 + swz_offset(r, ch & 7, 128), v[0], v[1], v[2], v[3]);
    }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // Warp roles.  The SM's warp arbiter favours the highest warp id, so the latency-critical
  // single-thread roles (producer, MMA issuer) live in the last warpgroup: under full softmax
  // load they still get an issue slot as soon as their barrier completes.
  //   warps 0-3 / 4-7: softmax slots 0 / 1   warps 8-11: epilogue
  //   warp 12: TMA producer   warp 13: MMA issuer   warp 14: mask packer
  if (w >= 12) {
    setmaxnreg_dec56();
    if (w == 12 && lane == 0) {
      // =========================================================== TMA producer
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      if (BIAS) tma_prefetch_desc(&tm_b);
      int m_s[2] = {0, 0}, j_s[2] = {0, 0};
      Unit un_s[2] = {decode_unit((int)blockIdx.x, nq, a.H),
                      decode_unit((int)blockIdx.x + G, nq, a.H)};
      for (int t = 0; t < TA; ++t) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (t >= (s ? TB : TA)) continue;
          const int m = m_s[s], j = j_s[s];
          const Unit un = un_s[s];
          const int e = ring_idx(s, t);
          const int st = e % NKV;
          if (j == 0) {
            const int qb = s * NQ + (m % NQ), use = m / NQ;
            mbar_wait(BAR(Q_EMPTY + qb), (use & 1) ^ 1);
            mbar_arrive_expect_tx(BAR(Q_FULL + qb), kTile);
            tma_load_4d(sQ + qb * kTile, &tm_q, BAR(Q_FULL + qb), 0, un.qt * 128, un.h, un.b);
          }
          unsigned long long* pd = (a.dbg && e < 64) ? a.dbg + 148 * 8 * 32 * 8 + ((size_t)blockIdx.x * 64 + e) * 4 : nullptr;
          if (pd) pd[0] = clock64();
          mbar_wait(BAR(KV_EMPTY + st), ((e / NKV) & 1) ^ 1);
          if (pd) pd[1] = clock64();
          mbar_arrive_expect_tx(BAR(KV_FULL + st), 2 * kTile);
          tma_load_4d(sKV + st * 2 * kTile, &tm_k, BAR(KV_FULL + st), 0, j * 128, un.h, un.b);
          tma_load_4d(sKV + st * 2 * kTile + kTile, &tm_v, BAR(KV_FULL + st), 0, j * 128, un.h,
                      un.b);
          if (BIAS) {
            const int bs = e % NB;
            const int bc = a.bias_batched ? un.b : 0;
            mbar_wait(BAR(B_EMPTY + bs), ((e / NB) & 1) ^ 1);
            mbar_arrive_expect_tx(BAR(B_FULL + bs), 32768);
            for (int r = 0; r < 2; ++r) {
              if (BIAS == 1)  // rows q, cols k
                tma_load_4d(sBias + bs * 32768 + r * 16384, &tm_b, BAR(B_FULL + bs),
                            j * 128 + r * 64, un.qt * 128, un.h, bc);
              else            // rows k, cols q
                tma_load_4d(sBias + bs * 32768 + r * 16384, &tm_b, BAR(B_FULL + bs),
                            un.qt * 128 + r * 64, j * 128, un.h, bc);
            }
          }
          if (++j_s[s] == nk) {
            j_s[s] = 0;
            m_s[s] = m + 1;
            un_s[s] = decode_unit((int)blockIdx.x + (2 * (m + 1) + s) * G, nq, a.H);
          }
        }
      }
    } else if (w == 14 && !all_keys_kept) {
      // =========================================================== mask packer (whole warp)
      // Packs the key-validity bits of every ring entry into maskw[stage]; the byte loads of
      // entry e+1 are issued before the ballots of entry e (software pipelined).
      int j0 = 0, j1 = 0, m0 = 0, m1 = 0;
      int b0u = decode_unit((int)blockIdx.x, nq, a.H).b;
      int b1u = decode_unit((int)blockIdx.x + G, nq, a.H).b;
      const int E = TA + TB;
      auto next_entry = [&](int e, int& b, int& j) {
        const int s = (e < 2 * TB) ? (e & 1) : 0;
        if (s == 0) {
          b = b0u; j = j0;
          if (++j0 == nk) { j0 = 0; ++m0; b0u = decode_unit((int)blockIdx.x + (2 * m0) * G, nq, a.H).b; }
        } else {
          b = b1u; j = j1;
          if (++j1 == nk) { j1 = 0; ++m1; b1u = decode_unit((int)blockIdx.x + (2 * m1 + 1) * G, nq, a.H).b; }
        }
      };
      auto load4 = [&](int b, int j, uint32_t (&raw)[4]) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int k = j * 128 + i * 32 + lane;
          raw[i] = k < a.Lk ? (a.mask ? (uint32_t)a.mask[(int64_t)b * a.mask_s0 +
                                                            (int64_t)k * a.mask_s1]
                                      : 1u)
                            : 0u;
        }
      };
      uint32_t raw_next[4] = {0, 0, 0, 0};
      int bb, jj;
      if (E > 0) {
        next_entry(0, bb, jj);
        load4(bb, jj, raw_next);
      }
      for (int e = 0; e < E; ++e) {
        uint32_t raw[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) raw[i] = raw_next[i];
        if (e + 1 < E) {
          next_entry(e + 1, bb, jj);
          load4(bb, jj, raw_next);
        }
        uint32_t words[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) words[i] = __ballot_sync(0xffffffffu, raw[i] != 0);
        const int st = e % NKV;
        if (lane == 0) {
          mbar_wait(BAR(KV_EMPTY + st), ((e / NKV) & 1) ^ 1);
          uint32_t* mwp = maskw + st * 8;
          mwp[0] = words[0]; mwp[1] = words[1]; mwp[2] = words[2]; mwp[3] = words[3];
          mwp[4] = (words[0] & words[1] & words[2] & words[3]) == ~0u;
          mbar_arrive(BAR(MW_FULL + st));
        }
        __syncwarp();
      }
    } else if (w == 13 && lane == 0) {
      // =========================================================== MMA issuer
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idesc_b = make_idesc_bf16(128, 128, 0, BIAS == 1 ? 1 : 0);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, DP, 0, 1);
      // Readiness probes with a per-stream condition cursor: a condition observed satisfied is
      // never probed again (each mbarrier test costs ~150 cycles), so one pass of the event
      // loop costs at most one probe per stream.
      auto ready_S = [&](int s, int t, int& c) {
        const int m = t / nk, j = t - m * nk;
        const int e = ring_idx(s, t);
        if (c == 0) {
          if (j == 0 && !mbar_try_wait(BAR(Q_FULL + s * NQ + m % NQ), (m / NQ) & 1)) return false;
          c = 1;
        }
        if (c == 1) {
          if (!mbar_try_wait(BAR(KV_FULL + e % NKV), (e / NKV) & 1)) return false;
          c = 2;
        }
        if (c == 2) {
          if (BIAS && !mbar_try_wait(BAR(B_FULL + e % NB), (e / NB) & 1)) return false;
          c = 3;
        }
        if (c == 3) {
          if (t >= 1 && !mbar_try_wait(BAR(S_EMPTY + s), (t - 1) & 1)) return false;
          c = 4;
        }
        return true;
      };
      auto ready_PV = [&](int s, int t, int& c) {
        const int m = t / nk, j = t - m * nk;
        if (c == 0) {
          if (!mbar_try_wait(BAR(P_FULL + s), t & 1)) return false;
          c = 1;
        }
        if (c == 1) {
          if (j == 0 && m >= 1 && !mbar_try_wait(BAR(O_EMPTY + s), (m - 1) & 1)) return false;
          c = 2;
        }
        return true;
      };
      auto issue_S = [&](int s, int t) {
        const int m = t / nk, j = t - m * nk;
        const int qb = s * NQ + m % NQ;
        const int e = ring_idx(s, t), st = e % NKV;
        if (a.dbg && e < 64) a.dbg[148 * 8 * 32 * 8 + ((size_t)blockIdx.x * 64 + e) * 4 + 2] = clock64();
        tc_fence_after();
        const uint32_t tS = tmem + s * 256;
        const uint32_t kb = sKV + st * 2 * kTile;
#pragma unroll
        for (int kk = 0; kk < DP / 16; ++kk)
          umma_bf16(tS, make_sdesc(sQ + qb * kTile + kk * 32, 16, 8 * kRowBytes, kSw),
                    make_sdesc(kb + kk * 32, 16, 8 * kRowBytes, kSw), idesc_s, kk > 0);
        if (BIAS) {
          const uint32_t bb = sBias + (e % NB) * 32768;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t ad = make_sdesc(sI + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, kSw128);
            const uint64_t bd =
                BIAS == 1 ? make_sdesc(bb + kk * 2048, 16384, 1024, kSw128)          // MN-major
                          : make_sdesc(bb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, kSw128);
            umma_bf16(tS, ad, bd, idesc_b, 1u);
          }
          umma_commit(BAR(B_EMPTY + e % NB));
        }
        umma_commit(BAR(S_FULL + s));
        if (j == nk - 1) umma_commit(BAR(Q_EMPTY + qb));
      };
      auto issue_PV = [&](int s, int t) {
        const int j = t % nk;
        const int e = ring_idx(s, t), st = e % NKV;
        if (a.dbg && e < 64) a.dbg[148 * 8 * 32 * 8 + ((size_t)blockIdx.x * 64 + e) * 4 + 3] = clock64();
        tc_fence_after();
        const uint32_t tP = tmem + s * 256 + 128, tO = tmem + s * 256 + 192;
        const uint32_t vb = sKV + st * 2 * kTile + kTile;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16_ts(tO, tP + kk * 8, make_sdesc(vb + kk * 16 * kRowBytes, 16384, 8 * kRowBytes, kSw),
                       idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        umma_commit(BAR(O_FULL + s));
        umma_commit(BAR(KV_EMPTY + st));
      };
      // event loop: S(t) of a slot may run ahead of its PV(t-1) by one tile (one S buffer per
      // slot, released by the softmax as soon as S is in registers)
      int nS0 = 0, nS1 = 0, nPV0 = 0, nPV1 = 0;
      int cS0 = 0, cS1 = 0, cP0 = 0, cP1 = 0;
      while (nPV0 < TA || nPV1 < TB) {
        if (nPV0 < nS0 && ready_PV(0, nPV0, cP0)) { issue_PV(0, nPV0++); cP0 = 0; }
        if (nS0 < TA && nS0 <= nPV0 + 1 && ready_S(0, nS0, cS0)) { issue_S(0, nS0++); cS0 = 0; }
        if (nPV1 < nS1 && ready_PV(1, nPV1, cP1)) { issue_PV(1, nPV1++); cP1 = 0; }
        if (nS1 < TB && nS1 <= nPV1 + 1 && ready_S(1, nS1, cS1)) { issue_S(1, nS1++); cS1 = 0; }
      }
    }
  } else if (w < 8) {
    setmaxnreg_inc184();
    // ============================================================= softmax warpgroups
    const int s = w >> 2;           // slot
    const int qd = w & 3;           // TMEM lane quadrant
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    const uint32_t tS = tmem + s * 256 + lane_base, tP = tS + 128, tO = tS + 192;
    const int Ts = s ? TB : TA;
    const float c2 = a.scale * kLog2e;  // S -> log2 units
    const uint64_t c2x2 = f2_pack(c2, c2);
    float m_ref = -INFINITY, l_run = 0.f;  // m_ref in raw-S units
    int m = 0, j = 0;
    for (int t = 0; t < Ts; ++t) {
      if (j == 0) {
        m_ref = -INFINITY;
        l_run = 0.f;
      }
      const int e = ring_idx(s, t);
      const int kst = e % NKV;
      unsigned long long* dbgp = nullptr;
      if (a.dbg && lane == 0 && t < 32)
        dbgp = a.dbg + (((size_t)blockIdx.x * 8 + w) * 32 + t) * 8;
      if (dbgp) dbgp[0] = clock64();
      mbar_wait(BAR(S_FULL + s), t & 1);
      tc_fence_after();
      if (dbgp) dbgp[1] = clock64();
      float x[128];
      {
        uint32_t r0[32], r1[32], r2[32], r3[32];
        tmem_ld32(tS, r0);
        tmem_ld32(tS + 32, r1);
        tmem_ld32(tS + 64, r2);
        tmem_ld32(tS + 96, r3);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          x[i] = __uint_as_float(r0[i]);
          x[32 + i] = __uint_as_float(r1[i]);
          x[64 + i] = __uint_as_float(r2[i]);
          x[96 + i] = __uint_as_float(r3[i]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(BAR(S_EMPTY + s));  // S is in registers: next S may start
      if (dbgp) dbgp[2] = clock64();
      if (a.flags & 128) {  // experiment: no softmax work
        if (!all_keys_kept) mbar_wait(BAR(MW_FULL + kst), (e / NKV) & 1);
        if (t >= 1) mbar_wait(BAR(O_FULL + s), (t - 1) & 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(BAR(P_FULL + s));
        if (j == nk - 1) {
          __syncwarp();
          if (lane == 0) mbar_arrive(BAR(ST_FULL + s * 2 + (m & 1)));
        }
        if (++j == nk) { j = 0; ++m; }
        continue;
      }
      if (!all_keys_kept) {  // key mask packed by the mask warp for this K/V stage
        mbar_wait(BAR(MW_FULL + kst), (e / NKV) & 1);
        if (!maskw[kst * 8 + 4]) {
          const uint4 mw4 = *reinterpret_cast<const uint4*>(maskw + kst * 8);
          const uint32_t mw[4] = {mw4.x, mw4.y, mw4.z, mw4.w};
#pragma unroll
          for (int c = 0; c < 128; ++c) x[c] = ((mw[c >> 5] >> (c & 31)) & 1u) ? x[c] : -INFINITY;
        }
      }
      // tile row max (raw S units): 8 independent 3-input-max chains
      float mx8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx8[i] = fmaxf(x[i], x[8 + i]);
#pragma unroll
      for (int c = 16; c < 128; c += 16)
#pragma unroll
        for (int i = 0; i < 8; ++i) mx8[i] = fmax3(mx8[i], x[c + i], x[c + 8 + i]);
      const float mx = fmax3(fmax3(mx8[0], mx8[1], mx8[2]), fmax3(mx8[3], mx8[4], mx8[5]),
                             fmaxf(mx8[6], mx8[7]));
      if (dbgp) dbgp[3] = clock64();
      // lazy online-softmax rescale (threshold 8 in log2 units)
      const float m_new = fmaxf(m_ref, mx);
      if (j == 0) {
        m_ref = m_new;
      } else {
        const bool need = (m_new - m_ref) * c2 > 8.f;
        if (__any_sync(0xffffffffu, need)) {
          const float alpha = need ? fast_exp2((m_ref - m_new) * c2) : 1.f;
          mbar_wait(BAR(O_FULL + s), (t - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c0 = 0; c0 < DP; c0 += 8) {
            uint32_t r[8];
            tmem_ld8(tO + c0, r);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 8; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
            tmem_st8(tO + c0, r);
          }
          tmem_wait_st();
          l_run *= alpha;
          if (need) m_ref = m_new;
        }
      }
      const float negm = m_ref == -INFINITY ? 0.f : -m_ref * c2;
      const uint64_t negm2 = f2_pack(negm, negm);
      uint64_t lsum[4] = {0, 0, 0, 0};  // 4 independent f32x2 partial sums (0.0f bits)
      uint32_t pk[64];
      if (dbgp) dbgp[4] = clock64();
      const int nexp = (a.flags & 32) ? 0 : 64;  // experiment: skip the exps (wrong results)
      if (nexp == 0)
#pragma unroll
        for (int i = 0; i < 64; ++i) pk[i] = 0;
#pragma unroll
      for (int i = 0; i < nexp; ++i) {
        float y0, y1;
        f2_unpack(f2_fma(f2_pack(x[2 * i], x[2 * i + 1]), c2x2, negm2), y0, y1);
        const float p0 = fast_exp2(y0), p1 = fast_exp2(y1);
        lsum[i & 3] = f2_add(lsum[i & 3], f2_pack(p0, p1));
        pk[i] = pack_bf16(p0, p1);
      }
      if (dbgp) dbgp[5] = clock64();
      // the previous PV of this slot must be done reading P before we overwrite it
      if (t >= 1) mbar_wait(BAR(O_FULL + s), (t - 1) & 1);
      tmem_st32(tP, *reinterpret_cast<uint32_t(*)[32]>(pk));
      tmem_st32(tP + 32, *reinterpret_cast<uint32_t(*)[32]>(pk + 32));
      tmem_wait_st();
      {
        const uint64_t l2 = f2_add(f2_add(lsum[0], lsum[1]), f2_add(lsum[2], lsum[3]));
        float l0, l1;
        f2_unpack(l2, l0, l1);
        l_run += l0 + l1;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(BAR(P_FULL + s));
      if (dbgp) dbgp[6] = clock64();
      if (j == nk - 1) {  // hand (l, m·scale) of the unit to the epilogue warpgroup
        const int row = qd * 32 + lane;
        float* st = stat + ((s * 2 + (m & 1)) * 2) * 128;
        st[row] = l_run;
        st[128 + row] = m_ref == -INFINITY ? -INFINITY : m_ref * a.scale;
        __syncwarp();
        if (lane == 0) mbar_arrive(BAR(ST_FULL + s * 2 + (m & 1)));
      }
      if (++j == nk) {
        j = 0;
        ++m;
      }
      if (dbgp) dbgp[7] = clock64();
    }
  } else {
    setmaxnreg_dec80();
    // ============================================================= epilogue warpgroup
    const int qd = w & 3;
    const int row = qd * 32 + lane;
    const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
    // gate rows are prefetched one unit ahead so their load latency overlaps the previous
    // unit's epilogue (the epilogue must never throttle the PV -> O_EMPTY -> PV chain)
    auto load_g = [&](int n, uint32_t (&gp4)[DP / 2]) {
#pragma unroll
      for (int i = 0; i < DP / 2; ++i) gp4[i] = 0u;
      if (!a.g || n >= N) return;
      const Unit un = decode_unit((int)blockIdx.x + n * G, nq, a.H);
      const int q = un.qt * 128 + row;
      if (q >= a.Lq) return;
      const __nv_bfloat16* gp = a.g + (int64_t)un.b * a.g_sb + (int64_t)un.h * a.g_sh +
                                (int64_t)q * a.g_sl;
#pragma unroll
      for (int d0 = 0; d0 < DP; d0 += 8) {
        if (d0 < a.D) {
          const uint4 v = *reinterpret_cast<const uint4*>(gp + d0);
          gp4[d0 / 2] = v.x; gp4[d0 / 2 + 1] = v.y; gp4[d0 / 2 + 2] = v.z; gp4[d0 / 2 + 3] = v.w;
        }
      }
    };
    uint32_t gnext[DP / 2];
    load_g(0, gnext);
    for (int n = 0; n < N; ++n) {
      const int s = n & 1, m = n >> 1;
      const int t_last = m * nk + nk - 1;
      const Unit un = decode_unit((int)blockIdx.x + n * G, nq, a.H);
      const int q = un.qt * 128 + row;
      const bool qv = q < a.Lq;
      uint32_t gpk[DP / 2];
#pragma unroll
      for (int i = 0; i < DP / 2; ++i) gpk[i] = gnext[i];
      load_g(n + 1, gnext);
      mbar_wait(BAR(ST_FULL + s * 2 + (m & 1)), (m >> 1) & 1);
      mbar_wait(BAR(O_FULL + s), t_last & 1);
      tc_fence_after();
      if (a.flags & 64) {  // experiment: no epilogue work
        __syncwarp();
        if (lane == 0) mbar_arrive(BAR(O_EMPTY + s));
        continue;
      }
      uint32_t ov[DP];
      const uint32_t tO = tmem + s * 256 + 192 + lane_base;
      if (DP == 16) {
        uint32_t r[16];
        tmem_ld16(tO, r);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) ov[i] = r[i];
      } else {
#pragma unroll
        for (int c0 = 0; c0 < DP; c0 += 32) {
          uint32_t r[32];
          tmem_ld32(tO + c0, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) ov[c0 + i] = r[i];
        }
      }
      const float* st = stat + ((s * 2 + (m & 1)) * 2) * 128;
      const float l_run = st[row], m_nat = st[128 + row];
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(BAR(O_EMPTY + s));
      if (qv) {
        const float inv = l_run > 0.f ? fast_rcp(l_run) : 0.f;
        __nv_bfloat16* op = a.o + (int64_t)un.b * a.o_sb + (int64_t)un.h * a.o_sh +
                            (int64_t)q * a.o_sl;
#pragma unroll
        for (int d0 = 0; d0 < DP; d0 += 8) {
          if (d0 >= a.D) break;
          float gv[8];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (a.g) {
              gv[2 * i] = inv * fast_sigmoid(bf16_lo(gpk[d0 / 2 + i]));
              gv[2 * i + 1] = inv * fast_sigmoid(bf16_hi(gpk[d0 / 2 + i]));
            } else {
              gv[2 * i] = gv[2 * i + 1] = inv;
            }
          }
          uint4 o4;
          o4.x = pack_bf16(__uint_as_float(ov[d0]) * gv[0], __uint_as_float(ov[d0 + 1]) * gv[1]);
          o4.y = pack_bf16(__uint_as_float(ov[d0 + 2]) * gv[2], __uint_as_float(ov[d0 + 3]) * gv[3]);
          o4.z = pack_bf16(__uint_as_float(ov[d0 + 4]) * gv[4], __uint_as_float(ov[d0 + 5]) * gv[5]);
          o4.w = pack_bf16(__uint_as_float(ov[d0 + 6]) * gv[6], __uint_as_float(ov[d0 + 7]) * gv[7]);
          *reinterpret_cast<uint4*>(op + d0) = o4;
        }
        a.lse[((int64_t)un.b * a.H + un.h) * a.Lq + q] =
            l_run > 0.f ? (m_nat == -INFINITY ? 0.f : m_nat) + __logf(l_run) : -INFINITY;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tmem);
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

template <int DP, int BIAS>
static cudaError_t launch_fwd_ws_t(const FwdLaunch& L, cudaStream_t st) {
  auto kern = fwd_ws_kernel<DP, BIAS>;
  const size_t smem = FwdCfg<DP, BIAS>::kSmem;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) {
    fprintf(stderr, "evo fwd_ws: cudaFuncSetAttribute(smem=%zu) failed: %s\n", smem,
            cudaGetErrorString(e));
    return e;
  }
  const int nq = (L.args.Lq + 127) / 128;
  const long long U = (long long)L.args.B * L.args.H * nq;
  if (U == 0) return cudaSuccess;
  const int grid = (int)(U < num_sms() ? U : num_sms());
  kern<<<grid, 512, smem, st>>>(L.tm_q, L.tm_k, L.tm_v, L.tm_b, L.args);
  e = cudaGetLastError();
  if (e != cudaSuccess)
    fprintf(stderr, "evo fwd_ws: launch (grid=%d smem=%zu) failed: %s\n", grid, smem,
            cudaGetErrorString(e));
  return e;
}

cudaError_t launch_fwd_ws_bf16(const FwdLaunch& L, int DP, int bias_mode, cudaStream_t st) {
#define EVO_FWS_CASE(dp, bm) \
  if (DP == dp && bias_mode == bm) return launch_fwd_ws_t<dp, bm>(L, st);
  EVO_FWS_CASE(16, 0) EVO_FWS_CASE(16, 1) EVO_FWS_CASE(16, 2)
  EVO_FWS_CASE(32, 0) EVO_FWS_CASE(32, 1) EVO_FWS_CASE(32, 2)
  EVO_FWS_CASE(64, 0) EVO_FWS_CASE(64, 1) EVO_FWS_CASE(64, 2)
#undef EVO_FWS_CASE
  return cudaErrorInvalidValue;
}

}  // namespace evo

extern "C" int evo_debug_fwd_timing(void* host, size_t bytes) {
  if (bytes > sizeof(evo::g_fwd_dbg)) bytes = sizeof(evo::g_fwd_dbg);
  return (int)cudaMemcpyFromSymbol(host, evo::g_fwd_dbg, bytes);
}
