// evo_kernels.cuh — argument blocks and launchers shared by the kernels and the C-ABI layer.
#pragma once
#include "evo_common.cuh"

namespace evo {

// Unsigned division by a runtime divisor d >= 1 without the integer-divide sequence (which goes
// through the XU pipe): q = (umulhi(n, m) + n) >> l with l = ceil(log2 d),
// m = floor(2^32 (2^l - d) / d) + 1; exact for n < 2^31 (round-up method, Hacker's Delight 10-8).
struct FastDiv {
  uint32_t d, m, l;
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  f.l = 0;
  while ((1ull << f.l) < d) ++f.l;
  f.m = (uint32_t)(((1ull << 32) * ((1ull << f.l) - d)) / d + 1);
  return f;
}
EVO_DEV uint32_t fdiv(uint32_t n, const FastDiv& f) { return (__umulhi(n, f.m) + n) >> f.l; }

// sets the thread-local text evo_last_error_detail() returns (evo_api.cu)
void set_error_detail(const char* msg);

constexpr int kMaxMaskWords = 512;  // Lk <= 16384
constexpr int kMaxLk = kMaxMaskWords * 32;

// ------------------------------------------------------------------ forward (bf16, tcgen05)
struct FwdArgs {
  int B, H, Lq, Lk, D;
  float scale;       // logits = scale * q·k + bias
  float scale_log2;  // scale * log2(e)
  int bias_batched;  // per-batch bias: TMA coordinate 3 = b
  const uint8_t* mask;
  int64_t mask_s0, mask_s1;
  const __nv_bfloat16* g;
  int64_t g_sb, g_sh, g_sl;
  __nv_bfloat16* o;
  int64_t o_sb, o_sh, o_sl;
  float* lse;
};
// forward (evo_fwd_occ.cu): K/V maps with 64-row boxes, Q read by threads
struct FwdOccLaunch {
  CUtensorMap tm_k, tm_v, tm_b;
  FwdArgs args;
  const __nv_bfloat16* q;
  int64_t q_sb, q_sh, q_sl;
};
cudaError_t launch_fwd_occ_bf16(const FwdOccLaunch& L, int DP, int bias_mode, cudaStream_t st);

// ------------------------------------------------------------------ backward (bf16)
struct BwdPreArgs {  // D_q, lse2, dA, dg  (all rows of [B,H,Lq])
  int B, H, Lq, D;
  const void* o;  // bf16 or f32 (dtype)
  const void* dout;
  int64_t o_sb, o_sh, o_sl;  // also dout strides
  const void* g;
  int64_t g_sb, g_sh, g_sl;  // also dg strides
  void* dg;
  const float* lse;
  float* lse2;   // lse*log2e, +inf for rows with no kept key (bf16 path) | lse (f32 path)
  float* Dvec;   // Σ_d dO·o
  void* dA;      // dO·sigmoid(g) (NULL when no gate), element strides below, d unit-stride
  int64_t a_sb, a_sh, a_sl;
  int negate;    // store -lse2 and -D (the fused backward's operand form)
  float* zacc;   // optional fp32 [B,H,Lq,D] accumulator zeroed here (strides below), else NULL
  int64_t z_sb, z_sh, z_sl;
  FastDiv fd_H, fd_Lq;  // filled by launch_bwd_pre
};
cudaError_t launch_bwd_pre(const BwdPreArgs& a, int f32, cudaStream_t st);

struct BwdMainArgs {  // dK, dV (and dQ partials) — CTA per (b, h, key tile)
  int B, H, Lq, Lk, D;
  float scale, scale_log2;
  int bias_batched;
  const uint8_t* mask;
  int64_t mask_s0, mask_s1;
  const float* lse2;
  const float* Dvec;
  __nv_bfloat16* dk;
  int64_t k_sb, k_sh, k_sl;
  __nv_bfloat16* dv;
  int64_t v_sb, v_sh, v_sl;
  __nv_bfloat16* dq;  // direct store when there is a single key tile
  int64_t q_sb, q_sh, q_sl;
  float* dq_acc;      // otherwise nk fp32 parts [nk][B,H,Lq,D] (plain stores; dq_convert sums
                      // them in key-tile order, so dq is bitwise deterministic)
};
struct BwdMainLaunch {
  CUtensorMap tm_q, tm_k, tm_v, tm_da, tm_b;
  BwdMainArgs args;
};
inline size_t bwd_main_smem_bytes(int DP) {
  // Pt, dSt, bias[2] (128 KB) | K, V, Q[2], dA[2] tiles | vectors[2] (2 KB) | barriers
  return 131072 + 6 * 128 * (size_t)DP * 2 + 2048 + 16 * 8 + 16;
}
cudaError_t launch_bwd_main_bf16(const BwdMainLaunch& L, int DP, int bias_mode, cudaStream_t st);

struct BwdBiasArgs {  // dbias partials — CTA per (h, q tile, k tile, batch chunk)
  int B, H, Lq, Lk, D;
  float scale_log2;
  int bias_batched;
  int nchunks, chunk;  // batch rows per chunk
  const uint8_t* mask;
  int64_t mask_s0, mask_s1;
  const float* lse2;
  const float* Dvec;
  float* partial;  // shared: [nchunks][H][Lq][Lk]; per-batch: [B][H][Lq][Lk]
};
struct BwdBiasLaunch {
  CUtensorMap tm_q, tm_k, tm_v, tm_da, tm_b;
  BwdBiasArgs args;
};
inline size_t bwd_bias_smem_bytes(int DP) {
  // per stage: Q, K, V, dA tiles + bias tile; 2 stages; barriers
  return 2 * (4 * 128 * (size_t)DP * 2 + 32768 + 1024) + 16 * 8 + 16;
}
cudaError_t launch_bwd_bias_bf16(const BwdBiasLaunch& L, int DP, int bias_mode, cudaStream_t st);

// Single-pass backward (evo_bwd_pb.cu with a shared bias, Lq <= 384; evo_bwd_nb.cu without):
// CTA per (h, 128-key tile, batch chunk); dK, dV, dQ and the chunk's dbias partial in one pass.
struct BwdFusedArgs {
  int B, H, Lq, Lk, D;
  float scale, scale_log2;
  int nchunks, chunk;
  const __nv_bfloat16* bias;  // shared bias [h, q, k] with element strides below (or NULL)
  int64_t b_sh, b_sq, b_sk;
  const uint8_t* mask;
  int64_t mask_s0, mask_s1;
  const float* lse2;  // [B*H][Lq_pad]
  const float* Dvec;
  __nv_bfloat16* dk;
  int64_t k_sb, k_sh, k_sl;
  __nv_bfloat16* dv;
  int64_t v_sb, v_sh, v_sl;
  __nv_bfloat16* dq;  // direct store when there is a single key tile
  int64_t q_sb, q_sh, q_sl;
  float* dq_acc;      // otherwise fp32: dq_reduce ? ONE accumulator every key tile reduce-adds
                      // into : nk parts, key tile kt's part (plain stores) at
  int64_t p_part, p_sb, p_sh, p_sl;  // dq_acc + kt*p_part + b*p_sb + h*p_sh + q*p_sl
  float* partial;     // [nchunks][H][Lq_pad][Lk_pad] fp32 dbias partials
  int dq_reduce;  // 1 (only when nk == 2, so 0 + a + b is order-independent and dq stays bitwise
                  // deterministic): both key tiles reduce-add into ONE fp32 accumulator (zeroed
                  // by bwd_pre); 0: one part per key tile, summed in key-tile order by dq_convert
  int bmode;  // bias: 1 k-contiguous (tm_b box [256 q][64 k], [128 q][64 k] when Lq > 256),
              // 2 q-contiguous (box [128 k][64 q])
  int t0;          // first query tile (0; 2 in the Σ-only pass of a 256 < Lq <= 384 call)
  int sigma_only;  // 1: only Σ_b dSᵀ of query tiles t0.. (no gradients)
  int kloop;       // no-bias kernel: 1 = each CTA walks every key tile of its (b, h) rows and
                   // accumulates dQ of all query tiles in TMEM (bf16 dQ, no fp32 parts);
                   // 0 = one key tile per CTA (grid H x nk x chunks)
  int dq_pair;     // pair-bias kernel, exactly two key tiles: the two key tiles of a (h, chunk)
                   // run as a 2-CTA cluster; rank 1 sends its fp32 dQ tile through distributed
                   // shared memory and rank 0 stores dq = scale·(dQ_0 + dQ_1) in bf16
};
struct BwdFusedLaunch {
  CUtensorMap tm_q, tm_k, tm_v, tm_da, tm_b;
  CUtensorMap tm_dq, tm_dk, tm_dv;  // output maps (dq: bf16 over dq, or fp32 over the dQ parts)
  BwdFusedArgs args;
};
// eligibility + resources of the fused path for head-dim pad DP and padded Lq
inline bool bwd_fused_supported(int DP, int Lq_pad, bool bias) {
  // the Σ_b dSᵀ accumulator needs up to 256 TMEM columns (queries beyond 256 get a Σ-only
  // second pass) and the resident biasᵀ Lq_pad·256 B of smem, so with a bias Lq <= 384
  const int cols = (bias ? (Lq_pad < 256 ? Lq_pad : 256) : 0) + 128 + 3 * DP + 32;
  return (!bias || Lq_pad <= 384) && cols <= 512 && (DP == 16 || DP == 32);
}
inline int bwd_fused_nchunks(int B, int H, int nk, int num_sms, int* chunk) {
  const int groups = H * nk;
  int nch = num_sms / (groups > 0 ? groups : 1);
  if (nch < 1) nch = 1;
  if (nch > B) nch = B;
  const int ch = (B + nch - 1) / nch;
  *chunk = ch;
  return (B + ch - 1) / ch;
}
// the no-bias backward (evo_bwd_nb.cu): same launch block and workspace, one 128-query tile per
// hand-off (N = 128 Sᵀ/dPᵀ MMAs); DP 16 or 32
cudaError_t launch_bwd_nb_bf16(const BwdFusedLaunch& L, int DP, cudaStream_t st);
// the pair-bias kernel (evo_bwd_pb.cu) for a shared bias, Lq <= 384 (above 256: the BIG variant,
// then a Σ-only launch with t0 = 2, sigma_only = 1): 64-query hand-offs processed by all eight
// compute warps, Σ_b dSᵀ in TMEM; DP 16 or 32
cudaError_t launch_bwd_pb_bf16(const BwdFusedLaunch& L, int DP, cudaStream_t st);
// the key-tile loop of the no-bias kernel keeps nq dQ accumulators (DP columns each) in TMEM
// next to Sᵀ, dPᵀ, Pᵀ (320 columns), dV and dK
inline bool bwd_nb_kloop_fits(int DP, int nq) { return 320 + 2 * DP + nq * DP <= 512; }

struct ReduceArgs {  // dbias[h,q,k] (bias strides) = Σ_c partial[c][h][q][k]
  int nparts, H, Lq, Lk;
  int64_t nb;        // leading count of the destination (1 shared, B per-batch)
  const float* partial;
  float* dbias;
  int64_t s_b, s_h, s_q, s_k;
  int q_fast;        // destination is q-contiguous
};
cudaError_t launch_dbias_reduce(const ReduceArgs& a, cudaStream_t st);

struct ConvertArgs {  // dq = bf16(scale * Σ_p acc[p])
  int B, H, Lq, D;
  float scale;
  const float* acc;
  int nparts;
  int64_t part_stride;  // elements between parts
  int64_t p_sb, p_sh, p_sl;  // element strides of one part (d unit-stride)
  __nv_bfloat16* dq;
  int64_t q_sb, q_sh, q_sl;
  FastDiv fd_nd, fd_H, fd_Lq;  // filled by launch_dq_convert
};
cudaError_t launch_dq_convert(const ConvertArgs& a, cudaStream_t st);

// ------------------------------------------------------------------ fp32 verification path
struct F32Args {
  int B, H, Lq, Lk, D;
  float scale;
  const float *q, *k, *v, *g, *bias;
  int64_t q_sb, q_sh, q_sl, k_sb, k_sh, k_sl, v_sb, v_sh, v_sl, g_sb, g_sh, g_sl;
  int bias_kind;
  int64_t b_sb, b_sh, b_sq, b_sk;
  const uint8_t* mask;
  int64_t mask_s0, mask_s1;
  float* o;
  int64_t o_sb, o_sh, o_sl;
  float* lse;
  // backward
  const float* dout;
  const float* dA;    // [B,H,Lq,D] contiguous, or dout (then strides = o strides)
  int64_t a_sb, a_sh, a_sl;
  const float* lse_in;
  const float* Dvec;
  float *dq, *dk, *dv, *dbias;
};
cudaError_t launch_fwd_f32(const F32Args& a, cudaStream_t st);
cudaError_t launch_bwd_f32(const F32Args& a, cudaStream_t st, int* nlaunch);

cudaError_t launch_fill_empty(float* lse, int64_t nrows, void* o, int dtype, int B, int H,
                              int Lq, int D, int64_t o_sb, int64_t o_sh, int64_t o_sl,
                              cudaStream_t st);

}  // namespace evo
