/*
 * evo_pair_bias.h — C ABI of the pair-bias side path: fused LayerNorm(z) + LinearNoBias(c_z -> H)
 * writing the head-major attention bias, and its backward.
 *
 * What it computes (§3.3.1 "LayerNormalization (LN)": "each CUDA thread block
 * [processes] multiple input rows", "normalization statistics were computed in a single pass",
 * and in the backward "weight and bias gradients were computed by a two-step reduction ... This
 * design effectively avoided expensive atomic operations"; SPEC.md L137-153 layernorm_fwd/bwd;
 * the bias projection of AF2 Alg. 7 l.3 / Alg. 13 l.3, cited at PAPER.md L178):
 *
 *   for every pair row (i, j):   mean = Σ_c z[i,j,c] / C,   var = Σ_c z² / C − mean²  (fp32, one pass)
 *                                rstd = 1 / sqrt(var + eps),  ẑ_c = (z_c − mean)·rstd
 *                                y_c  = ẑ_c·γ_c + β_c
 *                                bias[h, i, j] = Σ_c y_c · W[c, h]          (no bias term)
 *
 * Backward, given dbias[h, i, j] (fp32, e.g. evo_attn_bwd's output through the same strides):
 *   dy_c = Σ_h dbias[h,i,j]·W[c,h];   dW[c,h] = Σ_rows y_c·dbias[h];   dγ_c = Σ_rows dy_c·ẑ_c;
 *   dβ_c = Σ_rows dy_c;   dz_c = rstd·(dy_c·γ_c − mean_c'(dy·γ) − ẑ_c·mean_c'(dy·γ·ẑ))
 * with dW, dγ, dβ reduced in two steps (per-block partials in the workspace, then a column
 * reduction) — deterministic, no atomics.
 *
 * Layouts: z is [Li][Lj][C] through element strides z_str = (i, j, c) with c unit-stride; the
 * bias (bf16 out) and dbias (fp32 in) use b_str = (h, i, j) element strides, any order — so the
 * same call writes the [H, L, L] head-major bias, its transposed (end-node) orientation, or the
 * DAP storage [L, H, L].  γ, β: [C] fp32; W: [C][H] fp32 row-major; mean, rstd: [Li·Lj] fp32
 * (row r = i·Lj + j), written by the forward and read by the backward; dz: bf16 with z_str.
 *
 * Supported: C in {32, 64, 128, 256}, H in {4, 8, 16} (AF2: 8 for MSA row, 4 for triangle
 * attention), eps > 0.  Conventions as evo_attn.h: device
 * pointers, 16-byte-aligned tensors, asynchronous on `stream`, errors returned (EVO_E_*), details
 * in evo_last_error_detail(), no allocation on the hot path (workspace from the caller).
 */
#ifndef EVO_PAIR_BIAS_H
#define EVO_PAIR_BIAS_H

#include <stddef.h>
#include <stdint.h>

#include "evo_attn.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t Li, Lj;       /* pair rows: i extent, j extent                              */
  int32_t C;            /* channels c_z: 32, 64, 128 or 256                            */
  int32_t H;            /* heads: 4, 8 or 16                                           */
  float eps;            /* LayerNorm epsilon, > 0 (AF2: 1e-5)                          */
  int64_t z_str[3];     /* element strides of z / dz for (i, j, c); c must be 1        */
  int64_t b_str[3];     /* element strides of bias / dbias for (h, i, j)               */
} evo_pair_bias_desc_t;

evo_status_t evo_pair_bias_fwd(const evo_pair_bias_desc_t* d, const void* z, const float* gamma,
                               const float* beta, const float* W, void* bias, float* mean,
                               float* rstd, void* stream);

size_t evo_pair_bias_bwd_workspace_bytes(const evo_pair_bias_desc_t* d);

evo_status_t evo_pair_bias_bwd(const evo_pair_bias_desc_t* d, const void* z, const float* gamma,
                               const float* beta, const float* W, const float* mean,
                               const float* rstd, const float* dbias, void* dz, float* dgamma,
                               float* dbeta, float* dW, void* workspace, size_t workspace_bytes,
                               void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EVO_PAIR_BIAS_H */
