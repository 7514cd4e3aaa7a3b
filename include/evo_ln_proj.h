/*
 * evo_ln_proj.h — C ABI of the fused LayerNorm + batched input projection that feeds the
 * attention core: the "previous four GEMMs" of PAPER.md L273 and the GEMM batching of PAPER.md
 * L296-297 ("Four linear layers have no dependency on each other. We bundled these linear layers
 * into batch operations"); SPEC.md L174-182 qkvg_project.
 *
 *   for every row r:   μ_r = Σ_c x[r,c] / C,   σ²_r = Σ_c (x[r,c] − μ_r)² / C     (fp32)
 *                      y[r,c] = bf16( (x[r,c] − μ_r)·rstd_r·γ_c + β_c ),  rstd_r = 1/sqrt(σ²_r + eps)
 *                      out[r,n] = bf16( Σ_c y[r,c]·W[n,c] + b[n] )                  (fp32 accumulate)
 *
 * W is the four projection weights stacked along the output axis, in the nn.Linear [out, in]
 * layout: rows [0, H·D) = W_q, then W_k, W_v, W_g (any stacking — the kernel sees one [N, C]
 * matrix, so the MSA-global q/k/v/g of Alg. 19 with single-head k, v also fits).  b is an
 * optional fp32 [N] vector (AF2: zeros for q, k, v and the gate bias for g; NULL = no bias).
 * `out` row r holds the N projections contiguously, so each of q, k, v, g is a strided view
 * [rows, H, D] that evo_attn_fwd takes directly (row stride out_ld, head stride D).
 *
 * Layouts: x [rows][C] bf16, row stride x_ld elements (multiple of 8, c unit-stride); W [N][C]
 * bf16 dense; out [rows][N] bf16, row stride out_ld (>= N, multiple of 8); γ, β [C] fp32;
 * mean, rstd [rows] fp32 (written when non-NULL, for a LayerNorm backward).
 *
 * Supported: C in {64, 128, 256}, N a multiple of 64 (<= 2048), rows >= 0, eps > 0.  Device
 * pointers, 16-byte-aligned tensors, asynchronous on `stream`, errors returned (EVO_E_*), details
 * in evo_last_error_detail(), no allocation (conventions of evo_attn.h).
 */
#ifndef EVO_LN_PROJ_H
#define EVO_LN_PROJ_H

#include <stddef.h>
#include <stdint.h>

#include "evo_attn.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t rows;     /* M: rows of x / out                                          */
  int32_t C;        /* input channels: 64, 128 or 256                               */
  int32_t N;        /* stacked output features (4·H·D for q|k|v|g), multiple of 64  */
  float eps;        /* LayerNorm epsilon, > 0 (AF2: 1e-5)                           */
  int64_t x_ld;     /* row stride of x, elements                                    */
  int64_t out_ld;   /* row stride of out, elements                                  */
} evo_ln_proj_desc_t;

evo_status_t evo_ln_proj_fwd(const evo_ln_proj_desc_t* d, const void* x, const float* gamma,
                             const float* beta, const void* W, const float* b, void* out,
                             float* mean, float* rstd, void* stream);

/* The same kernel without the LayerNorm: out[r,n] = bf16( Σ_c x[r,c]·W[n,c] + b[n] ) — the
 * attention module's output projection (SURVEY.md §8(f) f2 "and the output projection";
 * [ext] AF2 Alg. 7 l.7 / Alg. 13 l.7, cited at PAPER.md L178), e.g. x = the gated attention
 * output [rows, H·D] and W = W_o [c, H·D].  Same layouts, limits and conventions as above; eps,
 * gamma, beta, mean and rstd do not apply. */
evo_status_t evo_linear_fwd(const evo_ln_proj_desc_t* d, const void* x, const void* W,
                            const float* b, void* out, void* stream);

/* Backward of evo_ln_proj_fwd (the chain rule through PAPER.md L273's fused
 * LayerNorm + four GEMMs).  Given dout = ∂L/∂out [rows][N] bf16 (row stride d->out_ld):
 *
 *   dy[r,c]  = Σ_n dout[r,n]·W[n,c]                                     (fp32, tcgen05)
 *   x̂[r,c]  = (x[r,c] − mean_r)·rstd_r                                 (mean, rstd: the forward's)
 *   dx[r,c]  = bf16( rstd_r·( dy·γ − (1/C)Σ_c dy·γ − x̂·(1/C)Σ_c dy·γ·x̂ ) )   row stride d->x_ld
 *   dγ[c]    = Σ_r dy[r,c]·x̂[r,c],   dβ[c] = Σ_r dy[r,c]                 (fp32 [C])
 *   dW[n,c]  = Σ_r dout[r,n]·y[r,c],  y = bf16(x̂·γ + β) (the forward's MMA operand)   (fp32 [N][C])
 *   db[n]    = Σ_r dout[r,n]                                             (fp32 [N], skipped if NULL)
 *
 * Every sum over rows is taken in a fixed order (bitwise repeatable).  `dx` is written, never read;
 * x, W, mean, rstd and dout are read only.  Workspace: evo_ln_proj_bwd_workspace_bytes(d) bytes of
 * device memory, 16-byte aligned, owned by the caller (partials of dγ/dβ, dW and db).
 * Supported: C in {64, 128, 256}; N a multiple of 128 (<= 2048).  Same alignment, error and
 * stream conventions as evo_ln_proj_fwd. */
size_t evo_ln_proj_bwd_workspace_bytes(const evo_ln_proj_desc_t* d);
evo_status_t evo_ln_proj_bwd(const evo_ln_proj_desc_t* d, const void* x, const float* gamma,
                             const float* beta, const void* W, const float* mean,
                             const float* rstd, const void* dout, void* dx, float* dgamma,
                             float* dbeta, float* dW, float* db, void* workspace,
                             size_t workspace_bytes, void* stream);

/* Backward of evo_linear_fwd (no LayerNorm): dx = bf16(dout·W), dW = doutᵀ·x, db = Σ_r dout.
 * Same layouts, workspace query (evo_ln_proj_bwd_workspace_bytes) and conventions. */
evo_status_t evo_linear_bwd(const evo_ln_proj_desc_t* d, const void* x, const void* W,
                            const void* dout, void* dx, float* dW, float* db, void* workspace,
                            size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EVO_LN_PROJ_H */
