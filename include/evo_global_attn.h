/*
 * evo_global_attn.h — C ABI of the extra-MSA global column attention core (SURVEY.md §8(f) row
 * f3; AF2 supplementary Alg. 19 MSAColumnGlobalAttention lines 3, 5, 6, cited at PAPER.md L178;
 * the extra-MSA stack: PAPER.md L156).
 *
 * For every column b (the residue axis of the extra MSA) and head h:
 *   q̄[b,h,:]   = Σ_s m[b,s]·q[b,s,h,:] / Σ_s m[b,s]                   (masked mean, reading R19)
 *   a[b,h,t]   = softmax_t( scale · q̄[b,h,:]·k[b,t,:] )  over kept t   (k, v: one shared head)
 *   o[b,s,h,:] = σ(g[b,s,h,:]) ⊙ Σ_t a[b,h,t]·v[b,t,:]
 * and the gradients w.r.t. q, k, v, g.  Hard mask (R5): masked sequences weigh 0; a column with
 * no kept sequence gives o = 0, lse = −inf and zero gradients.  The LayerNorm and projections of
 * Alg. 19 (lines 1, 2, 4, 7) are outside the core, as for the other modules.
 *
 * Layouts: q, g, o, dout, dq, dg: [B, S, H, D] through element strides (b, s, h) with d
 * unit-stride (o and dout share o_str; dq uses q_str, dg g_str); k, v, dk, dv: [B, S, D] through
 * (b, s) strides; mask: uint8 mask[b·s0 + s·s1] (1 keep).  bf16 tensors, fp32 statistics:
 * lse [B, H] and q̄ [B, H, D] are written by the forward and read by the backward.
 *
 * Supported: D in {8, 16, 32}, 1 <= H <= 16, H·S <= 16384 (the per-column score rows live in
 * shared memory), strides multiples of 8 elements except d.  Conventions as evo_attn.h (device
 * pointers, 16-byte alignment, stream-ordered, EVO_E_* status, evo_last_error_detail()).
 */
#ifndef EVO_GLOBAL_ATTN_H
#define EVO_GLOBAL_ATTN_H

#include <stddef.h>
#include <stdint.h>

#include "evo_attn.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t B;          /* columns (batch axis)                                  */
  int32_t S;          /* sequences attended over                               */
  int32_t H;          /* heads of q / g / o                                    */
  int32_t D;          /* head dim: 8, 16 or 32                                 */
  float scale;        /* canonically 1/sqrt(D)                                 */
  int64_t q_str[3];   /* (b, s, h) element strides of q / dq                   */
  int64_t k_str[2];   /* (b, s) element strides of k / dk                      */
  int64_t v_str[2];   /* (b, s) element strides of v / dv                      */
  int64_t g_str[3];   /* (b, s, h) element strides of g / dg                   */
  int64_t o_str[3];   /* (b, s, h) element strides of o / dout                 */
  int32_t has_mask;
  int64_t mask_str[2];
} evo_global_attn_desc_t;

evo_status_t evo_global_attn_fwd(const evo_global_attn_desc_t* d, const void* q, const void* k,
                                 const void* v, const uint8_t* mask, const void* g, void* o,
                                 float* lse, float* qbar, void* stream);

evo_status_t evo_global_attn_bwd(const evo_global_attn_desc_t* d, const void* q, const void* k,
                                 const void* v, const uint8_t* mask, const void* g,
                                 const float* lse, const float* qbar, const void* dout, void* dq,
                                 void* dk, void* dv, void* dg, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EVO_GLOBAL_ATTN_H */
