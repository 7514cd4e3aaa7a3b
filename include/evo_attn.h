/*
 * evo_attn.h — C ABI of the B200-native Evoformer gated multi-head attention with pair bias.
 *
 * The operation (§3.3.1 "Multi Head Attention": "a pair bias term is added to
 * the logits matrix before the softmax operation ... fuse all operations in MHA"; SPEC.md
 * L155-173 attn_pair_bias_fwd/bwd; AF2 supplementary Alg. 7/8/13/14 cited at PAPER.md L178):
 *
 *   for every batch row b (the axis that shares the bias), head h, query q:
 *     s[k]  = scale * Σ_d Q[b,h,q,d] K[b,h,k,d] + bias[(b,)h,q,k]       for keys with mask[b,k]≠0
 *     p[k]  = softmax_k(s)  (p = 0 at masked keys)       lse[b,h,q] = log Σ_k exp(s[k])
 *     O[b,h,q,d] = sigmoid(G[b,h,q,d]) * Σ_k p[k] V[b,h,k,d]      (gate absent: factor 1)
 *
 * and its gradient with respect to q, k, v, g and bias (bias gradient summed over b when the
 * bias is shared).  The four Evoformer modules of PAPER.md L169 map onto this one core by
 * strides only:
 *     MSA row (Alg. 7):  B = N_seq, L = N_res, shared bias b_ij, mask = msa_mask[s,:]
 *     MSA column (Alg. 8): B = N_res, L = N_seq, no bias, mask = msa_mask[:, r] (strided view)
 *     triangle start (Alg. 13): B = i, L = j, shared bias b_jk, mask = pair_mask[i,:]
 *     triangle end (Alg. 14):   B = j, L = i, shared bias b_ki (transposed view: q-stride 1),
 *                               mask = pair_mask[:, j] (strided view)
 *
 * Precision (reading R7): EVO_BF16 = bf16 inputs/outputs, fp32 accumulation and fp32
 * softmax statistics; P and dS are rounded to bf16 only as tensor-core operands.  EVO_F32 = fp32
 * inputs/outputs computed entirely in fp32 FFMA with accurate expf (verification mode).
 * lse is always fp32; dbias is always fp32.
 *
 * Mask (reading R5): hard mask.  A masked key gets weight exactly 0 and never
 * influences any output or gradient provided its K/V/bias values are finite.  A query row with
 * no kept key returns o = 0, lse = -inf, dq = dg = 0 and contributes nothing to dk/dv/dbias.
 *
 * Ownership and calling convention:
 *   - Every pointer is caller-owned DEVICE memory (q,k,v,g,o,lse,dout,dq,dk,dv,dg,dbias,bias,
 *     mask,workspace).  The library never allocates or frees on the hot path.
 *   - Calls are asynchronous and stream-ordered on `stream` (a cudaStream_t; NULL = legacy
 *     default stream).  Inputs are never written.  Outputs must not alias inputs.
 *   - Pointers must be 16-byte aligned; every non-unit stride, in bytes, must be a multiple of
 *     16 (TMA); the head dimension D is unit-stride.  Violations return EVO_E_ALIGN.
 *   - Errors are returned, never thrown; evo_last_error_detail() (thread-local) names the
 *     offending field.  Asynchronous device faults surface at the caller's next synchronisation.
 *   - Reentrant; the only global state is a per-device one-time kernel-attribute setup.
 */
#ifndef EVO_ATTN_H
#define EVO_ATTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EVO_ATTN_ABI_VERSION 1

typedef enum {
  EVO_OK = 0,
  EVO_E_INVALID = 1,     /* NULL descriptor / required pointer, bad enum, non-positive scale  */
  EVO_E_SHAPE = 2,       /* inconsistent shape or bias kind ("shape error")      */
  EVO_E_ALIGN = 3,       /* pointer not 16-B aligned or stride not a multiple of 16 B         */
  EVO_E_UNSUPPORTED = 4, /* D not in {8,16,32,64}, or bias with neither q nor k unit-stride   */
  EVO_E_WORKSPACE = 5,   /* workspace NULL or smaller than evo_attn_bwd_workspace_bytes()     */
  EVO_E_CUDA = 6         /* a CUDA launch / driver call failed                                */
} evo_status_t;

typedef enum { EVO_BF16 = 0, EVO_F32 = 1 } evo_dtype_t;

typedef enum {
  EVO_BIAS_NONE = 0,
  EVO_BIAS_SHARED = 1,   /* bias[h,q,k], broadcast over B ("broadcastable [H,L,L]") */
  EVO_BIAS_PER_BATCH = 2 /* bias[b,h,q,k] ("[B,H,L,L]")                           */
} evo_bias_kind_t;

typedef struct {
  int64_t B;            /* attention batch rows (the bias-sharing axis), >= 0                  */
  int32_t H;            /* heads, >= 1                                                          */
  int32_t Lq, Lk;       /* query / key lengths, >= 0 (any value; tile padding is inert)       */
  int32_t D;            /* head dim: 8, 16, 32 or 64                                            */
  int32_t dtype;        /* evo_dtype_t: element type of q,k,v,g,bias,o,dout,dq,dk,dv,dg         */
  float scale;          /* logits = scale*q·k + bias; canonically fp32(1/sqrt(D)); > 0          */
  /* element strides of the (b, h, l) axes; d is unit-stride.  dout uses o_str; dq, dk, dv, dg
     use q_str, k_str, v_str, g_str respectively. */
  int64_t q_str[3], k_str[3], v_str[3], g_str[3], o_str[3];
  int32_t bias_kind;    /* evo_bias_kind_t                                                      */
  int64_t bias_str[4];  /* element strides (b, h, q, k); b ignored for SHARED; exactly one of
                           the q / k strides must be 1 (k=1: row/start; q=1: end-node view).
                           dbias (fp32) is written with these same element strides.            */
  int32_t has_mask;     /* mask[b*mask_str[0] + k*mask_str[1]] (uint8): nonzero keep, 0 drop  */
  int64_t mask_str[2];
  int32_t has_gate;     /* 0: o = attention output (gate factor 1); g, dg must be NULL        */
} evo_attn_desc_t;

/* Host-only descriptor validation (no CUDA call): EVO_OK or the error the compute call would
   return for these arguments. */
evo_status_t evo_attn_validate(const evo_attn_desc_t* desc);

/* Forward.  o [B,H,Lq,D] (o_str, dtype); lse [B,H,Lq] contiguous fp32 (-inf for rows with no
   kept key).  bias NULL iff bias_kind == NONE; mask NULL iff !has_mask; g NULL iff !has_gate. */
evo_status_t evo_attn_fwd(const evo_attn_desc_t* desc, const void* q, const void* k,
                          const void* v, const void* bias, const uint8_t* mask, const void* g,
                          void* o, float* lse, void* stream);

/* Bytes of device workspace evo_attn_bwd needs for this descriptor (0 is possible). */
size_t evo_attn_bwd_workspace_bytes(const evo_attn_desc_t* desc);

/* Backward (recompute; needs the forward's o and lse).  dq, dk, dv overwritten (q/k/v strides,
   dtype); dg overwritten (g strides) — NULL iff !has_gate; dbias overwritten, fp32, bias_str
   strides, summed over B for SHARED — NULL iff bias_kind == NONE. */
evo_status_t evo_attn_bwd(const evo_attn_desc_t* desc, const void* q, const void* k,
                          const void* v, const void* bias, const uint8_t* mask, const void* g,
                          const void* o, const float* lse, const void* dout, void* dq, void* dk,
                          void* dv, void* dg, float* dbias, void* workspace,
                          size_t workspace_bytes, void* stream);

const char* evo_status_string(evo_status_t status);
const char* evo_last_error_detail(void);
int evo_abi_version(void);
/* Number of device kernels the calling thread's last evo_attn_fwd / evo_attn_bwd launched
   (memsets excluded); used by bench.py to report gpu_launches. */
int evo_last_launch_count(void);

/* Profiling hook (bench.py): while enabled on the calling thread, every kernel that
   evo_attn_fwd / evo_attn_bwd launches is bracketed by cudaEventRecord on the call's stream into
   caller-created events: kernel i runs between events[2i] and events[2i+1]; its name is
   evo_trace_label(i).  `events` is an array of cudaEvent_t; NULL disables.  Returns 0, or
   EVO_E_INVALID for a negative capacity.  Recording stops silently when capacity is reached. */
int evo_trace_enable(void** events, int capacity);
int evo_trace_count(void);           /* kernels recorded since evo_trace_enable */
const char* evo_trace_label(int i);  /* NULL if out of range */

#ifdef __cplusplus
}
#endif
#endif /* EVO_ATTN_H */
