"""The four Evoformer attention modules mapped onto the one attention core by strides only.

PAPER.md L169 lists the Evoformer's MHA modules (MSA row attention with pair bias, MSA column
attention, triangle attention around the starting and the ending node); AF2 supplementary
Alg. 7/8/13/14 (cited at PAPER.md L178) define them.  Every one of them is the same gated
pair-bias attention of include/evo_attn.h on a different (batch, attended) axis pair of the
projection tensors, so this module only builds strided views — no copies, no arithmetic.

Storage conventions:
  MSA projections   x[s, r, h, d]  (S = N_seq rows, R = N_res columns)
  pair projections  x[i, j, h, d]
  bias storage      E[q, h, k]     (head-major inside a query row: the layout the DAP all-gather
                                    produces, include/evo_dap.h)
  masks             msa_mask[s, r], pair_mask[i, j]  (uint8, 1 = keep)

  module  batch b  attended l  logical [B,H,L,D] view      bias[h,q,k]          mask[b,k]
  row     s        r           x.permute(0,2,1,3)          E[q,h,k]             msa_mask
  col     r        s           x.permute(1,2,0,3)          none                 msa_maskᵀ
  start   i        j           x.permute(0,2,1,3)          E[q,h,k] (b_jk)      pair_mask
  end     j        i           x.permute(1,2,0,3)          E[k,h,q] (b_ki)      pair_maskᵀ
"""
from __future__ import annotations

KINDS = ("row", "col", "start", "end")
_BATCH_MAJOR = {"row": True, "col": False, "start": True, "end": False}


def x_view(kind, x):
    """Logical [B, H, L, D] view of a projection tensor stored [A0, A1, H, D]."""
    return x.permute(0, 2, 1, 3) if _BATCH_MAJOR[kind] else x.permute(1, 2, 0, 3)


def x_storage(kind, xv):
    """Inverse of x_view: the [A0, A1, H, D] storage view of a logical [B, H, L, D] tensor."""
    return xv.permute(0, 2, 1, 3) if _BATCH_MAJOR[kind] else xv.permute(2, 0, 1, 3)


def bias_view(kind, E):
    """Logical bias[h, q, k] of the bias storage E[., h, .] (None passes through)."""
    if E is None:
        return None
    return E.permute(1, 2, 0) if kind == "end" else E.permute(1, 0, 2)


def bias_storage(kind, bv):
    """Inverse of bias_view (used for dbias, which the core writes with the bias strides)."""
    if bv is None:
        return None
    return bv.permute(2, 0, 1) if kind == "end" else bv.permute(1, 0, 2)


def mask_view(kind, mask):
    if mask is None:
        return None
    return mask if _BATCH_MAJOR[kind] else mask.t()


def attention_fwd(kind, q, k, v, g, E, mask, attn):
    """Module forward through `attn` (the evoattn binding).  Returns (o storage, o view, lse)."""
    qv, kv, vv = x_view(kind, q), x_view(kind, k), x_view(kind, v)
    gv = None if g is None else x_view(kind, g)
    o, lse = attn.fwd(qv, kv, vv, bias_view(kind, E), mask_view(kind, mask), gv)
    return x_storage(kind, o), o, lse


def attention_bwd(kind, q, k, v, g, E, mask, o_view, lse, dout_storage, attn, workspace=None):
    """Module backward.  Returns dq, dk, dv, dg (projection storage views) and dE (fp32 bias
    storage view, or None)."""
    qv, kv, vv = x_view(kind, q), x_view(kind, k), x_view(kind, v)
    gv = None if g is None else x_view(kind, g)
    r = attn.bwd(qv, kv, vv, o_view, lse, x_view(kind, dout_storage), bias_view(kind, E),
                 mask_view(kind, mask), gv, workspace=workspace)
    return {"dq": x_storage(kind, r["dq"]), "dk": x_storage(kind, r["dk"]),
            "dv": x_storage(kind, r["dv"]),
            "dg": None if r["dg"] is None else x_storage(kind, r["dg"]),
            "dE": bias_storage(kind, r["dbias"])}
