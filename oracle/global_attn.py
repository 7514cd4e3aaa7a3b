"""fp64 oracle of the extra-MSA global column attention core (AF2
supplementary Alg. 19 MSAColumnGlobalAttention, cited at PAPER.md L178; the extra-MSA stack is
PAPER.md L156).

TEST INFRASTRUCTURE ONLY (same rule as oracle/evo_oracle.c).

The attention core of Alg. 19, lines 3, 5 and 6 (the LayerNorm and the projections of lines 1,
2, 4, 7 are outside the core, as for the other modules), per column b and head h:
  3: q̄[b,h,:] = mean over the kept sequences s of q[b,s,h,:]           (reading R19: masked mean)
  5: a[b,h,t] = softmax_t( scale · q̄[b,h,:]·k[b,t,:] )  over kept t     (k, v: one shared head)
  6: o[b,s,h,:] = σ(g[b,s,h,:]) ⊙ Σ_t a[b,h,t] v[b,t,:]
Hard mask (R5): masked sequences get weight 0; a column with no kept sequence gives q̄ = 0,
lse = -inf, o = 0 and zero gradients.  Backward by the chain rule, written out in the same
order.  Parity: pinned by tests/test_oracle_global_attn.py.
"""
from __future__ import annotations

import numpy as np


def _sig(x):
    return 1.0 / (1.0 + np.exp(-x))


def global_attn_fwd(q, k, v, g, mask, scale):
    """q, g [B,S,H,D]; k, v [B,S,D]; mask [B,S] (nonzero = keep).  Returns o [B,S,H,D],
    lse [B,H], qbar [B,H,D], attn [B,H,D]."""
    q, k, v, g = (np.asarray(x, np.float64) for x in (q, k, v, g))
    m = (np.asarray(mask) != 0).astype(np.float64)
    cnt = m.sum(axis=1)                                             # [B]
    qbar = np.einsum("bs,bshd->bhd", m, q) / np.maximum(cnt, 1.0)[:, None, None]
    logits = scale * np.einsum("bhd,btd->bht", qbar, k)
    logits = np.where(m[:, None, :] > 0, logits, -np.inf)
    mx = logits.max(axis=2, keepdims=True)
    keep_any = cnt > 0
    mx = np.where(keep_any[:, None, None], mx, 0.0)
    e = np.exp(logits - mx)
    ssum = e.sum(axis=2, keepdims=True)
    a = np.where(keep_any[:, None, None], e / np.where(ssum > 0, ssum, 1.0), 0.0)
    lse = np.where(keep_any[:, None], (mx + np.log(np.where(ssum > 0, ssum, 1.0)))[..., 0], -np.inf)
    attn = np.einsum("bht,btd->bhd", a, v)
    o = _sig(g) * attn[:, None]
    return o, lse, qbar, attn


def global_attn_bwd(q, k, v, g, mask, scale, dout):
    """Gradients of <dout, o> w.r.t. q, k, v, g."""
    q, k, v, g, dout = (np.asarray(x, np.float64) for x in (q, k, v, g, dout))
    m = (np.asarray(mask) != 0).astype(np.float64)
    cnt = m.sum(axis=1)
    o, lse, qbar, attn = global_attn_fwd(q, k, v, g, mask, scale)
    logits = scale * np.einsum("bhd,btd->bht", qbar, k)
    a = np.where(m[:, None, :] > 0, np.exp(logits - np.where(np.isfinite(lse), lse, 0.0)[..., None]), 0.0)
    a = np.where((cnt > 0)[:, None, None], a, 0.0)
    sg = _sig(g)
    dattn = np.einsum("bshd,bshd->bhd", dout, sg)                 # line 6 through σ(g)
    dg = dout * attn[:, None] * sg * (1.0 - sg)
    dv = np.einsum("bht,bhd->btd", a, dattn)
    da = np.einsum("bhd,btd->bht", dattn, v)
    Dh = (a * da).sum(axis=2, keepdims=True)
    dlogit = a * (da - Dh)                                          # softmax backward
    dqbar = scale * np.einsum("bht,btd->bhd", dlogit, k)
    dk = scale * np.einsum("bht,bhd->btd", dlogit, qbar)
    dq = (m / np.maximum(cnt, 1.0)[:, None])[:, :, None, None] * dqbar[:, None]  # line 3
    return {"dq": dq, "dk": dk, "dv": dv, "dg": dg}
