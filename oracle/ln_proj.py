"""fp64 oracle of the LayerNorm + batched q/k/v/g projection (PAPER.md
L273 "fused LayerNorm, MHA and its previous four GEMMs", L296-297 "GEMM Batching: four linear
layers have no dependency on each other"; SPEC.md L174-182 qkvg_project; AF2 Alg. 7 l.1-4).

TEST INFRASTRUCTURE ONLY (same rule as oracle/evo_oracle.c).

  y = LayerNorm(x)·γ + β               (two-pass mean / biased variance, fp64)
  [q | k | v | g_logits] = y · [W_q | W_k | W_v | W_g] + [0 | 0 | 0 | b_g]
The four projections are computed as four separate products (the definition), so the pin
"equal to four separate GEMMs" is checked against the fused kernel, not assumed.
"""
from __future__ import annotations

import numpy as np


def ln_qkvg_fwd(x, gamma, beta, W, bias_g=None, eps=1e-5):
    """x [rows, C]; gamma, beta [C]; W [C, 4, N1] (q, k, v, g blocks of width N1 = H·D);
    bias_g [N1] or None.  Returns Y [rows, 4, N1] (q, k, v, gate logits)."""
    x = np.asarray(x, np.float64)
    mean = x.mean(axis=1, keepdims=True)
    var = ((x - mean) ** 2).mean(axis=1, keepdims=True)
    y = (x - mean) / np.sqrt(var + eps) * np.asarray(gamma, np.float64) + np.asarray(beta, np.float64)
    W = np.asarray(W, np.float64)
    out = np.stack([y @ W[:, j, :] for j in range(4)], axis=1)
    if bias_g is not None:
        out[:, 3, :] += np.asarray(bias_g, np.float64)
    return out


def linear_fwd(x, W, b=None):
    """out[r, n] = Σ_c x[r, c]·W[n, c] + b[n] (the output projection, [ext] AF2 Alg. 7 l.7);
    W in the nn.Linear [out, in] layout.  The definition, in fp64."""
    out = np.asarray(x, np.float64) @ np.asarray(W, np.float64).T
    if b is not None:
        out = out + np.asarray(b, np.float64)
    return out


def ln_proj_bwd(x, gamma, beta, W, dout, eps=1e-5, ln=True):
    """fp64 backward of out = LN(x)·Wᵀ + b (ln=True) or out = x·Wᵀ + b (ln=False), written from
    the chain rule in the order of the forward (the LayerNorm backward of
    [ext] Ba et al., as the paper's fused LN + GEMMs need it):
      dy = dout·W;  dW = doutᵀ·y;  db = Σ_r dout
      LN:  x̂ = (x − μ)/sqrt(σ² + eps),  dγ = Σ_r dy⊙x̂,  dβ = Σ_r dy,
           g = dy⊙γ,  dx = (g − mean_c(g) − x̂·mean_c(g⊙x̂)) / sqrt(σ² + eps)
    x [rows, C]; W [N, C] (nn.Linear layout); dout [rows, N].  Returns dict dx, dgamma, dbeta,
    dW, db (dgamma/dbeta None without LN)."""
    x = np.asarray(x, np.float64)
    W = np.asarray(W, np.float64)
    dout = np.asarray(dout, np.float64)
    if ln:
        mean = x.mean(axis=1, keepdims=True)
        var = ((x - mean) ** 2).mean(axis=1, keepdims=True)
        rstd = 1.0 / np.sqrt(var + eps)
        xh = (x - mean) * rstd
        y = xh * np.asarray(gamma, np.float64) + np.asarray(beta, np.float64)
    else:
        y = x
    dy = dout @ W
    out = {"dW": dout.T @ y, "db": dout.sum(axis=0), "dgamma": None, "dbeta": None}
    if ln:
        out["dgamma"] = (dy * xh).sum(axis=0)
        out["dbeta"] = dy.sum(axis=0)
        g = dy * np.asarray(gamma, np.float64)
        out["dx"] = (g - g.mean(axis=1, keepdims=True) - xh * (g * xh).mean(axis=1, keepdims=True)) * rstd
    else:
        out["dx"] = dy
    return out
