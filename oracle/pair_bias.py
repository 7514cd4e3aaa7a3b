"""fp64 oracle of the pair-bias side path: LayerNorm(z) followed by
LinearNoBias(c_z -> H) into the head-major bias, and its backward.

TEST INFRASTRUCTURE ONLY (same rule as oracle/evo_oracle.c): only tests/, __graft_entry__ and
bench.py may import it; the product path never does.

Written from the definitions, in the paper's order:
  PAPER.md L276-283 (§3.3.1 LayerNormalization): per-row statistics, y = ẑ·γ + β; the backward's
    weight/bias gradients are column sums over rows (the paper's two-step reduction is an
    implementation of that sum; here it is one plain sum);
  SPEC.md L137-153 (layernorm_fwd / layernorm_bwd);
  AF2 supplementary Alg. 7 l.3 / Alg. 13 l.3 (cited at PAPER.md L178): b_ij^h = LinearNoBias(LN(z_ij)).
The statistics use the textbook two-pass mean/variance in fp64 (the kernel's single pass is an
implementation choice).  Parity: pinned by tests/test_oracle_pair_bias.py.
"""
from __future__ import annotations

import numpy as np


def pair_bias_fwd(z, gamma, beta, W, eps=1e-5):
    """z [Li, Lj, C]; gamma, beta [C]; W [C, H].  Returns (bias [H, Li, Lj], mean, rstd [Li, Lj])."""
    z = np.asarray(z, np.float64)
    mean = z.mean(axis=-1)
    var = ((z - mean[..., None]) ** 2).mean(axis=-1)          # biased variance (LayerNorm)
    rstd = 1.0 / np.sqrt(var + eps)
    zhat = (z - mean[..., None]) * rstd[..., None]
    y = zhat * np.asarray(gamma, np.float64) + np.asarray(beta, np.float64)
    bias = np.einsum("ijc,ch->hij", y, np.asarray(W, np.float64))
    return bias, mean, rstd


def pair_bias_bwd(z, gamma, beta, W, dbias, eps=1e-5):
    """Gradients of <dbias, bias(z)> w.r.t. z, gamma, beta, W (dbias [H, Li, Lj])."""
    z = np.asarray(z, np.float64)
    gamma = np.asarray(gamma, np.float64)
    W = np.asarray(W, np.float64)
    dbias = np.asarray(dbias, np.float64)
    C = z.shape[-1]
    mean = z.mean(axis=-1)
    var = ((z - mean[..., None]) ** 2).mean(axis=-1)
    rstd = 1.0 / np.sqrt(var + eps)
    zhat = (z - mean[..., None]) * rstd[..., None]
    y = zhat * gamma + np.asarray(beta, np.float64)
    dy = np.einsum("hij,ch->ijc", dbias, W)                    # through Wᵀ
    dW = np.einsum("ijc,hij->ch", y, dbias)
    dgamma = (dy * zhat).sum(axis=(0, 1))
    dbeta = dy.sum(axis=(0, 1))
    g = dy * gamma                                             # d loss / d ẑ
    dz = rstd[..., None] * (g - g.mean(axis=-1, keepdims=True)
                            - zhat * (g * zhat).mean(axis=-1, keepdims=True))
    assert dz.shape[-1] == C
    return {"dz": dz, "dgamma": dgamma, "dbeta": dbeta, "dW": dW}
