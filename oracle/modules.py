"""AF2 module-level oracle wrappers (numpy, fp64) — TEST INFRASTRUCTURE ONLY.

These write the four attention modules that PAPER.md L169 (§2.1) names directly from the
AlphaFold2 supplementary algorithms the paper cites, each in its own notation,
so that the closed-form identity "ending-node attention equals starting-node attention on the
transposed pair" (north star) is a real check rather than a tautology:

* ``msa_row_attention_with_pair_bias``  — AF2 Alg. 7 (Fig. 6 missing)
* ``msa_column_attention``              — AF2 Alg. 8
* ``triangle_attention_start``          — AF2 Alg. 13:  a_ijk = softmax_k(q_ij·k_ik/√c + b_jk)
* ``triangle_attention_end``            — AF2 Alg. 14:  a_ijk = softmax_k(q_ij·k_kj/√c + b_ki)

Each returns the gated attention output o (before the output Linear, which is outside the
attention core) with shape [..., H, c], plus the projections it used so tests can feed the same
q/k/v/g/bias to the core oracle and to the CUDA path.

Mask convention: hard mask (reading R5) — masked keys get weight exactly 0 and a query
with no surviving key gets o = 0.
"""
from __future__ import annotations

import numpy as np


def layer_norm(x, gamma, beta, eps=1e-5):
    """LayerNorm over the last axis (two-pass mean/variance, fp64)."""
    x = np.asarray(x, np.float64)
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * gamma + beta


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def _masked_softmax(logits, keep):
    """softmax over the last axis with a hard mask; rows with no kept key -> all zeros."""
    logits = np.where(keep, logits, -np.inf)
    m = logits.max(axis=-1, keepdims=True)
    live = np.isfinite(m)
    m = np.where(live, m, 0.0)
    e = np.where(keep, np.exp(logits - m), 0.0)
    s = e.sum(axis=-1, keepdims=True)
    return np.where(live, e / np.where(live, s, 1.0), 0.0)


def make_params(rng, c_in, c_pair, H, c, with_pair_bias=True):
    """Random module weights (fp64): LN(x), q/k/v/g projections, pair LN + bias projection."""
    p = {
        "ln_g": 1.0 + 0.1 * rng.standard_normal(c_in), "ln_b": 0.1 * rng.standard_normal(c_in),
        "wq": rng.standard_normal((c_in, H, c)) / np.sqrt(c_in),
        "wk": rng.standard_normal((c_in, H, c)) / np.sqrt(c_in),
        "wv": rng.standard_normal((c_in, H, c)) / np.sqrt(c_in),
        "wg": rng.standard_normal((c_in, H, c)) / np.sqrt(c_in),
        "bg": np.ones((H, c)),  # AF2 initialises the gate bias to 1
    }
    if with_pair_bias:
        p["lnz_g"] = 1.0 + 0.1 * rng.standard_normal(c_pair)
        p["lnz_b"] = 0.1 * rng.standard_normal(c_pair)
        p["wb"] = rng.standard_normal((c_pair, H))
    return p


def _proj(x, p):
    q = np.einsum("...a,ahc->...hc", x, p["wq"])
    k = np.einsum("...a,ahc->...hc", x, p["wk"])
    v = np.einsum("...a,ahc->...hc", x, p["wv"])
    g = np.einsum("...a,ahc->...hc", x, p["wg"]) + p["bg"]
    return q, k, v, g


def msa_row_attention_with_pair_bias(m, z, p, msa_mask=None):
    """AF2 Alg. 7.  m [S,R,c_m], z [R,R,c_z], msa_mask [S,R].  o[s,i,h] = σ(g_si)
    Σ_j softmax_j(q_si·k_sj/√c + b_ij) v_sj.  Returns (o [S,R,H,c], proj)."""
    x = layer_norm(m, p["ln_g"], p["ln_b"])
    q, k, v, g = _proj(x, p)
    c = q.shape[-1]
    b = np.einsum("ija,ah->hij", layer_norm(z, p["lnz_g"], p["lnz_b"]), p["wb"])  # [H,R,R]
    logits = np.einsum("sihc,sjhc->shij", q, k) / np.sqrt(c) + b[None]
    S, R = m.shape[:2]
    keep = np.ones((S, 1, 1, R), bool) if msa_mask is None else (msa_mask[:, None, None, :] != 0)
    a = _masked_softmax(logits, keep)
    o = sigmoid(g) * np.einsum("shij,sjhc->sihc", a, v)
    return o, {"q": q, "k": k, "v": v, "g": g, "bias": b}


def msa_column_attention(m, p, msa_mask=None):
    """AF2 Alg. 8.  o[s,i,h] = σ(g_si) Σ_t softmax_t(q_si·k_ti/√c) v_ti.  Returns (o, proj)."""
    x = layer_norm(m, p["ln_g"], p["ln_b"])
    q, k, v, g = _proj(x, p)
    c = q.shape[-1]
    logits = np.einsum("sihc,tihc->ihst", q, k) / np.sqrt(c)
    S, R = m.shape[:2]
    keep = (np.ones((R, 1, 1, S), bool) if msa_mask is None
            else (msa_mask.T[:, None, None, :] != 0))
    a = _masked_softmax(logits, keep)
    o = sigmoid(g) * np.einsum("ihst,tihc->sihc", a, v)
    return o, {"q": q, "k": k, "v": v, "g": g}


def _tri_proj(z, p):
    x = layer_norm(z, p["ln_g"], p["ln_b"])
    q, k, v, g = _proj(x, p)
    b = np.einsum("ija,ah->hij", x, p["wb"])  # bias from the same normalised pair (Alg. 13 l.3)
    return q, k, v, g, b


def triangle_attention_start(z, p, pair_mask=None):
    """AF2 Alg. 13 (around the starting node).  a_ijk = softmax_k(q_ij·k_ik/√c + b_jk);
    o_ij = g_ij ⊙ Σ_k a_ijk v_ik.  Key (i,k) kept iff pair_mask[i,k].  Returns (o, proj)."""
    q, k, v, g, b = _tri_proj(z, p)
    c = q.shape[-1]
    logits = np.einsum("ijhc,ikhc->ihjk", q, k) / np.sqrt(c) + b[None]  # b[h,j,k]
    N = z.shape[0]
    keep = (np.ones((N, 1, 1, N), bool) if pair_mask is None
            else (pair_mask[:, None, None, :] != 0))  # keep[i,...,k]
    a = _masked_softmax(logits, keep)
    o = sigmoid(g) * np.einsum("ihjk,ikhc->ijhc", a, v)
    return o, {"q": q, "k": k, "v": v, "g": g, "bias": b}


def triangle_attention_end(z, p, pair_mask=None):
    """AF2 Alg. 14 (around the ending node), written directly — NOT via a transpose.
    a_ijk = softmax_k(q_ij·k_kj/√c + b_ki); o_ij = g_ij ⊙ Σ_k a_ijk v_kj.
    Key (k,j) kept iff pair_mask[k,j].  Returns (o, proj)."""
    q, k, v, g, b = _tri_proj(z, p)
    c = q.shape[-1]
    logits = (np.einsum("ijhc,kjhc->jhik", q, k) / np.sqrt(c)
              + np.transpose(b, (0, 2, 1))[None])  # b_ki laid out as [h, i, k]
    N = z.shape[0]
    keep = (np.ones((N, 1, 1, N), bool) if pair_mask is None
            else (pair_mask.T[:, None, None, :] != 0))  # keep[j,...,k] = mask[k,j]
    a = _masked_softmax(logits, keep)
    o = sigmoid(g) * np.einsum("jhik,kjhc->ijhc", a, v)
    return o, {"q": q, "k": k, "v": v, "g": g, "bias": b}
