"""Pins for the fp64 oracle against what the paper and the mathematics fix.

None of these re-types the oracle's own loops: each compares the oracle with a library routine
(torch float64 SDPA / autograd), a closed form, an invariant, a special case, brute-force finite
differences, or an independently written module formulation (oracle/modules.py, AF2 Alg. 7/8/
13/14 in einsum notation).  A dropped term, wrong sign/index or transposed operand in
oracle/evo_oracle.c fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import modules as M
from synth.gen import attention_case

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = max(np.max(np.abs(b)) if b.size else 0.0, 1e-300)
    return float(np.max(np.abs(a - b)) / den) if a.size else 0.0


def _case(B=2, H=2, L=7, D=4, seed=0, **kw):
    c = attention_case(B, H, L, L, D, seed=seed, **kw)
    return {k: (v.astype(np.float64) if isinstance(v, np.ndarray) and v.dtype != np.uint8 else v)
            for k, v in c.items()}


def _probs(q, k, bias=None, mask=None, scale=1.0):
    """Read the attention probabilities out of the oracle: zero-pad the head dim of q and k to
    Lk (dot products unchanged) and use V = identity, so o = p exactly (no gate)."""
    B, H, Lq, D = q.shape
    Lk = k.shape[2]
    Dp = max(D, Lk)
    pad = lambda x: np.concatenate([x, np.zeros(x.shape[:3] + (Dp - D,))], -1)
    eye = np.zeros((B, H, Lk, Dp))
    eye[:, :, np.arange(Lk), np.arange(Lk)] = 1.0
    o, _ = oracle.attn_fwd(pad(q), pad(k), eye, bias=bias, mask=mask, scale=scale)
    return o[..., :Lk]


# ---------------------------------------------------------------- P10: worked example (golden)
def test_p10_golden_worked_example():
    spec = json.load(open(os.path.join(GOLDEN, "p10_worked_example.json")))
    env = {"exp": math.exp, "log": math.log}
    for c in spec["cases"]:
        q = np.array(c["q"]).reshape(1, 1, 2, 1)
        k = np.array(c["k"]).reshape(1, 1, 2, 1)
        v = np.array(c["v"]).reshape(1, 1, 2, 1)
        bias = None if c["bias"] is None else np.array(c["bias"]).reshape(1, 2, 2)
        g = None if c["g"] is None else np.array(c["g"]).reshape(1, 1, 2, 1)
        o, lse = oracle.attn_fwd(q, k, v, bias=bias, g=g, scale=c["scale"])
        closed_o = [eval(e, env) for e in c["o_closed_form"]]
        closed_lse = [eval(e, env) for e in c["lse_closed_form"]]
        closed_p = [eval(e, env) for e in c["p_row0_closed_form"]]
        np.testing.assert_allclose(closed_o, c["o"], rtol=0, atol=1e-15)
        np.testing.assert_allclose(closed_p, c["p_row0"], rtol=0, atol=1e-15)
        np.testing.assert_allclose(o.ravel(), closed_o, rtol=0, atol=1e-14)
        np.testing.assert_allclose(lse.ravel(), closed_lse, rtol=0, atol=1e-14)
        # p row 0 via V = one-hot columns (D=2): o = p when no gate
        if g is None:
            p = _probs(q, k, bias=bias, scale=c["scale"])
            np.testing.assert_allclose(p[0, 0, 0], closed_p, rtol=0, atol=1e-15)


# ---------------------------------------------------------------- P1: softmax rows sum to 1
def test_p1_rows_sum_to_one_and_shift_invariance():
    c = _case(B=2, H=3, L=9, D=4, seed=1, gate=False)
    L = 9
    p = _probs(c["q"], c["k"], bias=c["bias"], scale=c["scale"])
    assert np.all(p >= 0)
    assert np.max(np.abs(p.sum(-1) - 1.0)) <= 1e-15 * L
    # per-row constant added to the bias leaves o unchanged and shifts lse by it
    shift = np.random.default_rng(7).standard_normal((3, L, 1)) * 5
    o1, l1 = oracle.attn_fwd(c["q"], c["k"], c["v"], bias=c["bias"], scale=c["scale"])
    o2, l2 = oracle.attn_fwd(c["q"], c["k"], c["v"], bias=c["bias"] + shift, scale=c["scale"])
    assert _rel(o2, o1) <= 1e-14
    np.testing.assert_allclose(l2 - l1, np.broadcast_to(shift[..., 0], l1.shape), atol=1e-12)


# ---------------------------------------------------------------- P2: vanilla MHA = torch SDPA
def test_p2_vanilla_equals_torch_sdpa_fwd_and_autograd_bwd():
    torch = pytest.importorskip("torch")
    c = _case(B=3, H=2, L=11, D=8, seed=2, bias=None, gate=False)
    o, _ = oracle.attn_fwd(c["q"], c["k"], c["v"], scale=c["scale"])
    tq, tk, tv = (torch.tensor(c[n], dtype=torch.float64, requires_grad=True) for n in "qkv")
    ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, scale=c["scale"])
    assert _rel(o, ref.detach().numpy()) <= 1e-14
    do = torch.tensor(c["dout"], dtype=torch.float64)
    ref.backward(do)
    gr = oracle.attn_bwd(c["q"], c["k"], c["v"], c["dout"], scale=c["scale"])
    for name, t in (("dq", tq), ("dk", tk), ("dv", tv)):
        assert _rel(gr[name], t.grad.numpy()) <= 1e-13, name


def _torch_unfused(c, torch):
    """The unfused four-op composition in float64 torch, differentiated by autograd."""
    t = {n: torch.tensor(c[n], dtype=torch.float64, requires_grad=True)
         for n in ("q", "k", "v", "g", "bias") if c[n] is not None}
    logits = torch.einsum("bhqd,bhkd->bhqk", t["q"], t["k"]) * c["scale"]
    if "bias" in t:
        logits = logits + (t["bias"] if t["bias"].dim() == 4 else t["bias"][None])
    keep = None
    if c["mask"] is not None:
        keep = torch.tensor(c["mask"] != 0)[:, None, None, :]
        logits = logits.masked_fill(~keep, float("-inf"))
    p = torch.softmax(logits, -1)
    p = torch.nan_to_num(p, nan=0.0)  # fully-masked rows -> 0 (reading R5)
    a = torch.einsum("bhqk,bhkd->bhqd", p, t["v"])
    o = torch.sigmoid(t["g"]) * a if "g" in t else a
    return t, o


@pytest.mark.parametrize("bias", ["shared", "batch", None])
@pytest.mark.parametrize("gate", [True, False])
def test_p2_general_case_equals_torch_autograd(bias, gate):
    torch = pytest.importorskip("torch")
    c = _case(B=3, H=2, L=10, D=4, seed=3, bias=bias, gate=gate, mask="prefix")
    t, o_ref = _torch_unfused(c, torch)
    o, _ = oracle.attn_fwd(c["q"], c["k"], c["v"], bias=c["bias"], mask=c["mask"], g=c["g"],
                           scale=c["scale"])
    assert _rel(o, o_ref.detach().numpy()) <= 1e-14
    o_ref.backward(torch.tensor(c["dout"], dtype=torch.float64))
    gr = oracle.attn_bwd(c["q"], c["k"], c["v"], c["dout"], bias=c["bias"], mask=c["mask"],
                         g=c["g"], scale=c["scale"])
    for name, key in (("dq", "q"), ("dk", "k"), ("dv", "v"), ("dg", "g"), ("dbias", "bias")):
        if key in t:
            assert _rel(gr[name], t[key].grad.numpy()) <= 1e-13, name


# ---------------------------------------------------------------- P3: L = 1 special case
def test_p3_single_key():
    c = _case(B=2, H=2, L=1, D=5, seed=4)
    o, lse = oracle.attn_fwd(c["q"], c["k"], c["v"], bias=c["bias"], g=c["g"], scale=c["scale"])
    sg = 1.0 / (1.0 + np.exp(-c["g"]))
    np.testing.assert_array_equal(o, sg * c["v"])
    s = c["scale"] * np.einsum("bhqd,bhkd->bhqk", c["q"], c["k"])[..., 0] + c["bias"][None, ..., 0]
    np.testing.assert_allclose(lse, s, atol=1e-15)
    gr = oracle.attn_bwd(c["q"], c["k"], c["v"], c["dout"], bias=c["bias"], g=c["g"],
                         scale=c["scale"])
    assert np.all(gr["dq"] == 0) and np.all(gr["dk"] == 0) and np.all(gr["dbias"] == 0)
    np.testing.assert_allclose(gr["dv"], c["dout"] * sg, atol=1e-15)


# ---------------------------------------------------------------- P4: masked keys are inert
def test_p4_masked_keys_inert():
    c = _case(B=3, H=2, L=9, D=4, seed=5, mask="prefix")
    c["mask"][1, 3] = 0  # an interior hole too
    c["mask"][:, 7] = 0  # a key masked in EVERY batch row: its (shared) bias column is inert too
    f = oracle.attn_fwd(c["q"], c["k"], c["v"], bias=c["bias"], mask=c["mask"], g=c["g"],
                        scale=c["scale"])
    gr = oracle.attn_bwd(c["q"], c["k"], c["v"], c["dout"], bias=c["bias"], mask=c["mask"],
                         g=c["g"], scale=c["scale"])
    rng = np.random.default_rng(99)
    dropped = c["mask"] == 0
    k2, v2, b2 = c["k"].copy(), c["v"].copy(), c["bias"].copy()
    for b in range(3):
        for kk in np.nonzero(dropped[b])[0]:
            k2[b, :, kk] = rng.standard_normal(k2[b, :, kk].shape) * 100
            v2[b, :, kk] = rng.standard_normal(v2[b, :, kk].shape) * 100
    # the shared bias is read by every batch row, so only the columns of keys masked in all
    # rows can be re-randomised (reading R5: masked keys never influence any output)
    all_dropped = np.nonzero(dropped.all(axis=0))[0]
    assert all_dropped.size > 0
    b2[:, :, all_dropped] = rng.standard_normal(b2[:, :, all_dropped].shape) * 100
    f2 = oracle.attn_fwd(c["q"], k2, v2, bias=b2, mask=c["mask"], g=c["g"], scale=c["scale"])
    gr2 = oracle.attn_bwd(c["q"], k2, v2, c["dout"], bias=b2, mask=c["mask"], g=c["g"],
                          scale=c["scale"])
    np.testing.assert_array_equal(f[0], f2[0])
    np.testing.assert_array_equal(f[1], f2[1])
    for n in ("dq", "dv", "dg", "dbias"):
        np.testing.assert_array_equal(gr[n], gr2[n])
    # dk at kept keys unchanged; dK = dV = 0 at masked keys
    for b in range(3):
        for kk in np.nonzero(dropped[b])[0]:
            assert np.all(gr["dk"][b, :, kk] == 0) and np.all(gr["dv"][b, :, kk] == 0)
    np.testing.assert_array_equal(gr["dk"], gr2["dk"])
    # p = 0 at masked keys (one-hot V read-out)
    p = _probs(c["q"], c["k"], bias=c["bias"], mask=c["mask"], scale=c["scale"])
    assert np.all(p[np.broadcast_to(dropped[:, None, None, :], p.shape)] == 0)
    # a bias column at a key masked in EVERY row gets zero gradient
    c["mask"][:, 8] = 0
    gr3 = oracle.attn_bwd(c["q"], c["k"], c["v"], c["dout"], bias=c["bias"], mask=c["mask"],
                          g=c["g"], scale=c["scale"])
    assert np.all(gr3["dbias"][:, :, 8] == 0)


# ---------------------------------------------------------------- P5: module identities
def _tri_setup(N=6, cz=8, H=2, c=3, seed=6):
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((N, N, cz))
    p = M.make_params(rng, cz, cz, H, c)
    mask = (rng.random((N, N)) > 0.2).astype(np.uint8)
    mask[2, :] = 0  # a fully masked start-row i=2
    return z, p, mask


def test_p5_end_equals_start_on_transposed_pair():
    z, p, mask = _tri_setup()
    o_end, _ = M.triangle_attention_end(z, p, mask)
    o_st, _ = M.triangle_attention_start(np.transpose(z, (1, 0, 2)), p, mask.T)
    assert _rel(o_end, np.transpose(o_st, (1, 0, 2, 3))) <= 1e-14


def test_p5_core_oracle_matches_module_formulations():
    """The C core (B = batch axis, L = attended axis) against AF2 Alg. 7/8/13/14 in einsum."""
    z, p, mask = _tri_setup()
    N, H, c = z.shape[0], 2, 3
    sc = 1.0 / np.sqrt(c)
    # triangle start: B = i, queries j, keys k, bias b[h,j,k], mask[i,k]
    o_ref, pr = M.triangle_attention_start(z, p, mask)
    tr = lambda x: np.transpose(x, (0, 2, 1, 3))  # [i,j,h,c] -> [i,h,j,c]
    o, _ = oracle.attn_fwd(tr(pr["q"]), tr(pr["k"]), tr(pr["v"]), bias=pr["bias"], mask=mask,
                           g=tr(pr["g"]), scale=sc)
    assert _rel(o, tr(o_ref)) <= 1e-14
    # triangle end: B = j, queries i, keys k, bias b_ki -> [h,i,k] = b[h,k,i], mask[k,j]
    o_ref, pr = M.triangle_attention_end(z, p, mask)
    tc = lambda x: np.transpose(x, (1, 2, 0, 3))  # [i,j,h,c] -> [j,h,i,c]
    o, _ = oracle.attn_fwd(tc(pr["q"]), tc(pr["k"]), tc(pr["v"]),
                           bias=np.transpose(pr["bias"], (0, 2, 1)), mask=mask.T,
                           g=tc(pr["g"]), scale=sc)
    assert _rel(o, tc(o_ref)) <= 1e-14
    # MSA row with pair bias (Alg. 7) and column (Alg. 8)
    rng = np.random.default_rng(8)
    S, R, cm, cz = 5, 6, 8, 4
    m = rng.standard_normal((S, R, cm))
    zz = rng.standard_normal((R, R, cz))
    pm = M.make_params(rng, cm, cz, H, c)
    msa_mask = (rng.random((S, R)) > 0.2).astype(np.uint8)
    o_ref, pr = M.msa_row_attention_with_pair_bias(m, zz, pm, msa_mask)
    o, _ = oracle.attn_fwd(tr(pr["q"]), tr(pr["k"]), tr(pr["v"]), bias=pr["bias"],
                           mask=msa_mask, g=tr(pr["g"]), scale=sc)
    assert _rel(o, tr(o_ref)) <= 1e-14
    o_ref, pr = M.msa_column_attention(m, pm, msa_mask)
    o, _ = oracle.attn_fwd(tc(pr["q"]), tc(pr["k"]), tc(pr["v"]), mask=msa_mask.T,
                           g=tc(pr["g"]), scale=sc)
    assert _rel(o, tc(o_ref)) <= 1e-14


# ---------------------------------------------------------------- P6: permutation equivariance
def test_p6_permutation_equivariance():
    c = _case(B=3, H=2, L=8, D=4, seed=9, mask="prefix")
    args = dict(scale=c["scale"])
    o, lse = oracle.attn_fwd(c["q"], c["k"], c["v"], bias=c["bias"], mask=c["mask"], g=c["g"],
                             **args)
    gr = oracle.attn_bwd(c["q"], c["k"], c["v"], c["dout"], bias=c["bias"], mask=c["mask"],
                         g=c["g"], **args)
    rng = np.random.default_rng(10)
    pk = rng.permutation(8)  # keys jointly: K, V, bias columns, mask
    o2, _ = oracle.attn_fwd(c["q"], c["k"][:, :, pk], c["v"][:, :, pk], bias=c["bias"][:, :, pk],
                            mask=c["mask"][:, pk], g=c["g"], **args)
    assert _rel(o2, o) <= 1e-14
    pq = rng.permutation(8)  # queries: o permutes, dbias rows permute
    o3, _ = oracle.attn_fwd(c["q"][:, :, pq], c["k"], c["v"], bias=c["bias"][:, pq],
                            mask=c["mask"], g=c["g"][:, :, pq], **args)
    assert _rel(o3, o[:, :, pq]) <= 1e-14
    pb = rng.permutation(3)  # batch: outputs permute, shared dbias unchanged
    gr4 = oracle.attn_bwd(c["q"][pb], c["k"][pb], c["v"][pb], c["dout"][pb], bias=c["bias"],
                          mask=c["mask"][pb], g=c["g"][pb], **args)
    assert _rel(gr4["dq"], gr["dq"][pb]) <= 1e-14
    assert _rel(gr4["dbias"], gr["dbias"]) <= 1e-13


# ---------------------------------------------------------------- P7: gradient identities
def test_p7_gradient_identities():
    c = _case(B=3, H=2, L=7, D=4, seed=11, mask="prefix")
    o, _ = oracle.attn_fwd(c["q"], c["k"], c["v"], bias=c["bias"], mask=c["mask"], g=c["g"],
                           scale=c["scale"])
    gr = oracle.attn_bwd(c["q"], c["k"], c["v"], c["dout"], bias=c["bias"], mask=c["mask"],
                         g=c["g"], scale=c["scale"])
    sg = 1.0 / (1.0 + np.exp(-c["g"]))
    scale_ref = np.max(np.abs(gr["dbias"]))
    assert np.max(np.abs(gr["dbias"].sum(-1))) <= 1e-14 * max(scale_ref, 1) * 7
    assert np.max(np.abs(gr["dk"].sum(2))) <= 1e-13
    dA = c["dout"] * sg
    live = (c["mask"].sum(-1) > 0)[:, None, None, None]
    np.testing.assert_allclose(gr["dv"].sum(2), (dA * live).sum(2), atol=1e-13)
    np.testing.assert_allclose(gr["dg"], c["dout"] * o * (1 - sg), atol=1e-15)


# ---------------------------------------------------------------- P8: finite differences
@pytest.mark.parametrize("bias", ["shared", "batch"])
def test_p8_finite_differences(bias):
    c = _case(B=2, H=2, L=5, D=3, seed=12, bias=bias, mask="prefix")
    args = dict(mask=c["mask"], scale=c["scale"])
    gr = oracle.attn_bwd(c["q"], c["k"], c["v"], c["dout"], bias=c["bias"], g=c["g"], **args)

    def f(q, k, v, bias_, g):
        o, _ = oracle.attn_fwd(q, k, v, bias=bias_, g=g, **args)
        return float(np.sum(o * c["dout"]))  # <dO, o>

    h = 1e-6
    names = ["q", "k", "v", "bias", "g"]
    for i, n in enumerate(names):
        x = c[n]
        num = np.zeros_like(x)
        for idx in np.ndindex(*x.shape):
            vals = [c[m].copy() for m in names]
            vals[i][idx] += h
            fp = f(*vals)
            vals[i][idx] -= 2 * h
            fm = f(*vals)
            num[idx] = (fp - fm) / (2 * h)
        key = {"q": "dq", "k": "dk", "v": "dv", "bias": "dbias", "g": "dg"}[n]
        assert _rel(gr[key], num) <= 1e-7, (n, _rel(gr[key], num))


# ---------------------------------------------------------------- P9: broadcast dbias = Σ_b
def test_p9_shared_dbias_is_sum_over_batch():
    c = _case(B=4, H=2, L=6, D=3, seed=13, mask="prefix")
    gs = oracle.attn_bwd(c["q"], c["k"], c["v"], c["dout"], bias=c["bias"], mask=c["mask"],
                         g=c["g"], scale=c["scale"])
    bb = np.broadcast_to(c["bias"][None], (4,) + c["bias"].shape).copy()
    gb = oracle.attn_bwd(c["q"], c["k"], c["v"], c["dout"], bias=bb, mask=c["mask"], g=c["g"],
                         scale=c["scale"])
    assert _rel(gs["dbias"], gb["dbias"].sum(0)) <= 1e-14
    for n in ("dq", "dk", "dv", "dg"):
        np.testing.assert_array_equal(gs[n], gb[n])


# ---------------------------------------------------------------- P11: linearity
def test_p11_linearity():
    c = _case(B=2, H=2, L=6, D=4, seed=14)
    o, _ = oracle.attn_fwd(c["q"], c["k"], c["v"], bias=c["bias"], g=c["g"], scale=c["scale"])
    o2, _ = oracle.attn_fwd(c["q"], c["k"], 2.5 * c["v"], bias=c["bias"], g=c["g"],
                            scale=c["scale"])
    assert _rel(o2, 2.5 * o) <= 1e-15
    o3, _ = oracle.attn_fwd(4.0 * c["q"], c["k"], c["v"], bias=c["bias"], g=c["g"],
                            scale=c["scale"] / 4.0)
    assert _rel(o3, o) <= 1e-14


# ---------------------------------------------------------------- P12: batch independence
def test_p12_batch_independence():
    c = _case(B=3, H=2, L=6, D=4, seed=15)
    o, _ = oracle.attn_fwd(c["q"], c["k"], c["v"], bias=c["bias"], g=c["g"], scale=c["scale"])
    q2 = c["q"].copy()
    q2[1] += 3.0
    o2, _ = oracle.attn_fwd(q2, c["k"], c["v"], bias=c["bias"], g=c["g"], scale=c["scale"])
    np.testing.assert_array_equal(o[[0, 2]], o2[[0, 2]])
    assert not np.array_equal(o[1], o2[1])


# ---------------------------------------------------------------- P13: fully-masked rows
def test_p13_fully_masked_rows():
    c = _case(B=4, H=2, L=6, D=3, seed=16, mask="prefix")
    c["mask"][2] = 0
    o, lse = oracle.attn_fwd(c["q"], c["k"], c["v"], bias=c["bias"], mask=c["mask"], g=c["g"],
                             scale=c["scale"])
    assert np.all(o[2] == 0) and np.all(np.isneginf(lse[2]))
    assert np.all(np.isfinite(lse[[0, 1, 3]]))
    gr = oracle.attn_bwd(c["q"], c["k"], c["v"], c["dout"], bias=c["bias"], mask=c["mask"],
                         g=c["g"], scale=c["scale"])
    for n in ("dq", "dk", "dv", "dg"):
        assert np.all(gr[n][2] == 0), n
    keep = [0, 1, 3]  # deleting the padding row changes nothing else
    gr2 = oracle.attn_bwd(c["q"][keep], c["k"][keep], c["v"][keep], c["dout"][keep],
                          bias=c["bias"], mask=c["mask"][keep], g=c["g"][keep], scale=c["scale"])
    assert _rel(gr2["dbias"], gr["dbias"]) <= 1e-14
    np.testing.assert_array_equal(gr2["dq"], gr["dq"][keep])


def test_oracle_rejects_bad_bias_shape():
    c = _case(B=2, H=2, L=5, D=3, seed=17)
    with pytest.raises(ValueError):
        oracle.attn_fwd(c["q"], c["k"], c["v"], bias=np.zeros((2, 5, 4)))
