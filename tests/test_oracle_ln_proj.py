"""Pins for the LN + q/k/v/g projection oracle (oracle/ln_proj.py)."""
import numpy as np
import torch

from oracle.ln_proj import linear_fwd, ln_qkvg_fwd


def test_equals_torch_layer_norm_and_linear():
    r = np.random.default_rng(0)
    x, g, b = r.standard_normal((9, 16)) * 3 + 2, 1 + 0.1 * r.standard_normal(16), 0.1 * r.standard_normal(16)
    W, bg = r.standard_normal((16, 4, 12)), r.standard_normal(12)
    out = ln_qkvg_fwd(x, g, b, W, bg)
    y = torch.nn.functional.layer_norm(torch.from_numpy(x), (16,), torch.from_numpy(g), torch.from_numpy(b), eps=1e-5)
    for j in range(4):
        ref = torch.nn.functional.linear(y, torch.from_numpy(W[:, j, :].T.copy()),
                                         torch.from_numpy(bg) if j == 3 else None).numpy()
        assert np.max(np.abs(out[:, j] - ref)) < 1e-12


def test_identity_like_rows():
    """rows that normalise to unit vectors e_c·sqrt(C) (γ=1, β=0) select weight rows."""
    C = 8
    x = np.full((C, C), -1.0)
    np.fill_diagonal(x, C - 1.0)                     # mean 0 per row, LN(x_c) ∝ e_c
    W = np.random.default_rng(1).standard_normal((C, 4, 3))
    out = ln_qkvg_fwd(x, np.ones(C), np.zeros(C), W, eps=0.0)
    y = (x - x.mean(1, keepdims=True)) / x.std(1, keepdims=True)
    for j in range(4):
        assert np.allclose(out[:, j], y @ W[:, j])


def test_linear_unit_rows_and_additivity():
    """Unit input rows select weight columns (x = I -> Wᵀ + b); the map is affine."""
    r = np.random.default_rng(2)
    W, b = r.standard_normal((6, 5)), r.standard_normal(6)
    assert np.array_equal(linear_fwd(np.eye(5), W, b), W.T + b)
    x1, x2 = r.standard_normal((3, 5)), r.standard_normal((3, 5))
    lhs = linear_fwd(x1 + x2, W, b) - b
    assert np.allclose(lhs, (linear_fwd(x1, W, b) - b) + (linear_fwd(x2, W, b) - b), atol=1e-12)


# ---- backward pins (oracle/ln_proj.py::ln_proj_bwd)
from oracle.ln_proj import ln_proj_bwd  # noqa: E402


def _torch_grads(x, g, b, W, dout, ln, eps=1e-5):
    xt = torch.from_numpy(x).requires_grad_(True)
    gt = torch.from_numpy(g).requires_grad_(True)
    bt = torch.from_numpy(b).requires_grad_(True)
    Wt = torch.from_numpy(W).requires_grad_(True)
    bias = torch.zeros(W.shape[0], dtype=torch.float64, requires_grad=True)
    y = torch.nn.functional.layer_norm(xt, (x.shape[1],), gt, bt, eps=eps) if ln else xt
    out = torch.nn.functional.linear(y, Wt, bias)
    out.backward(torch.from_numpy(dout))
    r = {"dx": xt.grad.numpy(), "dW": Wt.grad.numpy(), "db": bias.grad.numpy()}
    if ln:
        r["dgamma"], r["dbeta"] = gt.grad.numpy(), bt.grad.numpy()
    return r


def test_bwd_equals_torch_autograd():
    """The backward equals fp64 torch autograd of layer_norm + linear (library routine)."""
    r = np.random.default_rng(3)
    for ln in (True, False):
        x = r.standard_normal((11, 16)) * 2 + 1
        g, b = 1 + 0.2 * r.standard_normal(16), 0.1 * r.standard_normal(16)
        W, dout = r.standard_normal((24, 16)), r.standard_normal((11, 24))
        got = ln_proj_bwd(x, g, b, W, dout, ln=ln)
        ref = _torch_grads(x, g, b, W, dout, ln)
        for k in ("dx", "dW", "db") + (("dgamma", "dbeta") if ln else ()):
            assert np.max(np.abs(got[k] - ref[k])) < 1e-10 * max(1.0, np.max(np.abs(ref[k]))), k


def test_bwd_finite_differences():
    """Central differences of <dout, out> w.r.t. x, γ, β and W on a tiny problem."""
    r = np.random.default_rng(4)
    x = r.standard_normal((3, 8))
    g, b = 1 + 0.3 * r.standard_normal(8), 0.3 * r.standard_normal(8)
    W, dout = r.standard_normal((5, 8)), r.standard_normal((3, 5))
    got = ln_proj_bwd(x, g, b, W, dout)

    def f(x_, g_, b_, W_):  # the forward oracle with W as its q block (k, v, g blocks zero)
        W4 = np.zeros((8, 4, 5))
        W4[:, 0, :] = W_.T
        return float(np.sum(dout * ln_qkvg_fwd(x_, g_, b_, W4)[:, 0, :]))

    h = 1e-6
    for name, arr, idx in (("dx", x, (1, 3)), ("dgamma", g, (2,)), ("dbeta", b, (5,)),
                           ("dW", W, (4, 6))):
        p, m = arr.copy(), arr.copy()
        p[idx] += h
        m[idx] -= h
        args = {"dx": (x, g, b, W), "dgamma": (x, g, b, W), "dbeta": (x, g, b, W),
                "dW": (x, g, b, W)}[name]
        pos = {"dx": 0, "dgamma": 1, "dbeta": 2, "dW": 3}[name]
        ap, am = list(args), list(args)
        ap[pos], am[pos] = p, m
        fd = (f(*ap) - f(*am)) / (2 * h)
        assert abs(fd - got[name][idx]) < 1e-6 * max(1.0, abs(fd)), name


def test_bwd_ln_invariants():
    """LayerNorm output is invariant to shifting a row and to scaling it, so every row of dx is
    orthogonal to the ones vector and to x̂ (closed form: Σ_c dx = 0, Σ_c dx·x̂ = 0)."""
    r = np.random.default_rng(5)
    x = r.standard_normal((7, 32)) * 4 - 2
    g, b = r.standard_normal(32), r.standard_normal(32)
    W, dout = r.standard_normal((12, 32)), r.standard_normal((7, 12))
    got = ln_proj_bwd(x, g, b, W, dout, eps=0.0)
    xh = (x - x.mean(1, keepdims=True)) / x.std(1, keepdims=True)
    assert np.max(np.abs(got["dx"].sum(1))) < 1e-10
    assert np.max(np.abs((got["dx"] * xh).sum(1))) < 1e-10
