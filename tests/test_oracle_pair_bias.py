"""Pins for the pair-bias oracle (oracle/pair_bias.py) against library routines, closed forms
and finite differences (SPEC.md L137-153 examples)."""
import numpy as np
import pytest
import torch

from oracle.pair_bias import pair_bias_bwd, pair_bias_fwd


def _case(Li=5, Lj=6, C=16, H=3, seed=0):
    r = np.random.default_rng(seed)
    return (r.standard_normal((Li, Lj, C)), 1 + 0.1 * r.standard_normal(C),
            0.1 * r.standard_normal(C), r.standard_normal((C, H)) / np.sqrt(C),
            r.standard_normal((H, Li, Lj)))


def test_fwd_equals_torch_layer_norm_and_linear():
    z, g, b, W, _ = _case()
    bias, mean, rstd = pair_bias_fwd(z, g, b, W)
    t = torch.nn.functional.layer_norm(torch.from_numpy(z), (z.shape[-1],), torch.from_numpy(g),
                                       torch.from_numpy(b), eps=1e-5)
    ref = torch.einsum("ijc,ch->hij", t, torch.from_numpy(W)).numpy()
    assert np.max(np.abs(bias - ref)) < 1e-12
    assert np.allclose(mean, z.mean(-1)) and np.allclose(rstd, 1 / np.sqrt(z.var(-1) + 1e-5))


def test_bwd_equals_torch_autograd():
    z, g, b, W, dbias = _case(seed=1)
    tz, tg, tb, tW = (torch.from_numpy(x).requires_grad_() for x in (z, g, b, W))
    y = torch.nn.functional.layer_norm(tz, (z.shape[-1],), tg, tb, eps=1e-5)
    out = torch.einsum("ijc,ch->hij", y, tW)
    (out * torch.from_numpy(dbias)).sum().backward()
    r = pair_bias_bwd(z, g, b, W, dbias)
    for name, t in (("dz", tz), ("dgamma", tg), ("dbeta", tb), ("dW", tW)):
        assert np.max(np.abs(r[name] - t.grad.numpy())) < 1e-12, name


def test_constant_row_gives_beta_projection():
    """SPEC.md L143 example: a constant row normalises to 0, so y = β and bias = βᵀW."""
    z, g, b, W, _ = _case(Li=2, Lj=3)
    z[1, 2, :] = 3.25
    bias, _, _ = pair_bias_fwd(z, g, b, W)
    assert np.allclose(bias[:, 1, 2], b @ W, atol=1e-12)


def test_finite_differences():
    z, g, b, W, dbias = _case(Li=2, Lj=3, C=8, H=2, seed=2)
    r = pair_bias_bwd(z, g, b, W, dbias)
    loss = lambda z_, g_, b_, W_: float((pair_bias_fwd(z_, g_, b_, W_)[0] * dbias).sum())
    h = 1e-6
    for name, arr, pos in (("dz", z, 0), ("dgamma", g, 1), ("dbeta", b, 2), ("dW", W, 3)):
        num = np.zeros_like(arr)
        it = np.nditer(arr, flags=["multi_index"])
        for _ in it:
            k = it.multi_index
            args_p = [z.copy(), g.copy(), b.copy(), W.copy()]
            args_m = [z.copy(), g.copy(), b.copy(), W.copy()]
            args_p[pos][k] += h
            args_m[pos][k] -= h
            num[k] = (loss(*args_p) - loss(*args_m)) / (2 * h)
        err = np.max(np.abs(num - r[name])) / max(np.max(np.abs(r[name])), 1e-30)
        assert err < 1e-6, (name, err)


def test_zero_upstream_gives_zero_gradients():
    z, g, b, W, dbias = _case()
    r = pair_bias_bwd(z, g, b, W, np.zeros_like(dbias))
    assert all(np.all(r[k] == 0) for k in r)
