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
