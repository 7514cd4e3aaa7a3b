"""Fused LayerNorm + batched q/k/v/g projection (include/evo_ln_proj.h) on
the GPU through the C ABI against the fp64 oracle (oracle/ln_proj.py) on the same bf16 inputs:
normwise max relative error (R9) within 2e-2 for the bf16 projections, 1e-4 for the
fp32 row statistics (checked against their plain definition)."""
import numpy as np
import pytest
import torch

from gpu_harness import rel_err
from oracle.ln_proj import linear_fwd, ln_qkvg_fwd
from paper_2404_11068_b200 import evoattn

pytestmark = pytest.mark.gpu


def _inputs(rows, C, N1, seed, x_pad=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = (torch.randn((rows, C + x_pad), generator=g) * 2 + 0.5).to(torch.bfloat16)
    gamma = 1 + 0.1 * torch.randn(C, generator=g)
    beta = 0.1 * torch.randn(C, generator=g)
    W = (torch.randn((4 * N1, C), generator=g) / C ** 0.5).to(torch.bfloat16)  # [q;k;v;g] x C
    b = torch.zeros(4 * N1)
    b[3 * N1:] = 1 + 0.1 * torch.randn(N1, generator=g)                        # gate bias only
    return x, gamma, beta, W, b


def _oracle(x, gamma, beta, W, b, C, N1, rows_idx=None):
    xs = x[:, :C].double().numpy()
    if rows_idx is not None:
        xs = xs[rows_idx]
    Wo = W.double().numpy().reshape(4, N1, C).transpose(2, 0, 1)             # [C, 4, N1]
    return ln_qkvg_fwd(xs, gamma.double().numpy(), beta.double().numpy(), Wo,
                       b[3 * N1:].double().numpy()).reshape(len(xs), 4 * N1)


@pytest.mark.parametrize("rows,C,N1,x_pad,out_pad", [
    (300, 128, 128, 0, 0),     # triangle attention: c_z 128, 4 heads x 32 (N = 512), ragged tail
    (1000, 256, 256, 0, 0),    # MSA row / column: c_m 256, 8 heads x 32 (N = 1024)
    (77, 64, 64, 0, 0),        # extra MSA: c_e 64, 8 heads x 8 (N = 256), one partial tile
    (130, 64, 32, 8, 16),      # N = 128 (n-tile 128), strided x and out
    (257, 128, 48, 0, 64),     # N = 192 (n-tile 64)
    (128, 256, 256, 64, 0),    # exactly one tile, strided x
])
def test_ln_proj_parity(rows, C, N1, x_pad, out_pad):
    x, gamma, beta, W, b = _inputs(rows, C, N1, seed=rows + C, x_pad=x_pad)
    dev = torch.device("cuda:0")
    xd = x.to(dev)[:, :C]
    out = torch.full((rows, 4 * N1 + out_pad), 7.0, dtype=torch.bfloat16, device=dev)
    y, mean, rstd = evoattn.ln_proj_fwd(xd, gamma.to(dev), beta.to(dev), W.to(dev), b.to(dev),
                                        out=out[:, :4 * N1])
    torch.cuda.synchronize()
    ref = _oracle(x, gamma, beta, W, b, C, N1)
    assert rel_err(y.float().cpu().numpy(), ref) < 2e-2
    for j in range(4):  # each projection on its own (q, k, v, g blocks of the stacked output)
        blk = slice(j * N1, (j + 1) * N1)
        assert rel_err(y[:, blk].float().cpu().numpy(), ref[:, blk]) < 2e-2, j
    if out_pad:
        assert bool((out[:, 4 * N1:] == 7.0).all())  # padding columns untouched
    xs = x[:, :C].double().numpy()
    assert rel_err(mean.cpu().numpy(), xs.mean(1)) < 1e-4
    assert rel_err(rstd.cpu().numpy(), 1 / np.sqrt(xs.var(1) + 1e-5)) < 1e-4


def test_ln_proj_no_bias_and_empty():
    x, gamma, beta, W, _ = _inputs(200, 128, 64, seed=3)
    dev = torch.device("cuda:0")
    y, _, _ = evoattn.ln_proj_fwd(x.to(dev), gamma.to(dev), beta.to(dev), W.to(dev), None)
    ref = _oracle(x, gamma, beta, W, torch.zeros(256), 128, 64)
    assert rel_err(y.float().cpu().numpy(), ref) < 2e-2
    e, _, _ = evoattn.ln_proj_fwd(x[:0].to(dev), gamma.to(dev), beta.to(dev), W.to(dev), None)
    assert e.shape == (0, 256)


def test_ln_proj_full_size_sampled():
    """BASELINE.json configs[1] MSA row module input: 128 x 256 rows of c_m = 256 -> q|k|v|g
    (8 heads x 32); every output row is checked on a sample of 512 rows (one per tile and more)."""
    rows, C, N1 = 128 * 256, 256, 256
    x, gamma, beta, W, b = _inputs(rows, C, N1, seed=11)
    dev = torch.device("cuda:0")
    y, _, _ = evoattn.ln_proj_fwd(x.to(dev), gamma.to(dev), beta.to(dev), W.to(dev), b.to(dev))
    torch.cuda.synchronize()
    idx = np.unique(np.concatenate([np.arange(0, rows, 128) + np.arange(rows // 128) % 128,
                                    np.random.default_rng(0).integers(0, rows, 256)]))
    ref = _oracle(x, gamma, beta, W, b, C, N1, rows_idx=idx)
    assert rel_err(y.float().cpu().numpy()[idx], ref) < 2e-2


@pytest.mark.parametrize("rows,C,N", [(300, 256, 256), (1000, 128, 128), (77, 64, 192)])
def test_linear_parity(rows, C, N):
    """Output projection (evo_linear_fwd): the gated attention output [rows, H·D] times W_oᵀ."""
    g = torch.Generator(device="cpu").manual_seed(rows + N)
    x = torch.randn((rows, C), generator=g).to(torch.bfloat16)
    W = (torch.randn((N, C), generator=g) / C ** 0.5).to(torch.bfloat16)
    b = torch.randn(N, generator=g)
    dev = torch.device("cuda:0")
    y = evoattn.linear_fwd(x.to(dev), W.to(dev), b.to(dev))
    ref = linear_fwd(x.double().numpy(), W.double().numpy(), b.double().numpy())
    assert rel_err(y.float().cpu().numpy(), ref) < 2e-2
    y0 = evoattn.linear_fwd(x.to(dev), W.to(dev), None)
    assert rel_err(y0.float().cpu().numpy(), ref - b.double().numpy()) < 2e-2
