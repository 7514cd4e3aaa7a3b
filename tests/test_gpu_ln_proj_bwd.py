"""GPU parity of the f2 backward (evo_ln_proj_bwd / evo_linear_bwd, tcgen05 dgrad + wgrad)
against the fp64 oracle (oracle/ln_proj.py::ln_proj_bwd) at the AF2 module shapes, ragged row
counts and strided dout; normwise max relative error <= 2e-2 (bf16 I/O, R9); bitwise
repeatability of every output."""
import numpy as np
import pytest
import torch

from oracle.ln_proj import ln_proj_bwd as oracle_bwd
from paper_2404_11068_b200 import evoattn

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _rel(x, ref):
    x = x.double().cpu().numpy() if isinstance(x, torch.Tensor) else x
    return float(np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-30))


def _case(rows, C, N, seed, ld_pad=0):
    g = torch.Generator().manual_seed(seed)
    x = (torch.randn(rows, C, generator=g) * 2 + 0.5).to(torch.bfloat16)
    gamma = 1 + 0.2 * torch.randn(C, generator=g)
    beta = 0.2 * torch.randn(C, generator=g)
    W = (torch.randn(N, C, generator=g) / C ** 0.5).to(torch.bfloat16)
    dout_full = torch.randn(rows, N + ld_pad, generator=g).to(torch.bfloat16)
    return x, gamma, beta, W, dout_full


@pytest.mark.parametrize("rows,C,N,ld_pad", [(300, 64, 256, 0), (1000, 128, 512, 64),
                                             (257, 256, 1024, 0), (128, 256, 128, 0)])
def test_ln_proj_bwd_parity(rows, C, N, ld_pad):
    dev = torch.device("cuda:0")
    x, gamma, beta, W, dout_full = _case(rows, C, N, seed=rows + C)
    xd, gd, bd, Wd = x.to(dev), gamma.to(dev), beta.to(dev), W.to(dev)
    doutd = dout_full.to(dev)[:, :N]
    _, mean, rstd = evoattn.ln_proj_fwd(xd, gd, bd, Wd)
    r = evoattn.ln_proj_bwd(xd, gd, bd, Wd, mean, rstd, doutd)
    r2 = evoattn.ln_proj_bwd(xd, gd, bd, Wd, mean, rstd, doutd)
    torch.cuda.synchronize()
    ref = oracle_bwd(x.double().numpy(), gamma.double().numpy(), beta.double().numpy(),
                     W.double().numpy(), dout_full[:, :N].double().numpy())
    errs = {k: _rel(r[k], ref[k]) for k in ("dx", "dgamma", "dbeta", "dW", "db")}
    assert all(v <= TOL for v in errs.values()), errs
    for k in ("dx", "dgamma", "dbeta", "dW", "db"):
        assert torch.equal(r[k], r2[k]), k


@pytest.mark.parametrize("rows,C,N", [(200, 128, 256), (64, 256, 512)])
def test_linear_bwd_parity(rows, C, N):
    dev = torch.device("cuda:0")
    x, _, _, W, dout = _case(rows, C, N, seed=7)
    r = evoattn.linear_bwd(x.to(dev), W.to(dev), dout.to(dev))
    torch.cuda.synchronize()
    ref = oracle_bwd(x.double().numpy(), None, None, W.double().numpy(), dout.double().numpy(),
                     ln=False)
    errs = {k: _rel(r[k], ref[k]) for k in ("dx", "dW", "db")}
    assert all(v <= TOL for v in errs.values()), errs


def test_ln_proj_bwd_msa_fullsize_sampled():
    """The MSA row/column input at full size (N_seq·N_res = 32768 rows, c_m = 256 -> 4·H·D =
    1024): dW, dγ, dβ, db in full; dx on 256 sampled rows."""
    dev = torch.device("cuda:0")
    rows, C, N = 32768, 256, 1024
    x, gamma, beta, W, dout = _case(rows, C, N, seed=11)
    xd, gd, bd, Wd, dd = x.to(dev), gamma.to(dev), beta.to(dev), W.to(dev), dout.to(dev)
    _, mean, rstd = evoattn.ln_proj_fwd(xd, gd, bd, Wd)
    r = evoattn.ln_proj_bwd(xd, gd, bd, Wd, mean, rstd, dd)
    torch.cuda.synchronize()
    ref = oracle_bwd(x.double().numpy(), gamma.double().numpy(), beta.double().numpy(),
                     W.double().numpy(), dout.double().numpy())
    errs = {k: _rel(r[k], ref[k]) for k in ("dgamma", "dbeta", "dW", "db")}
    idx = np.random.default_rng(0).choice(rows, 256, replace=False)
    errs["dx"] = _rel(r["dx"][torch.from_numpy(idx).to(dev)], ref["dx"][idx])
    assert all(v <= TOL for v in errs.values()), errs
