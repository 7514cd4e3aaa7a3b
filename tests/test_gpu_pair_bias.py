"""Pair-bias side path (LN + LinearNoBias) on the GPU through the C ABI
(include/evo_pair_bias.h) against the fp64 oracle (oracle/pair_bias.py) on the same bf16
inputs; normwise max relative error (R9) within 2e-2 for the bf16 outputs (bias, dz)
and fp32 statistics / parameter gradients within 1e-3."""
import numpy as np
import pytest
import torch

from gpu_harness import rel_err
from oracle.pair_bias import pair_bias_bwd, pair_bias_fwd
from paper_2404_11068_b200 import evoattn

pytestmark = pytest.mark.gpu


def _inputs(Li, Lj, C, H, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    z = (torch.randn((Li, Lj, C), generator=g) * 2 + 0.5).to(torch.bfloat16)
    gamma = 1 + 0.1 * torch.randn(C, generator=g)
    beta = 0.1 * torch.randn(C, generator=g)
    W = torch.randn((C, H), generator=g) / C ** 0.5
    dbias = torch.randn((H, Li, Lj), generator=g)
    return z, gamma, beta, W, dbias


@pytest.mark.parametrize("Li,Lj,C,H,orient", [(32, 32, 32, 4, "hij"), (64, 48, 128, 4, "hij"),
                                              (40, 40, 128, 8, "jhi"), (16, 30, 256, 16, "ihj"),
                                              (256, 256, 128, 4, "hij"), (20, 24, 64, 8, "hij")])
def test_pair_bias_parity(Li, Lj, C, H, orient):
    z, gamma, beta, W, dbias = _inputs(Li, Lj, C, H, seed=Li + C)
    dev = torch.device("cuda:0")
    zd = z.to(dev)
    # output orientation: head-major [H,Li,Lj], the transposed end-node storage, or DAP [Li,H,Lj]
    perm = {"hij": (0, 1, 2), "jhi": (1, 2, 0), "ihj": (1, 0, 2)}[orient]
    inv = np.argsort(perm)
    store = torch.empty(tuple(np.array((H, Li, Lj))[list(perm)]), dtype=torch.bfloat16, device=dev)
    bview = store.permute(*inv)
    bias, mean, rstd = evoattn.pair_bias_fwd(zd, gamma.to(dev), beta.to(dev), W.to(dev),
                                             bias=bview)
    db_store = dbias.permute(*perm).contiguous().to(dev)
    r = evoattn.pair_bias_bwd(zd, gamma.to(dev), beta.to(dev), W.to(dev), mean, rstd,
                              db_store.permute(*inv))
    torch.cuda.synchronize()
    zf = z.double().numpy()
    rb, rm, rr = pair_bias_fwd(zf, gamma.double().numpy(), beta.double().numpy(), W.double().numpy())
    assert rel_err(bias.float().cpu().numpy(), rb) < 2e-2
    assert rel_err(mean.cpu().numpy(), rm) < 1e-3 and rel_err(rstd.cpu().numpy(), rr) < 1e-3
    g = pair_bias_bwd(zf, gamma.double().numpy(), beta.double().numpy(), W.double().numpy(),
                      dbias.double().numpy())
    assert rel_err(r["dz"].float().cpu().numpy(), g["dz"]) < 2e-2
    for n in ("dgamma", "dbeta", "dW"):
        assert rel_err(r[n].cpu().numpy(), g[n]) < 1e-3, n
