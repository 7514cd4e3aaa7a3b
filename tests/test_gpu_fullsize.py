"""Parity at the full bench sizes (BASELINE.json cfg 2/3 and the block's MSA column attention:
the four modules of one Evoformer block at N_res=256, N_seq=128), in the exact layouts, kernels
and launch configuration `bench.py` times (bench.make_module_inputs + the C ABI), against the
fp64 oracle on the same values — every output element compared, not a sample (the oracle does
one full block in seconds on the host cores)."""
import numpy as np
import pytest
import torch

import bench
import oracle
from gpu_harness import rel_err
from paper_2404_11068_b200 import evoattn

pytestmark = pytest.mark.gpu

TOL = 2e-2  # north star, bf16 I/O (R9)


def _logical(x):
    return x.float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("idx", range(len(bench.MODULES)), ids=[m[0] for m in bench.MODULES])
def test_bench_module_fullsize(idx):
    dev = torch.device("cuda:0")
    name, B, H, L, bias = bench.MODULES[idx]
    t = bench.make_module_inputs(torch, dev, name, B, H, L, bias, seed=100 + idx)
    o, lse = evoattn.fwd(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"])
    r = evoattn.bwd(t["q"], t["k"], t["v"], o, lse, t["dout"], t["bias"], t["mask"], t["g"])
    torch.cuda.synchronize()
    q, k, v, g, do = (_logical(t[n]) for n in ("q", "k", "v", "g", "dout"))
    bb = None if t["bias"] is None else _logical(t["bias"])
    m = t["mask"].cpu().numpy()
    ro, rl = oracle.attn_fwd(q, k, v, bb, m, g)
    rg = oracle.attn_bwd(q, k, v, do, bb, m, g)
    errs = {"o": rel_err(_logical(o), ro), "lse": rel_err(lse.cpu().numpy(), rl)}
    for n in ("dq", "dk", "dv", "dg", "dbias"):
        if rg[n] is not None:
            errs[n] = rel_err(_logical(r[n]), rg[n])
    bad = {k_: v_ for k_, v_ in errs.items() if not v_ <= TOL}
    assert not bad, f"{name}: {errs}"
