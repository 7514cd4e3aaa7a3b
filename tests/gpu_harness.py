"""Shared GPU-test harness: lay one seeded problem out on the device in a chosen storage layout,
run the CUDA path through the C ABI, run the oracle on the same values, and report the
normwise max relative error per output (reading R9:
err(t) = max_i |t_gpu,i - t_ref,i| / max_i |t_ref,i|)."""
from __future__ import annotations

import numpy as np
import torch

import oracle
from paper_2404_11068_b200 import evoattn
from synth.gen import attention_case


def rel_err(x, ref):
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    if ref.size == 0:
        return 0.0
    return float(np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-30))


def to_dev_x(a, dtype, layout, dev):
    """logical [B,H,L,D] numpy -> device view with the requested storage layout."""
    if layout == "bhld":
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype)
    if layout == "blhd":  # projection layout [B, L, H, D]
        return torch.from_numpy(np.ascontiguousarray(a.transpose(0, 2, 1, 3))).to(dev, dtype) \
            .permute(0, 2, 1, 3)
    if layout == "lbhd":  # column / end-node view: batch axis is the middle storage axis
        return torch.from_numpy(np.ascontiguousarray(a.transpose(2, 0, 1, 3))).to(dev, dtype) \
            .permute(1, 2, 0, 3)
    raise ValueError(layout)


def to_dev_bias(b, dtype, transposed, dev):
    """bias [H,Lq,Lk] (or [B,H,Lq,Lk]) -> device view; transposed = q-unit-stride storage."""
    t = torch.from_numpy(np.ascontiguousarray(b))
    if transposed:
        t = t.transpose(-1, -2).contiguous().to(dev, dtype).transpose(-1, -2)
    else:
        t = t.to(dev, dtype)
    return evoattn.pad_bias(t)


def to_dev_mask(m, transposed, dev):
    t = torch.from_numpy(np.ascontiguousarray(m))
    if transposed:
        return t.t().contiguous().to(dev).t()
    return t.to(dev)


def run_case(B, H, Lq, Lk, D, seed=0, bias="shared", bias_t=False, gate=True, mask="prefix",
             mask_t=False, layout="blhd", dtype=torch.bfloat16, bwd=True, case=None):
    dev = torch.device("cuda:0")
    c = case or attention_case(B, H, Lq, Lk, D, seed=seed, bias=bias, gate=gate, mask=mask,
                               bf16=(dtype == torch.bfloat16))
    t = {n: to_dev_x(c[n], dtype, layout, dev) for n in ("q", "k", "v", "dout")}
    g = to_dev_x(c["g"], dtype, layout, dev) if c["g"] is not None else None
    bt = to_dev_bias(c["bias"], dtype, bias_t, dev) if c["bias"] is not None else None
    mt = to_dev_mask(c["mask"], mask_t, dev) if c["mask"] is not None else None
    o, lse = evoattn.fwd(t["q"], t["k"], t["v"], bt, mt, g, c["scale"])
    out = {"o": o, "lse": lse}
    if bwd:
        out.update(evoattn.bwd(t["q"], t["k"], t["v"], o, lse, t["dout"], bt, mt, g, c["scale"]))
    torch.cuda.synchronize()
    ro, rl = oracle.attn_fwd(c["q"], c["k"], c["v"], c["bias"], c["mask"], c["g"], c["scale"])
    errs = {"o": rel_err(o.float().cpu().numpy(), ro)}
    lg = lse.cpu().numpy().astype(np.float64)
    fin = np.isfinite(rl)
    assert np.array_equal(np.isfinite(lg), fin), "lse -inf pattern differs"
    errs["lse"] = rel_err(lg[fin], rl[fin]) if fin.any() else 0.0
    if bwd:
        rg = oracle.attn_bwd(c["q"], c["k"], c["v"], c["dout"], c["bias"], c["mask"], c["g"],
                             c["scale"])
        # reading R9b: a reference gradient that is identically zero (e.g. dq, dk, dbias at
        # L = 1) is judged against the largest reference gradient magnitude of the same call
        gscale = max(float(np.max(np.abs(rg[n]))) for n in ("dq", "dk", "dv", "dg", "dbias")
                     if rg[n] is not None and rg[n].size)
        for n in ("dq", "dk", "dv", "dg", "dbias"):
            if rg[n] is not None:
                x = out[n].float().cpu().numpy()
                if rg[n].size and np.max(np.abs(rg[n])) == 0:
                    errs[n] = float(np.max(np.abs(x))) / max(gscale, 1e-30)
                else:
                    errs[n] = rel_err(x, rg[n])
    return errs, out, c
