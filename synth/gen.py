"""Seeded synthetic inputs shared by tests, smoke() and bench.py.

This module holds NO arithmetic of the method (no softmax, no attention, no gradients): it only
draws random numbers, rounds them to the bf16 grid and builds masks.  Both the CUDA path and the
oracle receive the same bytes from here (DESIGN.md §4 "input recipe"):

* q, k, v, g, bias, dO ~ N(0, 1) drawn in fp32 from ``numpy.random.Generator(PCG64(seed))``,
  then rounded to bf16 with round-to-nearest-even on the top 16 bits.
* masks: all-ones for timing; for parity a prefix-valid key mask per batch row with valid length
  ~ U[0.75·Lk, Lk] (cropped proteins / shallow MSAs), optionally with a fraction of batch rows
  fully masked (padding rows: every query of that row has no key — reading R5).
* scale = fp32(1/sqrt(D)) (reading R2).
"""
from __future__ import annotations

import numpy as np


def round_bf16(x) -> np.ndarray:
    """Round fp32 values to the nearest bf16-representable value (ties to even), returned as
    fp32.  NaN/Inf pass through."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    r = r.astype(np.uint32)
    out = r.view(np.float32).copy()
    nan = np.isnan(x)
    out[nan] = x[nan]
    return out


def bf16_bits(x) -> np.ndarray:
    """bf16 bit patterns (uint16) of values already on the bf16 grid."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    return (x.view(np.uint32) >> 16).astype(np.uint16)


def default_scale(D: int) -> float:
    return float(np.float32(1.0 / np.sqrt(D)))


def prefix_mask(rng, B: int, Lk: int, lo_frac: float = 0.75, fully_masked_frac: float = 0.0):
    """[B, Lk] uint8: row b keeps keys [0, n_b) with n_b ~ U[ceil(lo_frac*Lk), Lk]; a
    ``fully_masked_frac`` share of rows (at least one if > 0) keep nothing."""
    lo = max(1, int(np.ceil(lo_frac * Lk)))
    n = rng.integers(lo, Lk + 1, size=B)
    mask = (np.arange(Lk)[None, :] < n[:, None]).astype(np.uint8)
    if fully_masked_frac > 0 and B > 0:
        nfm = max(1, int(round(fully_masked_frac * B)))
        rows = rng.choice(B, size=min(nfm, B), replace=False)
        mask[rows] = 0
    return mask


def attention_case(B, H, Lq, Lk, D, seed=0, bias="shared", gate=True, mask="none",
                   fully_masked_frac=0.1, bf16=True):
    """One seeded attention problem in logical layouts (fp32 values, on the bf16 grid if
    ``bf16``): q,g,dout [B,H,Lq,D]; k,v [B,H,Lk,D]; bias [H,Lq,Lk] (shared), [B,H,Lq,Lk]
    (batch) or None; mask [B,Lk] uint8 or None."""
    rng = np.random.default_rng(seed)
    rnd = (lambda *s: round_bf16(rng.standard_normal(s, dtype=np.float32))) if bf16 else \
        (lambda *s: rng.standard_normal(s, dtype=np.float32))
    case = {
        "q": rnd(B, H, Lq, D), "k": rnd(B, H, Lk, D), "v": rnd(B, H, Lk, D),
        "g": rnd(B, H, Lq, D) if gate else None,
        "dout": rnd(B, H, Lq, D),
        "bias": None, "mask": None, "scale": default_scale(D),
    }
    if bias == "shared":
        case["bias"] = rnd(H, Lq, Lk)
    elif bias == "batch":
        case["bias"] = rnd(B, H, Lq, Lk)
    elif bias is not None:
        raise ValueError(bias)
    if mask == "prefix":
        case["mask"] = prefix_mask(rng, B, Lk)
    elif mask == "prefix_fm":
        case["mask"] = prefix_mask(rng, B, Lk, fully_masked_frac=fully_masked_frac)
    elif mask == "ones":
        case["mask"] = np.ones((B, Lk), np.uint8)
    elif mask != "none":
        raise ValueError(mask)
    return case


# BASELINE.json configs as concrete core calls.
CONFIGS = {
    # cfg 1: triangle start, N_res=32, c_z=32, 2 heads x 16 (oracle in seconds)
    "cfg1_tri_start": dict(B=32, H=2, L=32, D=16, bias="shared"),
    # cfg 2: MSA row attention with pair bias, N_seq=128, N_res=256, 8 x 32
    "cfg2_msa_row": dict(B=128, H=8, L=256, D=32, bias="shared"),
    # cfg 3: triangle start (and end, transposed view), N_res=256, 4 x 32
    "cfg3_tri": dict(B=256, H=4, L=256, D=32, bias="shared"),
    # MSA column attention inside the N_res=256 block: B=N_res, L=N_seq, no bias
    "msa_col": dict(B=256, H=8, L=128, D=32, bias=None),
    # cfg 4: extra-MSA column attention (global-free), N_extra=1024, 8 x 8
    "cfg4_extra_col": dict(B=256, H=8, L=1024, D=8, bias=None),
}
