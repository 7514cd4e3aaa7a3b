"""Out-of-bounds write detection without compute-sanitizer (closed on this GPU pool): every
output of the forward and backward is a strided VIEW inside a larger storage — gaps along l
(extra rows), h (an extra head slot) and k (dbias row padding) — with guard bands before and
after, all pre-filled with a sentinel bit pattern.  After the call every byte outside the views
must still hold the sentinel and every element inside must have been written (no sentinel
left), for ragged shapes that hit each kernel variant (fwd_occ with no / k-contiguous /
q-contiguous bias; the pair-bias backward at nk = 1 and with the 2-CTA dQ pair sum at D = 16
and 32; the no-bias backward at nk = 1, with fp32 parts, and with the in-CTA key-tile loop; the
two-pass backward; the fp32 verification path) and for the workspace (its tail guard)."""
import ctypes

import numpy as np
import pytest
import torch

from gpu_harness import to_dev_mask
from paper_2404_11068_b200 import evoattn
from synth.gen import attention_case

pytestmark = pytest.mark.gpu

GUARD = 4096
BF16_SENT = -32191  # 0x823F as int16: a bf16 denormal no kernel output is exactly equal to
F32_SENT = 0x7F8ABCDE  # a signalling-NaN bit pattern


def _sentinel_storage(n, dtype, dev):
    if dtype == torch.float32:
        s = torch.full((n + 2 * GUARD,), F32_SENT, dtype=torch.int32, device=dev)
        return s.view(torch.float32)
    s = torch.full((n + 2 * GUARD,), BF16_SENT, dtype=torch.int16, device=dev)
    return s.view(dtype)


def _x_view(storage, B, H, L, D, Lp, Hp, layout):
    """[B,H,L,D] view into storage[GUARD:] laid out as [B,Lp,Hp,D] (row) or [Lp,B,Hp,D]."""
    if layout == "blhd":
        base = storage[GUARD:GUARD + B * Lp * Hp * D].view(B, Lp, Hp, D)
        return base[:, :L, :H, :].permute(0, 2, 1, 3)
    base = storage[GUARD:GUARD + Lp * B * Hp * D].view(Lp, B, Hp, D)
    return base[:L, :, :H, :].permute(1, 2, 0, 3)


def _sent_mask(storage):
    if storage.dtype == torch.float32:
        return storage.view(torch.int32) == F32_SENT
    return storage.view(torch.int16) == BF16_SENT


def _check_storage(storage, view, name):
    """every element outside `view` still holds the sentinel, none inside does."""
    sent = _sent_mask(storage)
    inside = torch.zeros_like(sent)
    idx = torch.arange(storage.numel(), device=storage.device)
    # mark the view's elements through a same-strided view onto the index tensor
    iv = torch.as_strided(idx, view.shape, view.stride(), view.storage_offset())
    inside[iv.reshape(-1)] = True
    outside_bad = int((~sent & ~inside).sum())
    inside_bad = int((sent & inside).sum())
    assert outside_bad == 0, f"{name}: {outside_bad} elements written outside the output view"
    assert inside_bad == 0, f"{name}: {inside_bad} output elements never written"


CASES = [  # B, H, L, D, bias, bias_t, layout, dtype
    (3, 2, 200, 32, "shared", False, "blhd", torch.bfloat16),   # nk=2 reduce-add, k-contig bias
    (3, 2, 256, 32, "shared", True, "lbhd", torch.bfloat16),    # q-contiguous (end-node) bias
    (5, 2, 130, 32, None, False, "lbhd", torch.bfloat16),       # column layout, no bias
    (2, 2, 400, 16, None, False, "blhd", torch.bfloat16),       # nk=4 ordered parts, D=16
    (2, 1, 300, 32, "shared", False, "blhd", torch.bfloat16),   # two-pass (L > 256 with bias)
    (2, 1, 140, 64, "shared", False, "blhd", torch.bfloat16),   # two-pass (D = 64)
    (2, 2, 96, 32, "batch", False, "blhd", torch.bfloat16),     # per-batch bias
    (3, 2, 100, 32, "shared", False, "blhd", torch.float32),    # fp32 verification mode
    (4, 2, 1, 32, "shared", False, "blhd", torch.bfloat16),     # L = 1
    (3, 2, 250, 16, "shared", False, "blhd", torch.bfloat16),   # 2-CTA dQ pair sum at D = 16
    (40, 4, 300, 32, None, False, "lbhd", torch.bfloat16),      # no-bias key-tile loop (B·H >= SMs)
]


@pytest.mark.parametrize("case", CASES, ids=[str(c[:7]) for c in CASES])
def test_no_out_of_bounds_writes(case):
    B, H, L, D, bias, bt, layout, dt = case
    dev = torch.device("cuda:0")
    c = attention_case(B, H, L, L, D, seed=3, bias=bias, gate=True, mask="prefix_fm",
                       bf16=dt == torch.bfloat16)
    Lp, Hp = L + 5, H + 1
    n = B * Lp * Hp * D
    ins, outs = {}, {}
    for nm in ("q", "k", "v", "g", "dout"):
        st = _sentinel_storage(n, dt, dev)
        v = _x_view(st, B, H, L, D, Lp, Hp, layout)
        lay = np.ascontiguousarray(c[nm])
        v.copy_(torch.from_numpy(lay).to(dev, dt))
        ins[nm] = v
    for nm in ("o", "dq", "dk", "dv", "dg"):
        st = _sentinel_storage(n, dt, dev)
        outs[nm] = (st, _x_view(st, B, H, L, D, Lp, Hp, layout))
    bview = None
    if bias is not None:
        shp = c["bias"].shape
        Lkp = (L + 8 + 7) // 8 * 8  # padded k extent (16-byte-multiple strides for bf16 and fp32)
        lead = int(np.prod(shp[:-2]))
        bst = _sentinel_storage(lead * L * Lkp, dt, dev)
        full = bst[GUARD:GUARD + lead * L * Lkp].view(*shp[:-2], L, Lkp)
        bview = full[..., :L]
        if bt:  # q-contiguous: the view's last two axes are the storage's swapped ones
            full = bst[GUARD:GUARD + lead * L * Lkp].view(*shp[:-2], Lkp, L)
            bview = full[..., :L, :].transpose(-1, -2)
        bview.copy_(torch.from_numpy(c["bias"]).to(dev, dt))
        dst = _sentinel_storage(lead * L * Lkp, torch.float32, dev)
        dfull = dst[GUARD:GUARD + lead * L * Lkp].view(full.shape)
        dview = dfull[..., :L] if not bt else dfull[..., :L, :].transpose(-1, -2)
        assert dview.stride() == bview.stride()
        outs["dbias"] = (dst, dview)
    mask = to_dev_mask(c["mask"], layout == "lbhd", dev)
    lst = _sentinel_storage(B * H * L, torch.float32, dev)
    lse = lst[GUARD:GUARD + B * H * L].view(B, H, L)

    lib = evoattn.load()
    d = evoattn.make_desc(ins["q"], ins["k"], ins["v"], bview, mask, ins["g"], outs["o"][1],
                          c["scale"])
    P = evoattn._ptr
    evoattn._check(lib.evo_attn_fwd(ctypes.byref(d), P(ins["q"]), P(ins["k"]), P(ins["v"]),
                                    P(bview), P(mask), P(ins["g"]), P(outs["o"][1]), P(lse),
                                    evoattn._stream(None)))
    # dO takes o's strides (evo_attn.h); the input storage already has them
    ws_need = int(lib.evo_attn_bwd_workspace_bytes(ctypes.byref(d)))
    ws = torch.full((ws_need + 2 * GUARD,), 0x5A, dtype=torch.uint8, device=dev)
    wsv = ws[GUARD:GUARD + ws_need]
    evoattn._check(lib.evo_attn_bwd(
        ctypes.byref(d), P(ins["q"]), P(ins["k"]), P(ins["v"]), P(bview), P(mask), P(ins["g"]),
        P(outs["o"][1]), P(lse), P(ins["dout"]), P(outs["dq"][1]), P(outs["dk"][1]),
        P(outs["dv"][1]), P(outs["dg"][1]), P(outs["dbias"][1]) if bias else P(None),
        P(wsv) if ws_need else P(None), ws_need, evoattn._stream(None)))
    torch.cuda.synchronize()
    for nm, (st, v) in outs.items():
        _check_storage(st, v, nm)
    # lse: [B,H,L] contiguous between guards (rows with no kept key hold -inf, not the sentinel)
    _check_storage(lst, lse, "lse")
    assert torch.all(ws[:GUARD] == 0x5A) and torch.all(ws[GUARD + ws_need:] == 0x5A), \
        "workspace written outside [0, ws_bytes)"
    # inputs are never written (evo_attn.h)
    for nm, v in ins.items():
        assert torch.equal(v.float().cpu(), torch.from_numpy(np.ascontiguousarray(c[nm])).to(dt).float()), nm
