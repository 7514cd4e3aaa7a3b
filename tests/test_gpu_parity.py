"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded
inputs.  bf16 I/O: every output within normwise max relative error 2e-2; fp32 verification mode:
1e-5 (north star; reading R9).  Shapes span several 128-tiles and ragged tails."""
import numpy as np
import pytest
import torch

from gpu_harness import rel_err, run_case
from synth.gen import attention_case

pytestmark = pytest.mark.gpu

TOL = {torch.bfloat16: 2e-2, torch.float32: 1e-5}


def _assert(errs, dtype, ctx=""):
    bad = {k: v for k, v in errs.items() if not v <= TOL[dtype]}
    assert not bad, f"{ctx} errors over {TOL[dtype]}: {bad} (all: {errs})"


# (B, H, L, D, bias, bias_t, gate, mask, mask_t, layout)
CASES = [
    (2, 2, 128, 32, "shared", False, True, "prefix", False, "blhd"),     # one tile
    (3, 2, 256, 32, "shared", False, True, "prefix_fm", False, "blhd"),  # 2x2 tiles, padded rows
    (2, 3, 100, 32, "shared", False, True, "prefix", False, "bhld"),     # ragged single tile
    (2, 2, 200, 16, "shared", False, False, "none", False, "blhd"),      # ragged 2 tiles, D=16
    (2, 2, 129, 8, None, False, True, "prefix", True, "lbhd"),           # col-attn view, D=8
    (2, 2, 300, 64, "shared", False, True, "prefix", False, "blhd"),     # D=64, 3 tiles
    (2, 2, 256, 32, "shared", True, True, "prefix", True, "lbhd"),       # end-node view
    (2, 2, 130, 32, "batch", False, True, "prefix", False, "blhd"),      # per-batch bias
    (1, 1, 1, 16, "shared", False, True, "none", False, "bhld"),         # L = 1
    (2, 2, 17, 32, "shared", True, False, "prefix", False, "blhd"),      # tiny ragged, bias^T
    (2, 1, 384, 32, "shared", False, True, "prefix", False, "blhd"),     # cfg5-like L
    (2, 2, 520, 8, None, False, True, "prefix", True, "lbhd"),           # extra-MSA-like, 5 tiles
    (2, 1, 384, 32, None, False, True, "prefix_fm", False, "blhd"),      # no bias, 3 key tiles
    (6, 8, 256, 8, "shared", False, True, "prefix", False, "blhd"),      # extra-MSA row (f3) 8x8
]


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
def test_bf16_parity(case):
    B, H, L, D, bias, bias_t, gate, mask, mask_t, layout = case
    errs, _, _ = run_case(B, H, L, L, D, seed=1, bias=bias, bias_t=bias_t, gate=gate, mask=mask,
                          mask_t=mask_t, layout=layout)
    _assert(errs, torch.bfloat16, str(case))


@pytest.mark.parametrize("case", CASES[:8], ids=[str(c) for c in CASES[:8]])
def test_f32_verification_parity(case):
    B, H, L, D, bias, bias_t, gate, mask, mask_t, layout = case
    errs, _, _ = run_case(B, H, L, L, D, seed=2, bias=bias, bias_t=bias_t, gate=gate, mask=mask,
                          mask_t=mask_t, layout=layout, dtype=torch.float32)
    _assert(errs, torch.float32, str(case))


def test_unequal_lengths():
    errs, _, _ = run_case(2, 2, 70, 200, 32, seed=3, bias="shared", mask="prefix")
    _assert(errs, torch.bfloat16)


@pytest.mark.parametrize("B,H,Lq,Lk,D,bias_t,gate,layout", [
    (6, 3, 256, 140, 16, True, False, "lbhd"),
    (5, 2, 129, 256, 32, False, True, "blhd"),
    (7, 4, 256, 256, 32, True, True, "bhld"),
])
def test_bf16_parity_dq_pair_sum(B, H, Lq, Lk, D, bias_t, gate, layout):
    """A shared bias with two key tiles and Lq <= 256: the two key tiles of a head run as a
    2-CTA cluster that sums dQ on chip (each keeps one 64-query half of every tile, the peer's
    rows arrive by st.async); ragged key and query tiles, D = 16 and 32, gate on and off."""
    errs, _, _ = run_case(B, H, Lq, Lk, D, seed=17, bias="shared", bias_t=bias_t, gate=gate,
                          mask="prefix_fm", mask_t=layout == "lbhd", layout=layout)
    _assert(errs, torch.bfloat16, f"dq pair B={B} H={H} Lq={Lq} Lk={Lk} D={D}")


def test_seeds_cfg1_shape():
    for seed in range(5):
        errs, _, _ = run_case(32, 2, 32, 32, 16, seed=seed, bias="shared", mask="prefix_fm")
        _assert(errs, torch.bfloat16, f"seed {seed}")


def test_fully_masked_rows_are_zero():
    errs, out, c = run_case(4, 2, 64, 64, 32, seed=4, mask="prefix", bwd=True)
    m = c["mask"].copy()
    errs, out, c = run_case(4, 2, 64, 64, 32, seed=4, bwd=True, case=dict(
        c, mask=np.where(np.arange(4)[:, None] == 2, 0, m).astype(np.uint8)))
    assert torch.all(out["o"][2] == 0)
    assert torch.all(torch.isneginf(out["lse"][2]))
    assert torch.all(out["dq"][2] == 0) and torch.all(out["dg"][2] == 0)
    assert torch.all(out["dk"][2] == 0) and torch.all(out["dv"][2] == 0)
    _assert(errs, torch.bfloat16)


def test_masked_keys_inert_bitwise():
    """P4 on the GPU (reading R5): re-randomising K/V at every masked key, and the shared bias
    column of every key masked in ALL batch rows, changes no output bit — o, lse and all five
    gradients."""
    L = 192
    c = attention_case(2, 2, L, L, 32, seed=5, bias="shared", gate=True, mask="prefix")
    c["mask"][:, 180:] = 0  # keys masked in every batch row (their bias columns are inert)
    c["mask"][1, 17] = 0    # an interior hole
    _, out1, _ = run_case(2, 2, L, L, 32, case=c)
    rng = np.random.default_rng(0)
    c2 = dict(c)
    k, v, b = c["k"].copy(), c["v"].copy(), c["bias"].copy()
    drop = c["mask"] == 0
    for bb in range(2):
        idx = np.nonzero(drop[bb])[0]
        k[bb, :, idx] = np.round(rng.standard_normal(k[bb, :, idx].shape) * 8)
        v[bb, :, idx] = np.round(rng.standard_normal(v[bb, :, idx].shape) * 8)
    all_drop = np.nonzero(drop.all(axis=0))[0]
    assert all_drop.size >= 12
    b[:, :, all_drop] = np.round(rng.standard_normal(b[:, :, all_drop].shape) * 8)
    c2.update(k=k, v=v, bias=b)
    _, out2, _ = run_case(2, 2, L, L, 32, case=c2)
    for n in ("o", "lse", "dq", "dk", "dv", "dg", "dbias"):
        assert torch.equal(out1[n], out2[n]), n
    for bb in range(2):  # dK = dV = 0 at masked keys, dbias = 0 at keys masked everywhere
        idx = torch.from_numpy(np.nonzero(drop[bb])[0]).cuda()
        assert torch.all(out1["dk"][bb][:, idx] == 0) and torch.all(out1["dv"][bb][:, idx] == 0)
    assert torch.all(out1["dbias"][:, :, torch.from_numpy(all_drop).cuda()] == 0)


# every backward code path: fused with two key tiles (one fp32 dQ accumulator, reduce-add),
# fused with 3-8 key tiles (per-key-tile fp32 parts), the two-pass path (L > 256 with a bias,
# D = 64, per-batch bias; per-key-tile parts), many batch chunks
DET_CASES = [
    (4, 2, 256, 32, "shared", "blhd"),
    (4, 2, 256, 32, None, "blhd"),
    (2, 2, 384, 32, None, "blhd"),
    (2, 2, 520, 8, None, "lbhd"),
    (16, 8, 1024, 8, None, "lbhd"),
    (2, 2, 384, 32, "shared", "blhd"),
    (2, 2, 300, 64, "shared", "blhd"),
    (2, 2, 130, 32, "batch", "blhd"),
    (40, 2, 256, 32, "shared", "blhd"),
    (40, 4, 384, 32, None, "lbhd"),
]


@pytest.mark.parametrize("case", DET_CASES, ids=[str(c) for c in DET_CASES])
def test_deterministic(case):
    """Bitwise repeatability of every output, dq included (reduction orders in
    DESIGN.md §5): three runs of the same call give identical bits."""
    B, H, L, D, bias, layout = case
    _, a, _ = run_case(B, H, L, L, D, seed=6, bias=bias, mask="prefix", layout=layout)
    for _ in range(2):
        _, b, _ = run_case(B, H, L, L, D, seed=6, bias=bias, mask="prefix", layout=layout)
        for n in ("o", "lse", "dq", "dk", "dv", "dg", "dbias"):
            if a.get(n) is not None:
                assert torch.equal(a[n], b[n]), n


def test_gradient_identities():
    """P7 on the GPU output, with bounds derived from where the kernels round:

    * Σ_k dbias[h,q,k] = Σ_b (Σ_k P dP − D_q): exact arithmetic gives 0; the kernels' D_q is
      Σ_d dO·o with o rounded to bf16 (relative 2^-9 per element), so
      |Σ_k dbias[h,q,k]| <= 2^-8 · Σ_b Σ_d |dO·o| (+ fp32 summation, 2^-20 · Σ_k |dbias|).
    * Σ_k dV[k] = Σ_q (Σ_k P_qk) dA_q with P rounded to bf16 for the MMA (Σ_k |ΔP| <= 2^-9)
      and dv rounded to bf16: |Σ_k dv − Σ_q dA| <= 2^-8 · (Σ_q |dA| + Σ_k |dv|).
    * Σ_k dK[k] = scale · Σ_q (Σ_k bf16(dS_qk)) Q_q with |Σ_k dS_qk| = |ε_q| <= 2^-8 Σ_d|dO·o|
      and the bf16 rounding of dS: |Σ_k bf16(dS_qk) − Σ_k dS_qk| <= 2^-9 Σ_k |dS_qk| <= 2^-9
      (max_k |V_k·dA_q| + |D_q|), plus the bf16 rounding of dk (2^-8 Σ_k |dk|)."""
    B, H, L, D = 8, 2, 256, 32
    _, out, c = run_case(B, H, L, L, D, seed=7, mask="none")
    o = out["o"].double().cpu().numpy()
    dO, g, q, v = (c[n].astype(np.float64) for n in ("dout", "g", "q", "v"))
    scale = c["scale"]
    od = np.abs(dO * o).sum(-1)                       # [B,H,Lq]  Σ_d |dO·o|
    db = out["dbias"].double().cpu().numpy()          # [H,Lq,Lk]
    lhs = np.abs(db.sum(-1))
    rhs = 2.0 ** -8 * od.sum(0) + 2.0 ** -20 * np.abs(db).sum(-1) + 1e-30
    assert np.all(lhs <= rhs), float(np.max(lhs / rhs))
    dA = dO / (1.0 + np.exp(-g))
    dv = out["dv"].double().cpu().numpy()
    lhs = np.abs(dv.sum(2) - dA.sum(2))
    rhs = 2.0 ** -8 * (np.abs(dA).sum(2) + np.abs(dv).sum(2)) + 1e-30
    assert np.all(lhs <= rhs), float(np.max(lhs / rhs))
    dk = out["dk"].double().cpu().numpy()
    Dq = (dO * o).sum(-1)
    dP_max = np.abs(np.einsum("bhkd,bhqd->bhqk", v, dA)).max(-1)   # max_k |V_k·dA_q|
    per_q = 2.0 ** -8 * od + 2.0 ** -9 * (dP_max + np.abs(Dq))     # [B,H,Lq]
    lhs = np.abs(dk.sum(2))
    rhs = scale * np.einsum("bhq,bhqd->bhd", per_q, np.abs(q)) + 2.0 ** -8 * np.abs(dk).sum(2) \
        + 1e-30
    assert np.all(lhs <= rhs), float(np.max(lhs / rhs))


@pytest.mark.parametrize("bias_t", [False, True])
def test_bf16_parity_two_key_tiles(bias_t):
    """Two key tiles (fp32 dQ parts of the fused backward summed by dq_convert), k- and
    q-contiguous bias, against the oracle."""
    errs, _, _ = run_case(3, 2, 256, 256, 32, seed=5, bias="shared", bias_t=bias_t, gate=True,
                          mask="prefix", mask_t=False, layout="blhd")
    _assert(errs, torch.bfloat16, f"two key tiles bias_t={bias_t}")


@pytest.mark.parametrize("B,H,L,bias", [(64, 8, 64, None), (64, 8, 32, None), (40, 2, 256, "shared"),
                                        (200, 1, 128, "shared")])
def test_bf16_parity_many_batch_rows(B, H, L, bias):
    """Several batch rows per fused-backward CTA (batch chunks > 1): the per-row dK/dV drains,
    the cross-row Σ_b dSᵀ and the K/V ring reuse."""
    errs, _, _ = run_case(B, H, L, L, 32, seed=3, bias=bias, gate=True, mask="prefix",
                          mask_t=False, layout="blhd")
    _assert(errs, torch.bfloat16, f"B={B} H={H} L={L} bias={bias}")


@pytest.mark.parametrize("B,H,L,D,mask", [(40, 4, 300, 32, "prefix"), (38, 4, 520, 8, "prefix_fm"),
                                          (150, 1, 256, 16, "prefix"), (37, 4, 512, 32, "prefix_fm")])
def test_bf16_parity_nobias_key_tile_loop(B, H, L, D, mask):
    """No bias, several key tiles, B·H >= the SM count: the no-bias backward walks every key
    tile of a (b, h) row inside one CTA and accumulates dQ of all query tiles in TMEM (no fp32
    parts); the per-group keep mask, the row-level dQ drain and the ragged last tiles."""
    errs, _, _ = run_case(B, H, L, L, D, seed=13, bias=None, gate=True, mask=mask,
                          mask_t=True, layout="lbhd")
    _assert(errs, torch.bfloat16, f"kloop B={B} H={H} L={L} D={D}")


@pytest.mark.parametrize("B,H,L", [(40, 2, 256), (200, 1, 128)])
def test_bf16_parity_end_node_many_chunks(B, H, L):
    """End-node view (q-contiguous bias, transposed mask) with many batch chunks: the transposed
    dbias reduce over more partials than one load round holds (16), and the per-warp drains of
    the fused backward on the [J, I] storage."""
    errs, _, _ = run_case(B, H, L, L, 32, seed=7, bias="shared", bias_t=True, gate=True,
                          mask="prefix", mask_t=True, layout="lbhd")
    _assert(errs, torch.bfloat16, f"end-node B={B} H={H} L={L}")


def _random_cases(n, seed):
    """Seeded random problem shapes over the ABI's whole supported space (every kernel path:
    one to nine key tiles, 256 < L <= 384 with a bias, D = 8..64, per-batch / shared /
    transposed / no bias, masks with fully-masked rows, gate on/off, every storage layout)."""
    r = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        D = int(r.choice([8, 16, 32, 64]))
        bias = r.choice(["shared", "shared", None, "batch"])
        L = int(r.integers(1, 420))
        if bias == "batch":
            L = min(L, 200)
        B = int(r.integers(1, 5))
        H = int(r.integers(1, 5))
        layout = str(r.choice(["blhd", "lbhd", "bhld"]))
        bias_t = bool(bias == "shared" and r.random() < 0.4 and L % 8 == 0)
        mask = str(r.choice(["none", "prefix", "prefix_fm"]))
        out.append((B, H, L, D, None if bias is None else str(bias), bias_t, bool(r.random() < 0.8),
                    mask, layout == "lbhd", layout))
    return out


RANDOM_CASES = _random_cases(40, seed=2026)


@pytest.mark.parametrize("case", RANDOM_CASES, ids=[str(c) for c in RANDOM_CASES])
def test_random_shapes_parity(case):
    """Randomised sweep (seeded, reproducible): every output vs the oracle, bf16 tolerance."""
    B, H, L, D, bias, bias_t, gate, mask, mask_t, layout = case
    errs, _, _ = run_case(B, H, L, L, D, seed=L + 7 * D, bias=bias, bias_t=bias_t, gate=gate,
                          mask=mask, mask_t=mask_t, layout=layout)
    _assert(errs, torch.bfloat16, str(case))
