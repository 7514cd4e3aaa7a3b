"""Pins for the global column attention oracle (oracle/global_attn.py, AF2 Alg. 19 core)."""
import numpy as np
import pytest
import torch

import oracle
from oracle.global_attn import global_attn_bwd, global_attn_fwd


def _case(B=3, S=7, H=2, D=4, seed=0, masked=True):
    r = np.random.default_rng(seed)
    q, g = r.standard_normal((B, S, H, D)), r.standard_normal((B, S, H, D))
    k, v = r.standard_normal((B, S, D)), r.standard_normal((B, S, D))
    mask = np.ones((B, S), np.uint8)
    if masked:
        mask[1, min(4, S - 1):] = 0
        if B > 2:
            mask[2, :] = 0  # a column with no kept sequence
    return q, k, v, g, mask, 1 / np.sqrt(D)


def test_equals_core_oracle_with_one_query():
    """For each head, Alg. 19's core is the regular gated attention core with a single query
    q̄ (the C oracle, an independent implementation) and the gate applied per sequence."""
    q, k, v, g, mask, scale = _case(masked=False)
    o, lse, qbar, attn = global_attn_fwd(q, k, v, g, mask, scale)
    B, S, H, D = q.shape
    for h in range(H):
        qq = qbar[:, h][:, None, None, :]                     # [B, 1 head, 1 query, D]
        kk, vv = k[:, None], v[:, None]                       # [B, 1, S, D]
        oc, lc = oracle.attn_fwd(qq, kk, vv, None, mask, None, scale)
        assert np.max(np.abs(oc[:, 0, 0] - attn[:, h])) < 1e-12
        assert np.max(np.abs(lc[:, 0, 0] - lse[:, h])) < 1e-12
    assert np.allclose(o, 1 / (1 + np.exp(-g)) * attn[:, None])


def test_single_sequence_and_uniform_keys():
    q, k, v, g, mask, scale = _case(S=1, masked=False)
    o, _, _, attn = global_attn_fwd(q, k, v, g, mask, scale)
    assert np.allclose(attn, np.repeat(v[:, :1], q.shape[2], axis=1))       # a = 1
    q2, k2, v2, g2, mask2, _ = _case(masked=False, seed=3)
    k2[:] = k2[:, :1]                                                       # identical keys
    _, _, _, attn2 = global_attn_fwd(q2, k2, v2, g2, mask2, scale)
    assert np.allclose(attn2, v2.mean(axis=1)[:, None, :].repeat(q2.shape[2], axis=1))


def test_masked_sequences_are_inert_and_empty_column():
    q, k, v, g, mask, scale = _case()
    o, lse, _, _ = global_attn_fwd(q, k, v, g, mask, scale)
    q2, k2, v2 = q.copy(), k.copy(), v.copy()
    q2[1, 4:] += 5; k2[1, 4:] -= 3; v2[1, 4:] *= 7                        # finite changes
    o2, _, _, _ = global_attn_fwd(q2, k2, v2, g, mask, scale)
    assert np.array_equal(o[:, :4], o2[:, :4]) and np.array_equal(o[0], o2[0])
    assert np.all(o[2] == 0) and np.all(np.isneginf(lse[2]))
    r = global_attn_bwd(q, k, v, g, mask, scale, np.ones_like(q))
    assert np.all(r["dq"][1, 4:] == 0) and np.all(r["dk"][1, 4:] == 0) and np.all(r["dv"][1, 4:] == 0)
    assert all(np.all(r[n][2] == 0) for n in ("dq", "dk", "dv", "dg"))


def test_bwd_equals_torch_autograd():
    q, k, v, g, mask, scale = _case(seed=1)
    dout = np.random.default_rng(9).standard_normal(q.shape)
    tq, tk, tv, tg = (torch.from_numpy(x).requires_grad_() for x in (q, k, v, g))
    m = torch.from_numpy(mask.astype(np.float64))
    cnt = m.sum(1).clamp(min=1.0)
    qbar = torch.einsum("bs,bshd->bhd", m, tq) / cnt[:, None, None]
    logits = scale * torch.einsum("bhd,btd->bht", qbar, tk)
    logits = logits.masked_fill(m[:, None, :] == 0, float("-inf"))
    keep = (m.sum(1) > 0)[:, None, None]
    a = torch.where(keep, torch.softmax(torch.where(keep, logits, torch.zeros_like(logits)), -1)
                    * (m[:, None, :] > 0), torch.zeros_like(logits))
    attn = torch.einsum("bht,btd->bhd", a, tv)
    o = torch.sigmoid(tg) * attn[:, None]
    (o * torch.from_numpy(dout)).sum().backward()
    r = global_attn_bwd(q, k, v, g, mask, scale, dout)
    for n, t in (("dq", tq), ("dk", tk), ("dv", tv), ("dg", tg)):
        assert np.max(np.abs(r[n] - t.grad.numpy())) < 1e-12, n


def test_finite_differences():
    q, k, v, g, mask, scale = _case(B=2, S=4, H=2, D=3, seed=2)
    dout = np.random.default_rng(4).standard_normal(q.shape)
    r = global_attn_bwd(q, k, v, g, mask, scale, dout)
    loss = lambda *a: float((global_attn_fwd(*a, mask, scale)[0] * dout).sum())
    h = 1e-6
    for name, pos in (("dq", 0), ("dk", 1), ("dv", 2), ("dg", 3)):
        base = [q, k, v, g]
        arr = base[pos]
        num = np.zeros_like(arr)
        it = np.nditer(arr, flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            p_ = [x.copy() for x in base]; m_ = [x.copy() for x in base]
            p_[pos][idx] += h; m_[pos][idx] -= h
            num[idx] = (loss(*p_) - loss(*m_)) / (2 * h)
        err = np.max(np.abs(num - r[name])) / max(np.max(np.abs(r[name])), 1e-30)
        assert err < 1e-6, (name, err)
