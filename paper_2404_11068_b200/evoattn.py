"""Thin Python binding of the C ABI in ``include/evo_attn.h`` (argument marshalling only).

Every step of the attention path runs in ``libevoattn.so`` (hand-written sm_100a kernels).
PyTorch supplies device memory, the current CUDA stream and nothing else.  There is no CPU
fallback: if the library is missing, or a call returns an error, this module raises.

Tensor conventions (logical views; any strides, head dim unit-stride):
  q, g, o, dout : [B, H, Lq, D]        k, v : [B, H, Lk, D]
  bias          : [H, Lq, Lk] (shared over B) or [B, H, Lq, Lk]; q- or k-unit-stride
  mask          : [B, Lk] uint8/bool (nonzero = keep), any strides
  lse           : [B, H, Lq] fp32 contiguous
"""
from __future__ import annotations

import ctypes
import math
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libevoattn.so")
_lock = threading.Lock()
_lib = None

EVO_BF16, EVO_F32 = 0, 1
EVO_BIAS_NONE, EVO_BIAS_SHARED, EVO_BIAS_PER_BATCH = 0, 1, 2
STATUS = {0: "EVO_OK", 1: "EVO_E_INVALID", 2: "EVO_E_SHAPE", 3: "EVO_E_ALIGN",
          4: "EVO_E_UNSUPPORTED", 5: "EVO_E_WORKSPACE", 6: "EVO_E_CUDA"}


class EvoError(RuntimeError):
    def __init__(self, status, detail):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {detail}")


class Desc(ctypes.Structure):
    """Mirror of evo_attn_desc_t (natural C alignment, x86-64)."""
    _fields_ = [
        ("B", ctypes.c_int64), ("H", ctypes.c_int32), ("Lq", ctypes.c_int32),
        ("Lk", ctypes.c_int32), ("D", ctypes.c_int32), ("dtype", ctypes.c_int32),
        ("scale", ctypes.c_float),
        ("q_str", ctypes.c_int64 * 3), ("k_str", ctypes.c_int64 * 3),
        ("v_str", ctypes.c_int64 * 3), ("g_str", ctypes.c_int64 * 3),
        ("o_str", ctypes.c_int64 * 3),
        ("bias_kind", ctypes.c_int32), ("bias_str", ctypes.c_int64 * 4),
        ("has_mask", ctypes.c_int32), ("mask_str", ctypes.c_int64 * 2),
        ("has_gate", ctypes.c_int32),
    ]


class PairBiasDesc(ctypes.Structure):
    """Mirror of evo_pair_bias_desc_t (include/evo_pair_bias.h)."""
    _fields_ = [
        ("Li", ctypes.c_int64), ("Lj", ctypes.c_int64), ("C", ctypes.c_int32),
        ("H", ctypes.c_int32), ("eps", ctypes.c_float),
        ("z_str", ctypes.c_int64 * 3), ("b_str", ctypes.c_int64 * 3),
    ]


class GlobalAttnDesc(ctypes.Structure):
    """Mirror of evo_global_attn_desc_t (include/evo_global_attn.h)."""
    _fields_ = [
        ("B", ctypes.c_int64), ("S", ctypes.c_int32), ("H", ctypes.c_int32),
        ("D", ctypes.c_int32), ("scale", ctypes.c_float),
        ("q_str", ctypes.c_int64 * 3), ("k_str", ctypes.c_int64 * 2),
        ("v_str", ctypes.c_int64 * 2), ("g_str", ctypes.c_int64 * 3),
        ("o_str", ctypes.c_int64 * 3), ("has_mask", ctypes.c_int32),
        ("mask_str", ctypes.c_int64 * 2),
    ]


class LnProjDesc(ctypes.Structure):
    """Mirror of evo_ln_proj_desc_t (include/evo_ln_proj.h)."""
    _fields_ = [
        ("rows", ctypes.c_int64), ("C", ctypes.c_int32), ("N", ctypes.c_int32),
        ("eps", ctypes.c_float), ("x_ld", ctypes.c_int64), ("out_ld", ctypes.c_int64),
    ]


def lib_path() -> str:
    return _LIB_PATH


def load():
    """Load libevoattn.so (raises if it was not built — there is no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                raise RuntimeError(
                    f"{_LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g;"
                    " g.build()'` (no CPU or PyTorch fallback exists)")
            lib = ctypes.CDLL(_LIB_PATH)
            vp, sz, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
            dp = ctypes.POINTER(Desc)
            lib.evo_attn_validate.argtypes = [dp]
            lib.evo_attn_validate.restype = i32
            lib.evo_attn_fwd.argtypes = [dp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
            lib.evo_attn_fwd.restype = i32
            lib.evo_attn_bwd_workspace_bytes.argtypes = [dp]
            lib.evo_attn_bwd_workspace_bytes.restype = sz
            lib.evo_attn_bwd.argtypes = [dp] + [vp] * 15 + [sz, vp]
            lib.evo_attn_bwd.restype = i32
            lib.evo_status_string.argtypes = [i32]
            lib.evo_status_string.restype = ctypes.c_char_p
            lib.evo_last_error_detail.restype = ctypes.c_char_p
            lib.evo_abi_version.restype = i32
            lib.evo_last_launch_count.restype = i32
            lib.evo_trace_enable.argtypes = [vp, i32]
            lib.evo_trace_enable.restype = i32
            lib.evo_trace_count.restype = i32
            lib.evo_trace_label.argtypes = [i32]
            lib.evo_trace_label.restype = ctypes.c_char_p
            pdp = ctypes.POINTER(PairBiasDesc)
            lib.evo_pair_bias_fwd.argtypes = [pdp] + [vp] * 8
            lib.evo_pair_bias_fwd.restype = i32
            lib.evo_pair_bias_bwd_workspace_bytes.argtypes = [pdp]
            lib.evo_pair_bias_bwd_workspace_bytes.restype = sz
            lib.evo_pair_bias_bwd.argtypes = [pdp] + [vp] * 12 + [sz, vp]
            lib.evo_pair_bias_bwd.restype = i32
            gdp = ctypes.POINTER(GlobalAttnDesc)
            lib.evo_global_attn_fwd.argtypes = [gdp] + [vp] * 9
            lib.evo_global_attn_fwd.restype = i32
            lib.evo_global_attn_bwd.argtypes = [gdp] + [vp] * 13
            lib.evo_global_attn_bwd.restype = i32
            lib.evo_ln_proj_fwd.argtypes = [ctypes.POINTER(LnProjDesc)] + [vp] * 9
            lib.evo_ln_proj_fwd.restype = i32
            lib.evo_linear_fwd.argtypes = [ctypes.POINTER(LnProjDesc)] + [vp] * 5
            lib.evo_linear_fwd.restype = i32
            lib.evo_ln_proj_bwd_workspace_bytes.argtypes = [ctypes.POINTER(LnProjDesc)]
            lib.evo_ln_proj_bwd_workspace_bytes.restype = sz
            lib.evo_ln_proj_bwd.argtypes = [ctypes.POINTER(LnProjDesc)] + [vp] * 13 + [sz, vp]
            lib.evo_ln_proj_bwd.restype = i32
            lib.evo_linear_bwd.argtypes = [ctypes.POINTER(LnProjDesc)] + [vp] * 7 + [sz, vp]
            lib.evo_linear_bwd.restype = i32
            _lib = lib
    return _lib


def last_launch_count() -> int:
    return int(load().evo_last_launch_count())


def _check(rc):
    if rc != 0:
        raise EvoError(rc, load().evo_last_error_detail().decode())


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _str3(t):
    s = t.stride()
    if t.size(-1) > 1 and s[-1] != 1:
        raise ValueError("head dimension must be unit-stride")
    return (ctypes.c_int64 * 3)(s[0], s[1], s[2])


def make_desc(q, k, v, bias=None, mask=None, g=None, o=None, scale=None) -> Desc:
    """Build the descriptor for logical views q,k,v(,g,o) [B,H,L,D], bias [H|B,H,Lq,Lk]."""
    B, H, Lq, D = q.shape
    Lk = k.shape[2]
    if k.shape != (B, H, Lk, D) or v.shape != (B, H, Lk, D):
        raise ValueError(f"q {tuple(q.shape)} / k {tuple(k.shape)} / v {tuple(v.shape)} mismatch")
    d = Desc()
    d.B, d.H, d.Lq, d.Lk, d.D = B, H, Lq, Lk, D
    if q.dtype == torch.bfloat16:
        d.dtype = EVO_BF16
    elif q.dtype == torch.float32:
        d.dtype = EVO_F32
    else:
        raise TypeError(f"dtype {q.dtype} not supported (bf16, or fp32 verification mode)")
    for t in (k, v, g, bias, o):
        if t is not None and t.dtype != q.dtype:
            raise TypeError("q, k, v, g, bias, o must share one dtype")
    d.scale = float(scale) if scale is not None else float(torch.tensor(D ** -0.5,
                                                                       dtype=torch.float32))
    d.q_str, d.k_str, d.v_str = _str3(q), _str3(k), _str3(v)
    if o is not None:
        d.o_str = _str3(o)
    if g is not None:
        if g.shape != q.shape:
            raise ValueError("g must have q's shape")
        d.g_str, d.has_gate = _str3(g), 1
    if bias is not None:
        if bias.dim() == 3 and tuple(bias.shape) == (H, Lq, Lk):
            d.bias_kind = EVO_BIAS_SHARED
            s = bias.stride()
            d.bias_str = (ctypes.c_int64 * 4)(0, s[0], s[1], s[2])
        elif bias.dim() == 4 and tuple(bias.shape) == (B, H, Lq, Lk):
            d.bias_kind = EVO_BIAS_PER_BATCH
            d.bias_str = (ctypes.c_int64 * 4)(*bias.stride())
        else:  # bias shape neither [B,H,L,L] nor [H,L,L] -> shape error
            raise ValueError(f"bias shape {tuple(bias.shape)} is neither [H,Lq,Lk] nor [B,H,Lq,Lk]")
    if mask is not None:
        if tuple(mask.shape) != (B, Lk) or mask.dtype not in (torch.uint8, torch.bool):
            raise ValueError("mask must be uint8/bool [B, Lk]")
        d.has_mask = 1
        d.mask_str = (ctypes.c_int64 * 2)(*mask.stride())
    return d


def _alloc_like(t, dtype=None):
    """Output buffer with exactly t's strides (the ABI writes dq/dk/dv/dg/dbias with the
    strides of q/k/v/g/bias)."""
    dtype = t.dtype if dtype is None else dtype
    return torch.empty_strided(tuple(t.shape), tuple(t.stride()), dtype=dtype, device=t.device)


def _stream(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def fwd(q, k, v, bias=None, mask=None, g=None, scale=None, out=None, stream=None):
    """Forward.  Returns (o, lse); o has q's memory layout (``empty_like``)."""
    o = torch.empty_like(q) if out is None else out  # preserve_format: q's layout when dense
    B, H, Lq, _ = q.shape
    lse = torch.empty((B, H, Lq), dtype=torch.float32, device=q.device)
    d = make_desc(q, k, v, bias, mask, g, o, scale)
    m = mask.view(torch.uint8) if (mask is not None and mask.dtype == torch.bool) else mask
    _check(load().evo_attn_fwd(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(bias), _ptr(m),
                               _ptr(g), _ptr(o), _ptr(lse), _stream(stream)))
    return o, lse


def workspace_bytes(q, k, v, bias=None, mask=None, g=None, scale=None) -> int:
    d = make_desc(q, k, v, bias, mask, g, q, scale)
    return int(load().evo_attn_bwd_workspace_bytes(ctypes.byref(d)))


def bwd(q, k, v, o, lse, dout, bias=None, mask=None, g=None, scale=None, workspace=None,
        stream=None, dbias_out=None):
    """Backward.  Returns dict dq, dk, dv, dg (None without gate), dbias (fp32, bias layout;
    None without bias)."""
    if dout.stride() != o.stride():
        dout = dout.contiguous() if o.is_contiguous() else torch.empty_like(o).copy_(dout)
    d = make_desc(q, k, v, bias, mask, g, o, scale)
    ws_need = int(load().evo_attn_bwd_workspace_bytes(ctypes.byref(d)))
    if workspace is None or workspace.numel() < ws_need:
        workspace = torch.empty(max(ws_need, 1), dtype=torch.uint8, device=q.device)
    dq, dk, dv = _alloc_like(q), _alloc_like(k), _alloc_like(v)
    dg = _alloc_like(g) if g is not None else None
    dbias = None
    if bias is not None:
        dbias = _alloc_like(bias, torch.float32) if dbias_out is None else dbias_out
        if dbias.stride() != bias.stride():
            raise ValueError("dbias must have bias's strides (the library writes it that way)")
    m = mask.view(torch.uint8) if (mask is not None and mask.dtype == torch.bool) else mask
    _check(load().evo_attn_bwd(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(bias), _ptr(m),
                               _ptr(g), _ptr(o), _ptr(lse), _ptr(dout), _ptr(dq), _ptr(dk),
                               _ptr(dv), _ptr(dg), _ptr(dbias), _ptr(workspace), ws_need,
                               _stream(stream)))
    return {"dq": dq, "dk": dk, "dv": dv, "dg": dg, "dbias": dbias}


def pad_bias(bias):
    """Return a view of ``bias`` whose non-unit strides are multiples of 16 bytes (TMA rule in
    evo_attn.h); copies only when needed.  Layout marshalling, not arithmetic."""
    if bias is None:
        return None
    es = bias.element_size()
    last = bias.size(-1)
    if bias.stride(-1) == 1 and all((s * es) % 16 == 0 for s, n in
                                    zip(bias.stride()[:-1], bias.shape[:-1]) if n > 1):
        return bias
    mult = 16 // es
    lp = (last + mult - 1) // mult * mult
    buf = torch.zeros(*bias.shape[:-1], lp, dtype=bias.dtype, device=bias.device)
    buf[..., :last].copy_(bias)
    return buf[..., :last]


class EvoAttentionFunction(torch.autograd.Function):
    """o = sigmoid(g) ⊙ softmax(scale·q·kᵀ + bias, masked)·v through the C ABI."""

    @staticmethod
    def forward(ctx, q, k, v, bias, g, mask, scale):
        bias_p = pad_bias(bias)
        o, lse = fwd(q, k, v, bias_p, mask, g, scale)
        ctx.save_for_backward(q, k, v, bias_p, g, mask, o, lse)
        ctx.scale = scale
        ctx.bias_orig = bias is not None
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, bias_p, g, mask, o, lse = ctx.saved_tensors
        r = bwd(q, k, v, o, lse, do, bias_p, mask, g, ctx.scale)
        db = r["dbias"]
        if db is not None:
            db = db.to(bias_p.dtype)
        return r["dq"], r["dk"], r["dv"], db, r["dg"], None, None


def evo_attention(q, k, v, bias=None, g=None, mask=None, scale=None):
    """Differentiable gated pair-bias attention (bf16 or fp32-verification inputs)."""
    return EvoAttentionFunction.apply(q, k, v, bias, g, mask, scale)


# ----------------------------------------------------------------------------- pair-bias side path
def _pb_desc(z, W, eps, b):
    d = PairBiasDesc()
    d.Li, d.Lj, d.C = z.shape
    d.H = W.shape[1]
    d.eps = float(eps)
    d.z_str = (ctypes.c_int64 * 3)(*z.stride())
    d.b_str = (ctypes.c_int64 * 3)(*b.stride())
    return d


def pair_bias_fwd(z, gamma, beta, W, eps=1e-5, bias=None, stream=None):
    """LayerNorm(z) + LinearNoBias into the head-major bias (include/evo_pair_bias.h).
    z [Li, Lj, C] bf16 (channel unit-stride); gamma, beta [C] fp32; W [C, H] fp32 contiguous.
    ``bias``: optional bf16 output view [H, Li, Lj] with any strides (e.g. a transposed or DAP
    layout); default a new contiguous [H, Li, Lj].  Returns (bias, mean, rstd)."""
    Li, Lj, C = z.shape
    H = W.shape[1]
    if bias is None:
        bias = torch.empty((H, Li, Lj), dtype=torch.bfloat16, device=z.device)
    mean = torch.empty((Li, Lj), dtype=torch.float32, device=z.device)
    rstd = torch.empty_like(mean)
    d = _pb_desc(z, W, eps, bias)
    _check(load().evo_pair_bias_fwd(ctypes.byref(d), _ptr(z), _ptr(gamma), _ptr(beta),
                                    _ptr(W.contiguous()), _ptr(bias), _ptr(mean), _ptr(rstd),
                                    _stream(stream)))
    return bias, mean, rstd


def pair_bias_bwd(z, gamma, beta, W, mean, rstd, dbias, eps=1e-5, workspace=None, stream=None):
    """Backward of pair_bias_fwd given dbias [H, Li, Lj] fp32 (any strides).  Returns dict
    dz (bf16, z's strides), dgamma, dbeta [C], dW [C, H] (fp32)."""
    d = _pb_desc(z, W, eps, dbias)
    need = int(load().evo_pair_bias_bwd_workspace_bytes(ctypes.byref(d)))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(max(need, 1), dtype=torch.uint8, device=z.device)
    dz = _alloc_like(z)
    C, H = W.shape
    dgamma = torch.empty(C, dtype=torch.float32, device=z.device)
    dbeta = torch.empty_like(dgamma)
    dW = torch.empty((C, H), dtype=torch.float32, device=z.device)
    _check(load().evo_pair_bias_bwd(ctypes.byref(d), _ptr(z), _ptr(gamma), _ptr(beta),
                                    _ptr(W.contiguous()), _ptr(mean), _ptr(rstd), _ptr(dbias),
                                    _ptr(dz), _ptr(dgamma), _ptr(dbeta), _ptr(dW),
                                    _ptr(workspace), need, _stream(stream)))
    return {"dz": dz, "dgamma": dgamma, "dbeta": dbeta, "dW": dW}


# ----------------------------------------------------------------------------- global column attention
def _ga_desc(q, k, v, g, o, mask, scale):
    d = GlobalAttnDesc()
    d.B, d.S, d.H, d.D = q.shape
    d.scale = float(scale if scale is not None else 1.0 / math.sqrt(q.shape[-1]))
    d.q_str = (ctypes.c_int64 * 3)(*q.stride()[:3])
    d.k_str = (ctypes.c_int64 * 2)(*k.stride()[:2])
    d.v_str = (ctypes.c_int64 * 2)(*v.stride()[:2])
    d.g_str = (ctypes.c_int64 * 3)(*g.stride()[:3])
    d.o_str = (ctypes.c_int64 * 3)(*o.stride()[:3])
    if mask is not None:
        d.has_mask = 1
        d.mask_str = (ctypes.c_int64 * 2)(*mask.stride())
    return d


def global_attn_fwd(q, k, v, g, mask=None, scale=None, stream=None):
    """Extra-MSA global column attention core (include/evo_global_attn.h, AF2 Alg. 19 l.3/5/6).
    q, g [B, S, H, D]; k, v [B, S, D] (one shared head); mask [B, S].  Returns (o, lse, qbar)."""
    o = torch.empty_like(q)
    B, S, H, D = q.shape
    lse = torch.empty((B, H), dtype=torch.float32, device=q.device)
    qbar = torch.empty((B, H, D), dtype=torch.float32, device=q.device)
    d = _ga_desc(q, k, v, g, o, mask, scale)
    m = mask.view(torch.uint8) if (mask is not None and mask.dtype == torch.bool) else mask
    _check(load().evo_global_attn_fwd(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(m), _ptr(g),
                                      _ptr(o), _ptr(lse), _ptr(qbar), _stream(stream)))
    return o, lse, qbar


def global_attn_bwd(q, k, v, g, lse, qbar, dout, mask=None, scale=None, stream=None):
    """Backward of global_attn_fwd.  Returns dict dq, dk, dv, dg (the inputs' strides)."""
    o_like = dout if dout.stride() == q.stride() else dout.contiguous()
    d = _ga_desc(q, k, v, g, o_like, mask, scale)
    dq, dk, dv, dg = _alloc_like(q), _alloc_like(k), _alloc_like(v), _alloc_like(g)
    m = mask.view(torch.uint8) if (mask is not None and mask.dtype == torch.bool) else mask
    _check(load().evo_global_attn_bwd(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(m), _ptr(g),
                                      _ptr(lse), _ptr(qbar), _ptr(o_like), _ptr(dq), _ptr(dk),
                                      _ptr(dv), _ptr(dg), _stream(stream)))
    return {"dq": dq, "dk": dk, "dv": dv, "dg": dg}


def ln_proj_fwd(x, gamma, beta, W, b=None, eps=1e-5, out=None, stream=None):
    """Fused LayerNorm + stacked projection (include/evo_ln_proj.h).
    x [rows, C] bf16 (row stride x.stride(0)); W [N, C] bf16 (nn.Linear layout, q|k|v|g stacked);
    gamma, beta [C] fp32; b [N] fp32 or None.  Returns (out [rows, N] bf16, mean, rstd)."""
    rows, C = x.shape
    N = W.shape[0]
    if out is None:
        out = torch.empty((rows, N), dtype=torch.bfloat16, device=x.device)
    mean = torch.empty(rows, dtype=torch.float32, device=x.device)
    rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
    d = LnProjDesc()
    d.rows, d.C, d.N, d.eps = rows, C, N, eps
    d.x_ld, d.out_ld = x.stride(0), out.stride(0)
    _check(load().evo_ln_proj_fwd(ctypes.byref(d), _ptr(x), _ptr(gamma), _ptr(beta),
                                  _ptr(W.contiguous()), _ptr(b), _ptr(out), _ptr(mean),
                                  _ptr(rstd), _stream(stream)))
    return out, mean, rstd


def linear_fwd(x, W, b=None, out=None, stream=None):
    """out = x·Wᵀ + b on the tcgen05 projection kernel without the LayerNorm (evo_linear_fwd,
    include/evo_ln_proj.h): e.g. the attention output projection.  x [rows, C] bf16; W [N, C]
    bf16; b [N] fp32 or None."""
    rows, C = x.shape
    N = W.shape[0]
    if out is None:
        out = torch.empty((rows, N), dtype=torch.bfloat16, device=x.device)
    d = LnProjDesc()
    d.rows, d.C, d.N, d.eps = rows, C, N, 0.0
    d.x_ld, d.out_ld = x.stride(0), out.stride(0)
    _check(load().evo_linear_fwd(ctypes.byref(d), _ptr(x), _ptr(W.contiguous()), _ptr(b),
                                 _ptr(out), _stream(stream)))
    return out


def ln_proj_bwd(x, gamma, beta, W, mean, rstd, dout, eps=1e-5, want_db=True, workspace=None,
                stream=None):
    """Backward of ln_proj_fwd (include/evo_ln_proj.h evo_ln_proj_bwd): dout [rows, N] bf16 ->
    dict dx [rows, C] bf16, dgamma, dbeta [C] fp32, dW [N, C] fp32, db [N] fp32 (or None)."""
    rows, C = x.shape
    N = W.shape[0]
    dx = torch.empty((rows, C), dtype=torch.bfloat16, device=x.device)
    dgamma = torch.empty(C, dtype=torch.float32, device=x.device)
    dbeta = torch.empty(C, dtype=torch.float32, device=x.device)
    dW = torch.empty((N, C), dtype=torch.float32, device=x.device)
    db = torch.empty(N, dtype=torch.float32, device=x.device) if want_db else None
    d = LnProjDesc()
    d.rows, d.C, d.N, d.eps = rows, C, N, eps
    d.x_ld, d.out_ld = x.stride(0), dout.stride(0)
    L = load()
    need = int(L.evo_ln_proj_bwd_workspace_bytes(ctypes.byref(d)))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(max(need, 16), dtype=torch.uint8, device=x.device)
    _check(L.evo_ln_proj_bwd(ctypes.byref(d), _ptr(x), _ptr(gamma), _ptr(beta),
                             _ptr(W.contiguous()), _ptr(mean), _ptr(rstd), _ptr(dout), _ptr(dx),
                             _ptr(dgamma), _ptr(dbeta), _ptr(dW), _ptr(db), _ptr(workspace), need,
                             _stream(stream)))
    return {"dx": dx, "dgamma": dgamma, "dbeta": dbeta, "dW": dW, "db": db}


def linear_bwd(x, W, dout, want_db=True, workspace=None, stream=None):
    """Backward of linear_fwd (evo_linear_bwd): dx = dout·W (bf16), dW = doutᵀ·x, db."""
    rows, C = x.shape
    N = W.shape[0]
    dx = torch.empty((rows, C), dtype=torch.bfloat16, device=x.device)
    dW = torch.empty((N, C), dtype=torch.float32, device=x.device)
    db = torch.empty(N, dtype=torch.float32, device=x.device) if want_db else None
    d = LnProjDesc()
    d.rows, d.C, d.N, d.eps = rows, C, N, 0.0
    d.x_ld, d.out_ld = x.stride(0), dout.stride(0)
    L = load()
    need = int(L.evo_ln_proj_bwd_workspace_bytes(ctypes.byref(d)))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(max(need, 16), dtype=torch.uint8, device=x.device)
    _check(L.evo_linear_bwd(ctypes.byref(d), _ptr(x), _ptr(W.contiguous()), _ptr(dout), _ptr(dx),
                            _ptr(dW), _ptr(db), _ptr(workspace), need, _stream(stream)))
    return {"dx": dx, "dW": dW, "db": db}
