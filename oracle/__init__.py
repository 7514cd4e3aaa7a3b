"""fp64 CPU oracle for Evoformer gated pair-bias attention — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product package
``paper_2404_11068_b200`` never imports it, and the two share no code.

* ``attn_fwd`` / ``attn_bwd`` wrap the plain C definition in ``evo_oracle.c`` (
  PAPER.md L294 "a pair bias term is added to the logits matrix before the softmax").
* ``modules`` holds the AF2 module-level wrappers (row / column / triangle start / end).

All arrays are numpy float64 in the logical layouts documented in ``evo_oracle.c``; inputs are
converted with ``np.ascontiguousarray(x, dtype=np.float64)`` (exact for bf16/fp32 values).

Parity status: every function here is pinned (tests/test_oracle_pins.py, P1-P13); none is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "evo_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2 -fopenmp, no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            i64, dbl, vp, ci = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int
            lib.oracle_attn_fwd.argtypes = [i64, i64, i64, i64, i64, dbl, vp, vp, vp, ci, vp, vp,
                                            vp, vp, vp]
            lib.oracle_attn_fwd.restype = ci
            lib.oracle_attn_bwd.argtypes = [i64, i64, i64, i64, i64, dbl, vp, vp, vp, ci, vp, vp,
                                            vp, vp, vp, vp, vp, vp, vp]
            lib.oracle_attn_bwd.restype = ci
            lib.oracle_num_threads.restype = ci
            lib.oracle_set_num_threads.argtypes = [ci]
            _lib = lib
    return _lib


def _f64(x):
    return None if x is None else np.ascontiguousarray(x, dtype=np.float64)


def _ptr(x):
    return None if x is None else x.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def set_num_threads(n: int) -> None:
    _load().oracle_set_num_threads(int(n))


def _bias_kind(bias, B, H, Lq, Lk):
    if bias is None:
        return 0
    if bias.shape == (H, Lq, Lk):
        return 1
    if bias.shape == (B, H, Lq, Lk):
        return 2
    raise ValueError(f"bias shape {bias.shape} is neither [H,Lq,Lk] nor [B,H,Lq,Lk]")


def attn_fwd(q, k, v, bias=None, mask=None, g=None, scale=None):
    """Forward oracle. q,g [B,H,Lq,D]; k,v [B,H,Lk,D]; bias [H,Lq,Lk] or [B,H,Lq,Lk];
    mask [B,Lk] (nonzero = keep). ``scale`` defaults to fp32(1/sqrt(D)) widened to fp64
    (reading R2). Returns (o [B,H,Lq,D], lse [B,H,Lq])."""
    q, k, v, bias, g = map(_f64, (q, k, v, bias, g))
    B, H, Lq, D = q.shape
    Lk = k.shape[2]
    if scale is None:
        scale = float(np.float32(1.0 / np.sqrt(D)))
    kind = _bias_kind(bias, B, H, Lq, Lk)
    m = None if mask is None else np.ascontiguousarray(mask != 0, dtype=np.uint8)
    o = np.empty((B, H, Lq, D), np.float64)
    lse = np.empty((B, H, Lq), np.float64)
    rc = _load().oracle_attn_fwd(B, H, Lq, Lk, D, float(scale), _ptr(q), _ptr(k), _ptr(v), kind,
                                 _ptr(bias), _ptr(m), _ptr(g), _ptr(o), _ptr(lse))
    if rc:
        raise RuntimeError(f"oracle_attn_fwd failed rc={rc}")
    return o, lse


def attn_bwd(q, k, v, dout, bias=None, mask=None, g=None, scale=None):
    """Backward oracle (recompute). Returns dict dq, dk, dv, dg (None without gate),
    dbias (None without bias; [H,Lq,Lk] summed over B for the shared kind)."""
    q, k, v, bias, g, dout = map(_f64, (q, k, v, bias, g, dout))
    B, H, Lq, D = q.shape
    Lk = k.shape[2]
    if scale is None:
        scale = float(np.float32(1.0 / np.sqrt(D)))
    kind = _bias_kind(bias, B, H, Lq, Lk)
    m = None if mask is None else np.ascontiguousarray(mask != 0, dtype=np.uint8)
    dq = np.empty_like(q)
    dk = np.empty_like(k)
    dv = np.empty_like(v)
    dg = np.empty_like(q) if g is not None else None
    dbias = np.empty_like(bias) if bias is not None else None
    rc = _load().oracle_attn_bwd(B, H, Lq, Lk, D, float(scale), _ptr(q), _ptr(k), _ptr(v), kind,
                                 _ptr(bias), _ptr(m), _ptr(g), _ptr(dout), _ptr(dq), _ptr(dk),
                                 _ptr(dv), _ptr(dg), _ptr(dbias))
    if rc:
        raise RuntimeError(f"oracle_attn_bwd failed rc={rc}")
    return {"dq": dq, "dk": dk, "dv": dv, "dg": dg, "dbias": dbias}
