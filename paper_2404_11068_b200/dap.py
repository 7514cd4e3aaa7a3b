"""Dynamic Axial Parallelism (DAP) for the Evoformer attention modules.

PAPER.md L207: DAP "splits intermediate activations and associated computations of a single
training sample along a non-reductive axis"; L243: DAP adds all-gather and all-to-all
communications; SURVEY.md §8(e) gives the per-module shard axes:

  module  local batch rows        before the call                      after the bwd
  row     S/n  (m sharded on S)   AG(bias rows)                         RS(dbias)
  col     R/n  (m sharded on R)   a2a m: S-sharded -> R-sharded          reverse a2a (grads)
  start   I/n  (z sharded on I)   AG(bias rows)                         RS(dbias)
  end     J/n  (z sharded on J)   a2a z: I-sharded -> J-sharded; AG      RS(dbias); reverse a2a

Every (b, h) attention problem is independent, so each rank runs the unchanged attention core
(include/evo_attn.h) on its B/n batch rows; the only exchanges are the transposes between the
two shard axes and the bias all-gather / dbias reduce-scatter (include/evo_dap.h).

The attention-core block modelled here (`DapEvoformerAttention`) follows the data flow of one
Evoformer block with the projections/LayerNorm/transitions outside the core:
the row-attention output (c_m = H·D = 256 channels, exactly m's width) is transposed to feed the
column attention, the column output is transposed back (the next block's S-sharded m), and the
same for the pair stack (start -> end).  Backward runs in reverse with the reverse transposes.
That gives the paper's per-block count: 4 a2a fwd + 4 a2a bwd, 3 AG, 3 RS.

Two objects are injected so the host logic can be tested without a GPU:
  comm — `NcclDap` (libevodap.so, the product) or any object with n, rank, transpose(src, dir),
         allgather(src), reduce_scatter(src);
  attn — the `evoattn` binding (the product) or any object with its fwd/bwd signature.
"""
from __future__ import annotations

import ctypes
import os
import threading

from . import modules as M

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libevodap.so")
_lock = threading.Lock()
_lib = None


def load():
    """Load libevodap.so (raises if it was not built — there is no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                raise RuntimeError(f"{_LIB_PATH} is missing: run paper_2404_11068_b200/build.py")
            L = ctypes.CDLL(_LIB_PATH)
            L.evo_dap_last_error_detail.restype = ctypes.c_char_p
            L.evo_dap_a2a_staging_bytes.restype = ctypes.c_size_t
            L.evo_dap_a2a_staging_bytes.argtypes = [ctypes.c_void_p, ctypes.c_int64,
                                                    ctypes.c_int64, ctypes.c_int64]
            L.evo_dap_alltoall_transpose.argtypes = [
                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                ctypes.c_size_t, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                ctypes.c_void_p]
            L.evo_dap_allgather.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_size_t, ctypes.c_void_p]
            L.evo_dap_reduce_scatter_f32.argtypes = [ctypes.c_void_p, ctypes.c_void_p,
                                                     ctypes.c_void_p, ctypes.c_size_t,
                                                     ctypes.c_void_p]
            L.evo_dap_pack.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                       ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int32, ctypes.c_void_p]
            L.evo_dap_barrier.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
            L.evo_dap_wait.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double]
            L.evo_dap_init.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
                                       ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]
            L.evo_dap_destroy.argtypes = [ctypes.c_void_p]
            L.evo_dap_nranks.argtypes = [ctypes.c_void_p]
            L.evo_dap_rank.argtypes = [ctypes.c_void_p]
            _lib = L
    return _lib


def _nvtx(name):
    """NVTX range around a DAP phase or exchange (shows up in nsys / ncu timelines; a no-op
    context without CUDA, e.g. in the gloo tests)."""
    import contextlib
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.nvtx.range(name)
    except Exception:
        pass
    return contextlib.nullcontext()


def _check(rc):
    if rc != 0:
        from .evoattn import EvoError
        raise EvoError(rc, load().evo_dap_last_error_detail().decode())


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


def pack(src, dst, n, A_loc, Bd, C_bytes, direction, stream=None):
    """evo_dap_pack: the layout step of the transpose alone (tests / fused callers)."""
    _check(load().evo_dap_pack(_p(src), _p(dst), n, A_loc, Bd, C_bytes, direction,
                               _stream(stream)))


class _stdout_to_stderr:
    """Redirect the process-level stdout (fd 1) to stderr for the duration of a native call."""

    def __enter__(self):
        import sys
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)

    def __exit__(self, *exc):
        os.dup2(self.saved, 1)
        os.close(self.saved)


class NcclDap:
    """One NCCL communicator over the torch.distributed world (include/evo_dap.h).  The NCCL
    unique id travels over the torch.distributed store."""

    def __init__(self, store_key="evo_dap_uid"):
        import torch
        import torch.distributed as dist
        self.n = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.device = torch.cuda.current_device()
        L = load()
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _check(L.evo_dap_unique_id(uid))
        if self.n > 1:
            obj = [bytes(uid.raw) if self.rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid = ctypes.create_string_buffer(obj[0], 128)
        h = ctypes.c_void_p()
        with _stdout_to_stderr():  # NCCL's init banner must not land in a JSON-line stdout
            _check(L.evo_dap_init(self.n, self.rank, uid, self.device, ctypes.byref(h)))
        self.h = h
        self._scratch = torch.zeros(4, dtype=torch.float32, device="cuda")
        self._staging = None

    def close(self):
        if self.h:
            _check(load().evo_dap_destroy(self.h))
            self.h = None

    def _stage(self, nbytes):
        import torch
        if self._staging is None or self._staging.numel() < nbytes:
            self._staging = torch.empty(max(nbytes, 16), dtype=torch.uint8, device="cuda")
        return self._staging

    def transpose(self, src, direction, out=None, stream=None):
        """dir 0: src row shard [A/n, Bd, ...] -> column shard [A, Bd/n, ...]; dir 1 inverse.
        src must be contiguous (the shard storage)."""
        import torch
        if not src.is_contiguous():
            raise ValueError("transpose: src must be the contiguous shard storage")
        n = self.n
        rest = tuple(src.shape[2:])
        C_bytes = src.element_size()
        for s in rest:
            C_bytes *= s
        if direction == 0:
            A, Bd = src.shape[0] * n, src.shape[1]
            shape = (A, Bd // n) + rest
        else:
            A, Bd = src.shape[0], src.shape[1] * n
            shape = (A // n, Bd) + rest
        dst = out if out is not None else torch.empty(shape, dtype=src.dtype, device=src.device)
        nst = int(load().evo_dap_a2a_staging_bytes(self.h, A, Bd, C_bytes))
        st = self._stage(nst)
        with _nvtx(f"dap.transpose.dir{direction}"):
            _check(load().evo_dap_alltoall_transpose(self.h, _p(src), _p(dst), _p(st), nst, A, Bd,
                                                     C_bytes, direction, _stream(stream)))
        return dst

    def allgather(self, src, out=None, stream=None):
        import torch
        if not src.is_contiguous():
            raise ValueError("allgather: src must be contiguous")
        dst = out if out is not None else torch.empty((src.shape[0] * self.n,) + tuple(src.shape[1:]),
                                                      dtype=src.dtype, device=src.device)
        with _nvtx("dap.allgather"):
            _check(load().evo_dap_allgather(self.h, _p(src), _p(dst),
                                            src.numel() * src.element_size(), _stream(stream)))
        return dst

    def reduce_scatter(self, src, out=None, stream=None):
        import torch
        if not src.is_contiguous() or src.dtype != torch.float32:
            raise ValueError("reduce_scatter: src must be contiguous fp32")
        dst = out if out is not None else torch.empty((src.shape[0] // self.n,) + tuple(src.shape[1:]),
                                                      dtype=src.dtype, device=src.device)
        with _nvtx("dap.reduce_scatter"):
            _check(load().evo_dap_reduce_scatter_f32(self.h, _p(src), _p(dst), dst.numel(),
                                                     _stream(stream)))
        return dst

    def barrier(self, stream=None):
        _check(load().evo_dap_barrier(self.h, _p(self._scratch), _stream(stream)))

    def wait(self, stream=None, timeout_s=300.0):
        """Block until `stream` is idle while polling NCCL's asynchronous error state; a
        peer failure or a hang longer than timeout_s aborts the communicator and raises
        (evo_dap_wait, include/evo_dap.h)."""
        _check(load().evo_dap_wait(self.h, _stream(stream), float(timeout_s)))


# ----------------------------------------------------------------------------- shard plan
def shard(n, rank, extent, what):
    """(start, stop) of rank's slice of an axis of `extent` split evenly over n ranks."""
    if extent % n:
        raise ValueError(f"DAP-{n}: {what} = {extent} is not divisible by {n}")
    w = extent // n
    return rank * w, (rank + 1) * w


def plan(n, n_seq, n_res, heads_m=8, heads_z=4, head_dim=32):
    """Local call shapes of the four modules under DAP-n:
    name -> (B_local, H, L).  Raises if an axis does not divide."""
    shard(n, 0, n_seq, "N_seq")
    shard(n, 0, n_res, "N_res")
    return {"row": (n_seq // n, heads_m, n_res), "col": (n_res // n, heads_m, n_seq),
            "start": (n_res // n, heads_z, n_res), "end": (n_res // n, heads_z, n_res)}


def block_flops(n_seq, n_res, heads_m=8, heads_z=4, head_dim=32):
    """Algorithmic fwd+bwd flops of the block's four attention calls (12·B·H·L²·D each)."""
    f = 12.0 * head_dim
    return f * (n_seq * heads_m * n_res ** 2 + n_res * heads_m * n_seq ** 2
                + 2 * n_res * heads_z * n_res ** 2)


# ----------------------------------------------------------------------------- the block
class DapEvoformerAttention:
    """The four attention modules of one Evoformer block on this rank's DAP shards.

    Local inputs (storage layouts of modules.py; the rank's shard along the DAP axis):
      row   q,k,v,g [S/n, R, Hm, D]   E_row   [R/n, Hm, R] (bias rows of this rank)
      col   k,v,g   [S, R/n, Hm, D]   (q is the transposed row output)
      start q,k,v,g [I/n, J, Hz, D]   E_start [J/n, Hz, J]
      end   k,v,g   [I, J/n, Hz, D]   E_end   [I/n, Hz, I]  (q is the transposed start output)
      masks (storage orientation, this rank's slice): mask_row = msa_mask[S/n rows],
      mask_col = msa_mask[:, R/n cols], mask_start = pair_mask[I/n rows],
      mask_end = pair_mask[:, J/n cols]
    forward() returns the block outputs m_next [S/n, R, Hm·D] and z_next [I/n, J, Hz·D];
    backward(dm_next, dz_next) returns every input gradient on its shard (dbias shards fp32).
    """

    def __init__(self, comm, attn, inputs, pair=None):
        """pair = (comm2, stream): run the pair stack (triangle start/end and their exchanges)
        on `stream` with its own communicator while the MSA stack runs on the caller's stream
        (one stack's collectives overlap the other's attention); the two
        stacks of the attention core are independent inside a block.  None: one stream."""
        self.comm, self.attn, self.x = comm, attn, inputs
        self.n, self.rank = comm.n, comm.rank
        self.pair = pair

    def _fork(self):
        """-> (pair-stack comm, stream context, join()): fork the pair stack onto its stream."""
        import contextlib
        if self.pair is None:
            return self.comm, contextlib.nullcontext(), (lambda *outs: None)
        import torch
        comm2, st2 = self.pair
        main = torch.cuda.current_stream()
        st2.wait_stream(main)

        def join(*outs):
            main.wait_stream(st2)
            for t in outs:  # produced on the pair stream, consumed on the caller's
                if t is not None:
                    t.record_stream(main)
        return comm2, torch.cuda.stream(st2), join

    def forward(self):
        x, c = self.x, self.comm
        s = {}
        cz, ctx, join = self._fork()
        with ctx, _nvtx("dap.fwd.pair_stack"):
            z_next = self._forward_pair(x, cz, s)
        with _nvtx("dap.fwd.msa_stack"):
            self._forward_msa(x, c, s)
        join(z_next, s["o_st"], s["o_end"])
        self.saved = s
        return s.pop("m_next"), z_next, {"o_row": s.pop("o_row"), "o_col": s.pop("o_col"),
                                         "o_start": s["o_st"], "o_end": s["o_end"]}

    def _forward_msa(self, x, c, s):
        # MSA stack: bias AG -> row attention -> a2a (S -> R) -> column attention -> a2a back
        s["E_row"] = c.allgather(x["E_row"])
        o_row, o_row_v, s["lse_row"] = M.attention_fwd("row", x["row_q"], x["row_k"], x["row_v"],
                                                       x["row_g"], s["E_row"], x["mask_row"],
                                                       self.attn)
        s["o_row_v"] = o_row_v
        S_loc, R, Hm, D = o_row.shape
        s["col_q"] = c.transpose(o_row.reshape(S_loc, R, Hm * D), 0).view(S_loc * self.n, R // self.n, Hm, D)
        o_col, s["o_col_v"], s["lse_col"] = M.attention_fwd("col", s["col_q"], x["col_k"], x["col_v"],
                                                            x["col_g"], None, x["mask_col"],
                                                            self.attn)
        s["m_next"] = c.transpose(o_col.reshape(o_col.shape[0], o_col.shape[1], Hm * D), 1)
        s["o_row"], s["o_col"] = o_row, o_col

    def _forward_pair(self, x, c, s):
        # pair stack: bias AG -> triangle start -> a2a (I -> J) -> triangle end -> a2a back
        s["E_start"] = c.allgather(x["E_start"])
        o_st, s["o_st_v"], s["lse_st"] = M.attention_fwd("start", x["st_q"], x["st_k"], x["st_v"],
                                                         x["st_g"], s["E_start"], x["mask_start"],
                                                         self.attn)
        I_loc, J, Hz, Dz = o_st.shape
        s["end_q"] = c.transpose(o_st.reshape(I_loc, J, Hz * Dz), 0).view(I_loc * self.n, J // self.n, Hz, Dz)
        s["E_end"] = c.allgather(x["E_end"])
        o_end, s["o_end_v"], s["lse_end"] = M.attention_fwd("end", s["end_q"], x["end_k"], x["end_v"],
                                                            x["end_g"], s["E_end"], x["mask_end"],
                                                            self.attn)
        z_next = c.transpose(o_end.reshape(o_end.shape[0], o_end.shape[1], Hz * Dz), 1)
        s["o_st"], s["o_end"] = o_st, o_end
        return z_next

    def backward(self, dm_next, dz_next):
        x, c, s = self.x, self.comm, self.saved
        g = {}
        cz, ctx, join = self._fork()
        with ctx, _nvtx("dap.bwd.pair_stack"):
            self._backward_pair(x, cz, s, g, dz_next)
        with _nvtx("dap.bwd.msa_stack"):
            self._backward_msa(x, c, s, g, dm_next)
        join(*g.values())
        return g

    def _backward_pair(self, x, c, s, g, dz_next):
        # pair stack, reversed: dz (I-sharded) -> J-sharded -> end bwd -> RS(dE_end); dq_end -> I
        Hz, Dz = x["st_q"].shape[2], x["st_q"].shape[3]
        d_end = c.transpose(dz_next.contiguous(), 0)
        d_end = d_end.view(d_end.shape[0], d_end.shape[1], Hz, Dz)
        r = M.attention_bwd("end", s["end_q"], x["end_k"], x["end_v"], x["end_g"], s["E_end"],
                            x["mask_end"], s["o_end_v"], s["lse_end"], d_end, self.attn)
        g["end_k"], g["end_v"], g["end_g"] = r["dk"], r["dv"], r["dg"]
        g["E_end"] = c.reduce_scatter(_dense(r["dE"]))
        dq_end = r["dq"]  # [I, J/n, Hz, D] storage
        d_st = c.transpose(_dense(dq_end).reshape(dq_end.shape[0], dq_end.shape[1], Hz * Dz), 1)
        d_st = d_st.view(d_st.shape[0], d_st.shape[1], Hz, Dz)
        r = M.attention_bwd("start", x["st_q"], x["st_k"], x["st_v"], x["st_g"], s["E_start"],
                            x["mask_start"], s["o_st_v"], s["lse_st"], d_st, self.attn)
        g["st_q"], g["st_k"], g["st_v"], g["st_g"] = r["dq"], r["dk"], r["dv"], r["dg"]
        g["E_start"] = c.reduce_scatter(_dense(r["dE"]))

    def _backward_msa(self, x, c, s, g, dm_next):
        # MSA stack, reversed: dm (S-sharded) -> R-sharded -> col bwd; dq_col -> S -> row bwd
        Hm, D = x["row_q"].shape[2], x["row_q"].shape[3]
        d_col = c.transpose(dm_next.contiguous(), 0)
        d_col = d_col.view(d_col.shape[0], d_col.shape[1], Hm, D)
        r = M.attention_bwd("col", s["col_q"], x["col_k"], x["col_v"], x["col_g"], None,
                            x["mask_col"], s["o_col_v"], s["lse_col"], d_col, self.attn)
        g["col_k"], g["col_v"], g["col_g"] = r["dk"], r["dv"], r["dg"]
        dq_col = r["dq"]
        d_row = c.transpose(_dense(dq_col).reshape(dq_col.shape[0], dq_col.shape[1], Hm * D), 1)
        d_row = d_row.view(d_row.shape[0], d_row.shape[1], Hm, D)
        r = M.attention_bwd("row", x["row_q"], x["row_k"], x["row_v"], x["row_g"], s["E_row"],
                            x["mask_row"], s["o_row_v"], s["lse_row"], d_row, self.attn)
        g["row_q"], g["row_k"], g["row_v"], g["row_g"] = r["dq"], r["dk"], r["dv"], r["dg"]
        g["E_row"] = c.reduce_scatter(_dense(r["dE"]))


class DapEvoformerStack:
    """`n_blocks` Evoformer blocks' attention cores chained (PAPER.md L264 / SURVEY §8(f) f4: the
    48-block stack under one CUDA graph): block i+1's MSA-row query is block i's m_next and its
    triangle-start query is block i's z_next (the projections between blocks are outside the
    attention core); the backward chains dm/dz back through the blocks.  The per-block k, v, g,
    bias and mask tensors are shared by every block (synthetic inputs; the timing is the same as
    with distinct tensors of the same shapes)."""

    def __init__(self, comm, attn, inputs, n_blocks, pair=None):
        self.blocks = []
        self.x0 = inputs
        for _ in range(n_blocks):
            self.blocks.append(DapEvoformerAttention(comm, attn, dict(inputs), pair))

    def forward(self):
        m, z = None, None
        for i, blk in enumerate(self.blocks):
            if i > 0:
                S_loc, R, _ = m.shape
                blk.x["row_q"] = m.view(S_loc, R, *self.x0["row_q"].shape[2:])
                I_loc, J, _ = z.shape
                blk.x["st_q"] = z.view(I_loc, J, *self.x0["st_q"].shape[2:])
            m, z, _ = blk.forward()
        return m, z

    def backward(self, dm_next, dz_next):
        dm, dz = dm_next, dz_next
        g = None
        for blk in reversed(self.blocks):
            g = blk.backward(dm, dz)
            dm = g["row_q"].reshape(g["row_q"].shape[0], g["row_q"].shape[1], -1)
            dz = g["st_q"].reshape(g["st_q"].shape[0], g["st_q"].shape[1], -1)
        return dm, dz, g


def _dense(t):
    """The core writes outputs with the strides of the corresponding input; the storage views
    used here are therefore contiguous already.  Refuse silently-copying layouts."""
    if not t.is_contiguous():
        raise ValueError("expected a contiguous storage view (layout contract of modules.py)")
    return t


def make_block_inputs(torch, n, rank, n_seq, n_res, heads_m=8, heads_z=4, head_dim=32, seed=0,
                      device="cpu", dtype=None, mask="ones"):
    """Seeded synthetic block inputs (DESIGN.md §3 recipe: N(0,1), bf16-rounded) generated as
    full tensors on the host and sliced to this rank's DAP shards.  Returns (local dict, full
    dict); the full dict (host) is what single-GPU / oracle references consume."""
    dtype = dtype or torch.bfloat16
    gen = torch.Generator(device="cpu").manual_seed(seed)
    S, R, I = n_seq, n_res, n_res
    Hm, Hz, D = heads_m, heads_z, head_dim

    def rnd(*shape):
        return torch.randn(shape, generator=gen).to(torch.bfloat16)

    full = {}
    for p in ("row_q", "row_k", "row_v", "row_g", "col_k", "col_v", "col_g"):
        full[p] = rnd(S, R, Hm, D)
    for p in ("st_q", "st_k", "st_v", "st_g", "end_k", "end_v", "end_g"):
        full[p] = rnd(I, I, Hz, D)
    full["E_row"] = rnd(R, Hm, R)
    full["E_start"] = rnd(I, Hz, I)
    full["E_end"] = rnd(I, Hz, I)
    full["dm_next"] = rnd(S, R, Hm * D)
    full["dz_next"] = rnd(I, I, Hz * D)
    if mask == "ones":
        full["msa_mask"] = torch.ones((S, R), dtype=torch.uint8)
        full["pair_mask"] = torch.ones((I, I), dtype=torch.uint8)
    else:  # prefix-valid crops: residues beyond n_valid and rows beyond s_valid
        nv = max(1, (3 * R) // 4 + int(torch.randint(0, R // 4 + 1, (1,), generator=gen)))
        sv = max(1, S // 2 + int(torch.randint(0, S // 2 + 1, (1,), generator=gen)))
        mm = torch.zeros((S, R), dtype=torch.uint8)
        mm[:sv, :nv] = 1
        pm = torch.zeros((I, I), dtype=torch.uint8)
        pm[:nv, :nv] = 1
        full["msa_mask"], full["pair_mask"] = mm, pm

    s0, s1 = shard(n, rank, S, "N_seq")
    r0, r1 = shard(n, rank, R, "N_res")
    loc = {}
    for p in ("row_q", "row_k", "row_v", "row_g"):
        loc[p] = full[p][s0:s1]
    for p in ("col_k", "col_v", "col_g"):
        loc[p] = full[p][:, r0:r1]
    for p in ("st_q", "st_k", "st_v", "st_g"):
        loc[p] = full[p][r0:r1]
    for p in ("end_k", "end_v", "end_g"):
        loc[p] = full[p][:, r0:r1]
    for p in ("E_row", "E_start", "E_end"):
        loc[p] = full[p][r0:r1]
    loc["dm_next"] = full["dm_next"][s0:s1]
    loc["dz_next"] = full["dz_next"][r0:r1]
    loc["mask_row"] = full["msa_mask"][s0:s1]
    loc["mask_col"] = full["msa_mask"][:, r0:r1]
    loc["mask_start"] = full["pair_mask"][r0:r1]
    loc["mask_end"] = full["pair_mask"][:, r0:r1]
    loc = {k: v.contiguous().to(device=device, dtype=(v.dtype if v.dtype == torch.uint8 else dtype))
           for k, v in loc.items()}
    return loc, full
