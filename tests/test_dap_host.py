"""DAP host logic on CPU (no GPU): world_size-2 `gloo` processes run the block's DAP data flow
(paper_2404_11068_b200/dap.py) with the collectives done by torch.distributed/gloo and the
attention by the fp64 oracle, and every rank's shard of every output and gradient is compared
with an UNSHARDED reference written out here directly from the module definitions (AF2 Alg.
7/8/13/14 index conventions).  This pins the shard plan, the transpose
directions, the bias all-gather / dbias reduce-scatter layouts and the mask slicing; the NCCL
library itself is covered by the GPU tests (tests/test_gpu_dap.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2404_11068_b200 import dap

SHAPE = dict(n_seq=8, n_res=12, heads_m=2, heads_z=2, head_dim=8)


# ----------------------------------------------------------------------------- test shims
class GlooComm:
    """The three DAP exchanges with plain torch.distributed collectives (reference semantics
    of include/evo_dap.h: row shard [A/n, Bd, ...] <-> column shard [A, Bd/n, ...])."""

    def __init__(self):
        self.n, self.rank = dist.get_world_size(), dist.get_rank()

    def _gather(self, t):
        parts = [torch.empty_like(t) for _ in range(self.n)]
        dist.all_gather(parts, t.contiguous())
        return parts

    def transpose(self, src, direction):
        parts = self._gather(src)
        if direction == 0:  # rows -> columns
            full = torch.cat(parts, 0)
            w = full.shape[1] // self.n
            return full[:, self.rank * w:(self.rank + 1) * w].contiguous()
        full = torch.cat(parts, 1)
        h = full.shape[0] // self.n
        return full[self.rank * h:(self.rank + 1) * h].contiguous()

    def allgather(self, src):
        return torch.cat(self._gather(src), 0)

    def reduce_scatter(self, src):
        t = src.clone()
        dist.all_reduce(t)
        h = t.shape[0] // self.n
        return t[self.rank * h:(self.rank + 1) * h].contiguous()


class PackA2AComm(GlooComm):
    """The transpose exactly as libevodap performs it (csrc/evo_dap.cu,
    evo_dap_alltoall_transpose): dir 0 packs the row shard [A/n][Bd][C] into [n][A/n][Bd/n·C]
    (swap01 of [A/n][n][W] with W = Bd/n·C, the evo_dap_pack formula), one all-to-all of
    equal contiguous blocks, and the received buffer IS the column shard [A][Bd/n][C] (no
    unpack); dir 1 sends the column shard's contiguous row blocks as they are and unpacks
    [n][A/n][W] -> [A/n][n][W].  Byte-level layout checked against GlooComm's gather/slice
    semantics by running the whole block with it."""

    @staticmethod
    def _swap01(x, X, Y):  # [X][Y][W] -> [Y][X][W]: the evo_dap_pack kernel's mapping
        return x.reshape(X, Y, -1).permute(1, 0, 2).contiguous()

    def transpose(self, src, direction):
        n = self.n
        src = src.contiguous()
        rest = tuple(src.shape[2:])
        if direction == 0:
            A_loc, Bd = src.shape[0], src.shape[1]
            send = self._swap01(src, A_loc, n).reshape(-1)          # [n][A/n][W]
            recv = torch.empty_like(send)
            dist.all_to_all_single(recv, send)
            return recv.reshape((A_loc * n, Bd // n) + rest)       # [A][Bd/n][C], no unpack
        A, W_loc = src.shape[0], src.shape[1]
        send = src.reshape(-1)                                     # row blocks j·A/n.. -> rank j
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send)
        return self._swap01(recv, n, A // n).reshape((A // n, W_loc * n) + rest)


class OracleAttn:
    """The attention core's fwd/bwd signature on top of the fp64 oracle; outputs take the
    strides of the matching input, as the C ABI does."""

    @staticmethod
    def _like(t, arr):
        out = torch.empty_strided(tuple(t.shape), tuple(t.stride()), dtype=torch.float64)
        out.copy_(torch.from_numpy(np.asarray(arr)))
        return out

    def fwd(self, q, k, v, bias, mask, g):
        o, lse = oracle.attn_fwd(q.numpy(), k.numpy(), v.numpy(),
                                 None if bias is None else bias.numpy(),
                                 None if mask is None else mask.numpy(),
                                 None if g is None else g.numpy())
        return self._like(q, o), torch.from_numpy(lse)

    def bwd(self, q, k, v, o, lse, dout, bias=None, mask=None, g=None, workspace=None):
        r = oracle.attn_bwd(q.numpy(), k.numpy(), v.numpy(), dout.numpy(),
                            None if bias is None else bias.numpy(),
                            None if mask is None else mask.numpy(),
                            None if g is None else g.numpy())
        return {"dq": self._like(q, r["dq"]), "dk": self._like(k, r["dk"]),
                "dv": self._like(v, r["dv"]),
                "dg": None if g is None else self._like(g, r["dg"]),
                "dbias": None if bias is None else self._like(bias, r["dbias"])}


# ----------------------------------------------------------------------------- reference
def unsharded_reference(full):
    """The block on full tensors, written from the module definitions (no dap.py/modules.py):
    row: batch s, attend r, bias b[h,q=r1,k=r2] = E_row[r1,h,r2];  col: batch r, attend s;
    start: batch i, attend j, bias E_start[j,h,k];  end: batch j, attend i, bias b_ki =
    E_end[k,h,i]; masks msa_mask[s,r], pair_mask[i,j]."""
    f = {k: v.double().numpy() for k, v in full.items()}
    bhld = lambda x: x.transpose(0, 2, 1, 3)       # [A0,A1,H,D] -> [A0,H,A1,D]
    bhld_t = lambda x: x.transpose(1, 2, 0, 3)     # [A0,A1,H,D] -> [A1,H,A0,D]
    from_bhld = lambda y: y.transpose(0, 2, 1, 3)
    from_bhld_t = lambda y: y.transpose(2, 0, 1, 3)
    mm, pm = f["msa_mask"], f["pair_mask"]
    out = {}
    # forward
    o_row, _ = oracle.attn_fwd(bhld(f["row_q"]), bhld(f["row_k"]), bhld(f["row_v"]),
                               f["E_row"].transpose(1, 0, 2), mm, bhld(f["row_g"]))
    o_row_s = from_bhld(o_row)                                   # [S,R,H,D]
    o_col, _ = oracle.attn_fwd(bhld_t(o_row_s), bhld_t(f["col_k"]), bhld_t(f["col_v"]), None,
                               mm.T, bhld_t(f["col_g"]))
    o_col_s = from_bhld_t(o_col)
    o_st, _ = oracle.attn_fwd(bhld(f["st_q"]), bhld(f["st_k"]), bhld(f["st_v"]),
                              f["E_start"].transpose(1, 0, 2), pm, bhld(f["st_g"]))
    o_st_s = from_bhld(o_st)
    b_end = f["E_end"].transpose(1, 2, 0)                        # [h, q=i, k] = E_end[k,h,i]
    o_end, _ = oracle.attn_fwd(bhld_t(o_st_s), bhld_t(f["end_k"]), bhld_t(f["end_v"]), b_end,
                               pm.T, bhld_t(f["end_g"]))
    o_end_s = from_bhld_t(o_end)
    out.update(o_row=o_row_s, o_col=o_col_s, o_start=o_st_s, o_end=o_end_s)
    S, R, Hm, D = o_row_s.shape
    I, J, Hz, _ = o_st_s.shape
    # backward
    dz = f["dz_next"].reshape(I, J, Hz, D)
    r = oracle.attn_bwd(bhld_t(o_st_s), bhld_t(f["end_k"]), bhld_t(f["end_v"]), bhld_t(dz),
                        b_end, pm.T, bhld_t(f["end_g"]))
    out.update(end_k=from_bhld_t(r["dk"]), end_v=from_bhld_t(r["dv"]), end_g=from_bhld_t(r["dg"]),
               E_end=r["dbias"].transpose(2, 0, 1))
    d_st = from_bhld_t(r["dq"])
    r = oracle.attn_bwd(bhld(f["st_q"]), bhld(f["st_k"]), bhld(f["st_v"]), bhld(d_st),
                        f["E_start"].transpose(1, 0, 2), pm, bhld(f["st_g"]))
    out.update(st_q=from_bhld(r["dq"]), st_k=from_bhld(r["dk"]), st_v=from_bhld(r["dv"]),
               st_g=from_bhld(r["dg"]), E_start=r["dbias"].transpose(1, 0, 2))
    dm = f["dm_next"].reshape(S, R, Hm, D)
    r = oracle.attn_bwd(bhld_t(o_row_s), bhld_t(f["col_k"]), bhld_t(f["col_v"]), bhld_t(dm),
                        None, mm.T, bhld_t(f["col_g"]))
    out.update(col_k=from_bhld_t(r["dk"]), col_v=from_bhld_t(r["dv"]), col_g=from_bhld_t(r["dg"]))
    d_row = from_bhld_t(r["dq"])
    r = oracle.attn_bwd(bhld(f["row_q"]), bhld(f["row_k"]), bhld(f["row_v"]), bhld(d_row),
                        f["E_row"].transpose(1, 0, 2), mm, bhld(f["row_g"]))
    out.update(row_q=from_bhld(r["dq"]), row_k=from_bhld(r["dk"]), row_v=from_bhld(r["dv"]),
               row_g=from_bhld(r["dg"]), E_row=r["dbias"].transpose(1, 0, 2))
    out["m_next"] = o_col_s.reshape(S, R, Hm * D)
    out["z_next"] = o_end_s.reshape(I, J, Hz * D)
    return out


# which axis of each full reference tensor is this rank's shard: (axis, extent key)
SHARD_AXIS = {
    "o_row": (0, "S"), "o_col": (1, "R"), "o_start": (0, "R"), "o_end": (1, "R"),
    "m_next": (0, "S"), "z_next": (0, "R"),
    "row_q": (0, "S"), "row_k": (0, "S"), "row_v": (0, "S"), "row_g": (0, "S"),
    "col_k": (1, "R"), "col_v": (1, "R"), "col_g": (1, "R"),
    "st_q": (0, "R"), "st_k": (0, "R"), "st_v": (0, "R"), "st_g": (0, "R"),
    "end_k": (1, "R"), "end_v": (1, "R"), "end_g": (1, "R"),
    "E_row": (0, "R"), "E_start": (0, "R"), "E_end": (0, "R"),
}


def _local_slice(ref, name, n, rank):
    axis, ext = SHARD_AXIS[name]
    size = ref.shape[axis] // n
    sl = [slice(None)] * ref.ndim
    sl[axis] = slice(rank * size, (rank + 1) * size)
    return ref[tuple(sl)]


def _compare(got, ref, name):
    got = got.double().numpy() if isinstance(got, torch.Tensor) else got
    err = np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-300)
    assert err < 1e-12, f"{name}: rel err {err:.3e}"


def _worker(rank, n, port, mask, q, comm_cls=GlooComm):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=n)
        oracle.set_num_threads(1)
        loc, full = dap.make_block_inputs(torch, n, rank, **SHAPE, seed=7, dtype=torch.float64,
                                          mask=mask)
        blk = dap.DapEvoformerAttention(comm_cls(), OracleAttn(), loc)
        m_next, z_next, outs = blk.forward()
        grads = blk.backward(loc["dm_next"], loc["dz_next"])
        ref = unsharded_reference(full)
        got = dict(outs, m_next=m_next, z_next=z_next, **grads)
        for name in SHARD_AXIS:
            _compare(got[name], _local_slice(ref[name], name, n, rank), name)
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # surface the failure in the parent
        import traceback
        q.put((rank, traceback.format_exc()))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n,mask,comm", [(1, "ones", "gather"), (2, "ones", "gather"),
                                         (2, "prefix", "gather"), (4, "prefix", "gather"),
                                         (2, "prefix", "pack_a2a"), (4, "prefix", "pack_a2a")])
def test_dap_block_matches_unsharded(n, mask, comm):
    """comm = "gather": the exchanges' reference semantics; "pack_a2a": the transposes as
    libevodap lays them out (pack formula + one equal-block all-to-all, PackA2AComm)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    cls = GlooComm if comm == "gather" else PackA2AComm
    procs = [ctx.Process(target=_worker, args=(r, n, port, mask, q, cls)) for r in range(n)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(n))
    for p in procs:
        p.join(timeout=60)
    for r in range(n):
        assert res[r] == "ok", f"rank {r}:\n{res[r]}"


def test_plan_and_flops():
    p = dap.plan(8, 128, 256)
    assert p == {"row": (16, 8, 256), "col": (32, 8, 128), "start": (32, 4, 256),
                 "end": (32, 4, 256)}
    with pytest.raises(ValueError):
        dap.plan(3, 128, 256)
    # 12·B·H·L²·D summed over the block (90.2 GFLOP at N_res=256, N_seq=128)
    assert abs(dap.block_flops(128, 256) - 90.19e9) / 90.19e9 < 1e-3
    assert dap.shard(4, 3, 256, "x") == (192, 256)


def test_transpose_semantics_single_process():
    """GlooComm-free check of the pack layout (dir 0 then dir 1 is the identity, and dir 0's
    output block j holds column block j) using the formula of include/evo_dap.h."""
    n, A_loc, Bd, C = 4, 3, 8, 5
    src = torch.arange(A_loc * Bd * C, dtype=torch.float64).reshape(A_loc, Bd, C)
    W = Bd // n
    packed = src.reshape(A_loc, n, W, C).permute(1, 0, 2, 3)  # evo_dap_pack dir 0
    for j in range(n):
        assert torch.equal(packed[j], src[:, j * W:(j + 1) * W])
    back = packed.permute(1, 0, 2, 3).reshape(A_loc, Bd, C)  # evo_dap_pack dir 1
    assert torch.equal(back, src)
