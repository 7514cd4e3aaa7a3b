"""DAP on the GPU (one B200): the pack/unpack kernel of the all-to-all transpose bit-exact
against the layout formula of include/evo_dap.h for n = 1..8, the NCCL communicator at
world size 1, and the whole block's DAP data flow through the C ABIs against the fp64 oracle's
unsharded block (tests/test_dap_host.py::unsharded_reference)."""
import pytest
import torch

from paper_2404_11068_b200 import dap, evoattn

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("direction", [0, 1])
@pytest.mark.parametrize("A_loc,W,C_bytes", [(3, 2, 16), (16, 4, 512), (32, 16, 256), (1, 1, 48)])
def test_pack_kernel_bit_exact(n, direction, A_loc, W, C_bytes):
    Bd = W * n
    g = torch.Generator(device="cpu").manual_seed(n * 100 + A_loc)
    src = torch.randint(0, 256, (A_loc * Bd * C_bytes,), generator=g, dtype=torch.uint8).cuda()
    dst = torch.full_like(src, 0xAB)
    dap.pack(src, dst, n, A_loc, Bd, C_bytes, direction)
    torch.cuda.synchronize()
    if direction == 0:  # [A_loc][n][W·C] -> [n][A_loc][W·C]
        ref = src.view(A_loc, n, W * C_bytes).permute(1, 0, 2).reshape(-1)
    else:               # [n][A_loc][W·C] -> [A_loc][n][W·C]
        ref = src.view(n, A_loc, W * C_bytes).permute(1, 0, 2).reshape(-1)
    assert torch.equal(dst, ref)


def test_pack_validation():
    x = torch.zeros(64, dtype=torch.uint8, device="cuda")
    with pytest.raises(evoattn.EvoError, match="EVO_E_ALIGN"):
        dap.pack(x, x.clone(), 2, 1, 2, 8, 0)          # C_bytes not a multiple of 16
    with pytest.raises(evoattn.EvoError, match="EVO_E_SHAPE"):
        dap.pack(x, x.clone(), 2, 1, 3, 16, 0)         # Bd not divisible by n


def test_nccl_world1_collectives():
    comm = dap.NcclDap()
    assert comm.n == 1 and comm.rank == 0
    x = torch.randn(6, 4, 8, device="cuda").to(torch.bfloat16)
    assert torch.equal(comm.transpose(x, 0), x)
    assert torch.equal(comm.transpose(x, 1), x)
    assert torch.equal(comm.allgather(x), x)
    f = torch.randn(5, 3, 4, device="cuda")
    assert torch.equal(comm.reduce_scatter(f), f)
    comm.barrier()
    torch.cuda.synchronize()
    comm.close()


def test_dap_block_world1_matches_oracle():
    from test_dap_host import unsharded_reference, SHARD_AXIS
    shape = dict(n_seq=32, n_res=64, heads_m=8, heads_z=4, head_dim=32)
    loc, full = dap.make_block_inputs(torch, 1, 0, **shape, seed=3, device="cuda",
                                      mask="prefix")
    comm = dap.NcclDap()
    blk = dap.DapEvoformerAttention(comm, evoattn, loc)
    m_next, z_next, outs = blk.forward()
    grads = blk.backward(loc["dm_next"], loc["dz_next"])
    torch.cuda.synchronize()
    ref = unsharded_reference(full)
    got = dict(outs, m_next=m_next, z_next=z_next, **grads)
    for name in SHARD_AXIS:
        a = got[name].double().cpu()
        r = torch.from_numpy(ref[name].copy())
        # normwise max relative error, the parity norm of every other GPU test (R9)
        err = float((a - r).abs().max() / max(float(r.abs().max()), 1e-30))
        assert err < 2e-2, f"{name}: {err:.3e}"
    comm.close()


def test_dap_block_overlap_is_bitwise_identical():
    """The pair stack on its own stream + communicator (overlapping the MSA stack) changes no
    output bit of the block's forward or backward (same kernels, same inputs, §5b orders)."""
    shape = dict(n_seq=32, n_res=64, heads_m=8, heads_z=4, head_dim=32)
    loc, _ = dap.make_block_inputs(torch, 1, 0, **shape, seed=4, device="cuda", mask="prefix")
    comm = dap.NcclDap()
    comm2 = dap.NcclDap(store_key="evo_dap_uid_pair")
    outs = []
    for pair in (None, (comm2, torch.cuda.Stream())):
        blk = dap.DapEvoformerAttention(comm, evoattn, dict(loc), pair)
        m_next, z_next, _ = blk.forward()
        g = blk.backward(loc["dm_next"], loc["dz_next"])
        comm.wait(torch.cuda.current_stream())
        torch.cuda.synchronize()
        outs.append(dict(g, m_next=m_next, z_next=z_next))
    for k, v in outs[0].items():
        if v is not None:
            assert torch.equal(v, outs[1][k]), k
    comm2.close()
    comm.close()


def test_dap_stack_chains_blocks():
    """DapEvoformerStack: block 2's queries are block 1's outputs (m_next, z_next), and the
    backward chains dm/dz back — checked against two explicitly chained blocks."""
    shape = dict(n_seq=16, n_res=32, heads_m=8, heads_z=4, head_dim=32)
    loc, _ = dap.make_block_inputs(torch, 1, 0, **shape, seed=5, device="cuda")
    comm = dap.NcclDap()
    st = dap.DapEvoformerStack(comm, evoattn, loc, 2, None)
    m, z = st.forward()
    dm, dz, _ = st.backward(loc["dm_next"], loc["dz_next"])
    b1 = dap.DapEvoformerAttention(comm, evoattn, dict(loc))
    m1, z1, _ = b1.forward()
    x2 = dict(loc, row_q=m1.view(loc["row_q"].shape), st_q=z1.view(loc["st_q"].shape))
    b2 = dap.DapEvoformerAttention(comm, evoattn, x2)
    m2, z2, _ = b2.forward()
    g2 = b2.backward(loc["dm_next"], loc["dz_next"])
    g1 = b1.backward(g2["row_q"].reshape(m1.shape), g2["st_q"].reshape(z1.shape))
    torch.cuda.synchronize()
    assert torch.equal(m, m2) and torch.equal(z, z2)
    assert torch.equal(dm, g1["row_q"].reshape(dm.shape))
    assert torch.equal(dz, g1["st_q"].reshape(dz.shape))
    comm.close()
