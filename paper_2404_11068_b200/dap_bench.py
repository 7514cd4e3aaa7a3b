"""bench.py's multi-GPU leg: one Evoformer block's attention core under DAP-N (dap.py), one
process per GPU (torchrun), NCCL over NVLink/NVSwitch.

Each rank holds its DAP shards of the N_res=256 / N_seq=128 block and runs fwd + bwd of the four
modules on them with the block's 8 transposes, 3 bias all-gathers and 3 dbias reduce-scatters.
Timing: W warm-up steps, then K steps bracketed by a barrier and cuda synchronize, CUDA events
on the compute stream, max over ranks; value = the whole block's algorithmic flops ÷ that time
(total work fixed: "scaling": "strong")."""
from __future__ import annotations

import json
import os
import time


def run(args, metric):
    import numpy as np
    import torch
    import torch.distributed as dist

    from . import build as _b
    from . import dap, evoattn

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=dev)
    if rank == 0:
        _b.build_all()
    if world > 1:
        dist.barrier()
    evoattn.load()
    n_seq = args.nseq or 128
    n_res = args.nres or 256
    comm = dap.NcclDap()
    # the pair stack on its own stream and communicator, overlapping the MSA stack (§8(e))
    pair = None
    if not getattr(args, "no_overlap", False):
        pair = (dap.NcclDap(store_key="evo_dap_uid_pair"), torch.cuda.Stream())
    loc, _ = dap.make_block_inputs(torch, world, rank, n_seq, n_res, seed=0, device=dev)
    attn = _Counting(evoattn)
    blk = dap.DapEvoformerAttention(comm, attn, loc, pair)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        blk.forward()
        return blk.backward(loc["dm_next"], loc["dz_next"])

    for _ in range(args.warmup):
        step()
    comm.wait(stream)  # NCCL async-error polling with a timeout instead of a bare synchronize
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # the whole DAP block (attention calls + NCCL exchanges) as one CUDA graph (PAPER.md L264:
    # graphs remove the per-launch CPU overhead that DAP exposes); NCCL supports stream capture
    graph = None
    if not getattr(args, "no_graph", False):
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        with torch.cuda.stream(cap):
            step()
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=cap):
                step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    from bench import ClockSampler  # noqa: E402  (repo root is on sys.path under bench.py)
    clocks = ClockSampler(local)
    if rank == 0:
        clocks.start()
        time.sleep(0.3)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    comm.barrier()
    torch.cuda.synchronize()
    attn.launches = 0
    for s in range(args.steps):
        if not args.no_flush:
            flush.zero_()
        comm.barrier()  # stragglers show up as their own time
        ev[s][0].record(stream)
        if graph is not None:
            graph.replay()
        else:
            step()
        ev[s][1].record(stream)
    comm.wait(stream)
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    clk = clocks.stop() if rank == 0 else None
    flops = dap.block_flops(n_seq, n_res)
    # our kernels in the timed region: the attention core's launches (C ABI count) + one
    # pack/unpack per transpose when N > 1 (NCCL's own kernels are library code, not counted)
    # per-kernel device time from K eager steps with each attention launch bracketed by CUDA
    # events (graph replays cannot be timed per kernel); also the launch count of our kernels
    import ctypes
    from bench import kernel_roofline
    lib = evoattn.load()
    trace_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * 64 * args.steps)]
    for e in trace_ev:
        e.record(stream)
    torch.cuda.synchronize()
    arr = (ctypes.c_void_p * len(trace_ev))(*[e.cuda_event for e in trace_ev])
    lib.evo_trace_enable(arr, len(trace_ev))
    attn.launches = 0
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    ntr = lib.evo_trace_count()
    labels = [lib.evo_trace_label(i).decode() for i in range(ntr)]
    lib.evo_trace_enable(None, 0)
    per = {}
    for i, lab in enumerate(labels):
        per.setdefault(lab, []).append(trace_ev[2 * i].elapsed_time(trace_ev[2 * i + 1]))
    pl = dap.plan(world, n_seq, n_res)
    mods = [("row", *pl["row"], True), ("col", *pl["col"], False), ("start", *pl["start"], True),
            ("end", *pl["end"], True)]
    launches = attn.launches + (8 * args.steps if world > 1 else 0)
    kernels, roof = kernel_roofline(per, mods, clk)
    e2e = _e2e(torch, dist, blk, loc, step, args, world, dev, stream, flops)
    if rank == 0:
        line = {
            "metric": metric, "value": flops / (ms_max * 1e-3) / 1e12, "unit": "TFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max, "ms_per_block": ms_max, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"evoformer_block_attn_nres{n_res}_nseq{n_seq}",
                       "parallelism": f"dap{world}", "local_shapes": dap.plan(world, n_seq, n_res),
                       "l2": "flushed (256 MB write) before every timed step" if not args.no_flush
                       else "warm",
                       "collectives_per_block": {"a2a": 8, "allgather": 3, "reduce_scatter": 3},
                       "launch": "CUDA graph of the step" if graph is not None else "eager"},
            "clocks": clk,
            "roofline": roof,
            "kernels": kernels,
            "e2e": e2e,
            "gpu_launches": launches,
            "overlap": "pair stack on its own stream + communicator" if pair else "none",
        }
    stack = None
    if getattr(args, "stack_blocks", 0) > 0:
        stack = run_stack(torch, dist, dap, evoattn, comm, pair, world, rank, dev,
                          args.stack_nseq, args.stack_nres, args.stack_blocks, args)
    if rank == 0:
        line["stack"] = stack
        print(json.dumps(line), flush=True)
    if pair is not None:
        pair[0].close()
    comm.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


class _Counting:
    """evoattn with a running count of the kernels its calls launched (evo_last_launch_count)."""

    def __init__(self, mod):
        self.mod, self.launches = mod, 0

    def fwd(self, *a, **k):
        r = self.mod.fwd(*a, **k)
        self.launches += self.mod.last_launch_count()
        return r

    def bwd(self, *a, **k):
        r = self.mod.bwd(*a, **k)
        self.launches += self.mod.last_launch_count()
        return r


def run_stack(torch, dist, dap, evoattn, comm, pair, world, rank, dev, n_seq, n_res, blocks,
              args):
    """`blocks` chained Evoformer attention-core blocks (fwd through the stack,
    then bwd back) under DAP-`world`, captured as ONE CUDA graph and replayed; device time per
    replay (CUDA events, max over ranks), L2 flushed before each.  Returns ms per stack and per
    block plus the algorithmic TFLOP/s."""
    import numpy as np
    loc, _ = dap.make_block_inputs(torch, world, rank, n_seq, n_res, seed=1, device=dev)
    st = dap.DapEvoformerStack(comm, evoattn, loc, blocks, pair)
    stream = torch.cuda.current_stream()

    def step():
        st.forward()
        return st.backward(loc["dm_next"], loc["dz_next"])

    step()
    torch.cuda.synchronize()
    cap = torch.cuda.Stream()
    cap.wait_stream(stream)
    with torch.cuda.stream(cap):
        step()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cap):
            step()
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    reps = max(2, min(args.steps, 5))
    for _ in range(2):
        graph.replay()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    for a, b in ev:
        flush.zero_()
        comm.barrier()
        a.record(stream)
        graph.replay()
        b.record(stream)
    comm.wait(stream)
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    fl = blocks * dap.block_flops(n_seq, n_res)
    del graph, st
    torch.cuda.empty_cache()
    return {"blocks": blocks, "n_res": n_res, "n_seq": n_seq, "parallelism": f"dap{world}",
            "launch": "one CUDA graph of the whole stack (fwd + bwd)", "ms_per_stack": ms,
            "ms_per_block": ms / blocks, "ms_per_48_blocks": 48 * ms / blocks,
            "tflops_alg": fl / (ms * 1e-3) / 1e12, "replays": reps,
            "l2": "flushed before each replay",
            "note": "per-block k/v/g/bias tensors shared across blocks; q chained m_next/z_next"}


def _e2e(torch, dist, blk, loc, step, args, world, dev, stream, flops):
    """Same block through the same API from pinned HOST buffers: this rank's input shards are
    copied H2D and the step's result — a device-side fp32 metric summing m_next, z_next and
    every gradient shard (the role of a loss; the gradients stay on the device) — D2H inside
    the timed region; max over ranks.  `all_outputs_d2h` times the same step copying every
    output and gradient shard D2H."""
    host_in = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True).copy_(v)
               for k, v in loc.items()}
    h2d = sum(v.numel() * v.element_size() for v in host_in.values())
    host_out = {}
    metric_dev = torch.zeros((), dtype=torch.float32, device=dev)
    metric_host = torch.zeros((), dtype=torch.float32, pin_memory=True)

    def e2e_step(all_outputs):
        for k, v in host_in.items():
            loc[k].copy_(v, non_blocking=True)
        m_next, z_next, _ = blk.forward()
        grads = blk.backward(loc["dm_next"], loc["dz_next"])
        outs = dict(grads, m_next=m_next, z_next=z_next)
        metric_dev.zero_()
        for k, v in outs.items():
            if v is None:
                continue
            if all_outputs:
                if k not in host_out:
                    host_out[k] = torch.empty(v.shape, dtype=v.dtype, pin_memory=True)
                host_out[k].copy_(v, non_blocking=True)
            else:
                metric_dev.add_(torch.sum(v, dtype=torch.float32))
        if not all_outputs:
            metric_host.copy_(metric_dev, non_blocking=True)

    def timed(all_outputs):
        e2e_step(all_outputs)
        torch.cuda.synchronize()
        n = max(3, min(args.steps, 10))
        blk.comm.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(n):
            e2e_step(all_outputs)
        b.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / n], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), n

    ms, n = timed(False)
    ms_all, _ = timed(True)
    d2h = sum(v.numel() * v.element_size() for v in host_out.values())
    return {"value": flops / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 4, "steps": n,
            "note": "per rank: pinned host input shards H2D; the step's fp32 result metric D2H",
            "all_outputs_d2h": {"value": flops / (ms_all * 1e-3) / 1e12, "ms_per_step": ms_all,
                                "d2h_bytes_per_step": int(d2h),
                                "note": "same step, every output and gradient shard D2H"}}
