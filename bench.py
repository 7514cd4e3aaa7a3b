#!/usr/bin/env python
"""Benchmark: Evoformer gated pair-bias attention, fwd+bwd, one Evoformer block at N_res=256.

BASELINE.json metric: "Evoformer attn fwd+bwd TFLOP/s & ms/block at N_res=256 (1/2/4/8 B200,
% peak)".  One step = the four attention modules of one Evoformer block (row,
column, triangle start, triangle end), each forward + backward through the C ABI, on seeded
synthetic tensors shaped like OpenFold/MLPerf initial training (N_res=256, N_seq=128,
8/4 heads of 32; BASELINE.json configs 2-3 + the block's MSA column attention):

  row    B=N_seq=128  H=8 L=N_res=256 D=32  shared bias b_ij   (msa_mask rows)
  col    B=N_res=256  H=8 L=N_seq=128 D=32  no bias            (msa_mask columns, strided view)
  start  B=N_res=256  H=4 L=N_res=256 D=32  shared bias b_jk   (pair_mask rows)
  end    B=N_res=256  H=4 L=N_res=256 D=32  bias b_ki (q-contiguous view), strided q/k/v/mask

value = algorithmic TFLOP/s = Σ 12·B·H·L²·D over the four calls ÷ device time per step
(the bwd recompute of S is not credited).  Projections / LayerNorm are outside the
attention core and excluded.  Under torchrun (N > 1) the block runs under Dynamic Axial
Parallelism (paper_2404_11068_b200/dap.py): rank r holds N_seq/N MSA rows and N_res/N pair rows,
NCCL all-to-all transposes between row and column phases, bias all-gather / dbias
reduce-scatter; value = whole-job TFLOP/s with max-over-ranks device time ("scaling": "strong").

`--impl reference` times the fp64 CPU oracle (the only reference that exists: the paper ships no
code) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "Evoformer attn fwd+bwd TFLOP/s & ms/block at N_res=256 (1/2/4/8 B200, % peak)"
N_RES, N_SEQ, C_HEAD = 256, 128, 32
MODULES = [  # name, B, H, L, bias
    ("row", N_SEQ, 8, N_RES, True),
    ("col", N_RES, 8, N_SEQ, False),
    ("start", N_RES, 4, N_RES, True),
    ("end", N_RES, 4, N_RES, True),
]


def alg_flops(B, H, L, D):
    return 12.0 * B * H * L * L * D


def kernel_alg(name, B, H, L, D, bias):
    """Algorithmic work of one launch of kernel `name` on a (B,H,L,L,D) call:
    returns (flops, bytes, exps)."""
    X = B * H * L * D  # elements of one [B,H,L,D] tensor
    P = B * H * L * L  # score elements
    bb = 2 * H * L * L if bias else 0
    if name == "fwd_bf16":  # q,k,v,g in, o out (bf16); bias; mask; lse out
        return 4.0 * P * D, 10.0 * X + bb + B * L + 4 * B * H * L, float(P)
    if name == "bwd_pre":  # o, dO, g in; dA, dg out (bf16); lse in; D, lse2 out (fp32)
        return 0.0, 10.0 * X + 12.0 * B * H * L, 0.0
    if name == "bwd_main":  # q,k,v,dA in; dq,dk,dv out; lse2/D in; bias; mask
        return 8.0 * P * D, 14.0 * X + 8.0 * B * H * L + bb + B * L, float(P)
    if name == "bwd_bias":  # dbias (fp32) written once; inputs already counted in bwd_main
        return 0.0, 2.0 * bb, float(P)
    if name == "bwd_fused":  # q,k,v,dA + lse2/D + bias + mask in; dq,dk,dv (bf16) + dbias out
        return 8.0 * P * D, 14.0 * X + 8.0 * B * H * L + 3.0 * bb + B * L, float(P)
    if name in ("dq_convert",):
        return 0.0, 6.0 * X, 0.0
    if name == "dbias_reduce":
        return 0.0, 2.0 * bb, 0.0
    return 0.0, 0.0, 0.0


def kernel_roofline(per, modules, clk):
    """Per-kernel table and the dominant kernel's roofline object from per-launch device times
    (ms, lists keyed by the C ABI trace label) and the calls' shapes [(name, B, H, L, bias)]:
    achieved = algorithmic work per launch (kernel_alg, averaged over the modules) ÷ the mean
    launch time; peak = MEASURED_PEAKS.json; MUFU peak = 148 SMs x 16 ex2/clk x the SM clock
    sampled under load."""
    calls = []
    for name, B, H, L, bias in modules:
        calls.append(("fwd_bf16", B, H, L, bias))
        calls += [("bwd_pre", B, H, L, bias), ("bwd_fused", B, H, L, bias)]
        if L > 128:
            calls.append(("dq_convert", B, H, L, bias))
        if bias:
            calls.append(("dbias_reduce", B, H, L, bias))
    work = {}
    for kname, B, H, L, bias in calls:
        f, by, ex = kernel_alg(kname, B, H, L, C_HEAD, bias)
        w = work.setdefault(kname, [0.0, 0.0, 0.0, 0])
        w[0] += f; w[1] += by; w[2] += ex; w[3] += 1
    tot_traced = sum(sum(v) for v in per.values())
    kernels = {}
    for k, v in per.items():
        n = len(v)
        w = work.get(k, [0, 0, 0, 1])
        per_launch_ms = sum(v) / n
        f, by, ex = w[0] / w[3], w[1] / w[3], w[2] / w[3]
        kernels[k] = {"launches": n, "ms_per_launch": per_launch_ms,
                      "share": sum(v) / tot_traced,
                      "tflops": f / (per_launch_ms * 1e-3) / 1e12,
                      "gbs": by / (per_launch_ms * 1e-3) / 1e9,
                      "gexps": ex / (per_launch_ms * 1e-3) / 1e9}
    dom = max(kernels, key=lambda k: kernels[k]["share"])
    pk = measured_peaks()
    sm_mhz = (clk or {}).get("sm_mhz") or pk["sm_max_mhz"]
    mufu_peak = 148 * 16 * sm_mhz * 1e6 / 1e9  # Gex2/s (16 ex2/clk/SM)
    dk = kernels[dom]
    fr_t = dk["tflops"] / pk["bf16_tflops"]
    fr_h = dk["gbs"] / pk["hbm_gbs"]
    fr_x = dk["gexps"] / mufu_peak
    if fr_x >= max(fr_t, fr_h):
        roof = {"bound": "alu", "achieved": dk["gexps"], "peak": mufu_peak, "unit": "Gexp2/s",
                "frac": fr_x}
    elif fr_h >= fr_t:
        roof = {"bound": "hbm", "achieved": dk["gbs"], "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": fr_h}
    else:
        roof = {"bound": "tensor", "achieved": dk["tflops"], "peak": pk["bf16_tflops"],
                "unit": "TFLOP/s", "frac": fr_t}
    roof.update({"kernel": dom, "traffic": load_traffic(dom), "peak_source": pk["source"],
                 "fracs": {"tensor": fr_t, "hbm": fr_h, "mufu": fr_x},
                 "mufu_peak_note": f"148 SM x 16 ex2/clk x {sm_mhz:.0f} MHz (median SM clock "
                                   "under load)"})
    return kernels, roof


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-i", str(self.index), "-lms", "100"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sms.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        busy = [s for s in sms if mx and s > 0.3 * mx] or sms
        return {"sm_mhz": float(np.median(busy)) if busy else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sms)}


# ----------------------------------------------------------------------------- peaks
def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "sm_max_mhz": d.get("sm_max_mhz", 1965.0), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "sm_max_mhz": 1965.0, "source": "fallback"}


# ----------------------------------------------------------------------------- workload
def make_module_inputs(torch, dev, name, B, H, L, bias, seed):
    """Seeded synthetic inputs in the projection storage layouts of DESIGN.md §4."""
    from synth.gen import round_bf16  # noqa: F401  (same recipe as the parity tests)
    g = torch.Generator(device="cpu").manual_seed(seed)
    D = C_HEAD
    if name in ("row", "start"):  # storage [B, L, H, D] (m[s,r] / z[i,j] projections)
        shape, perm = (B, L, H, D), (0, 2, 1, 3)
    else:  # col / end: batch axis is the 2nd storage axis: storage [L, B, H, D]
        shape, perm = (L, B, H, D), (1, 2, 0, 3)
    t = {}
    for n in ("q", "k", "v", "g", "dout"):
        t[n] = torch.randn(shape, generator=g).to(dev, torch.bfloat16).permute(*perm)
    t["bias"] = None
    if bias:
        bt = torch.randn((H, L, L), generator=g).to(dev, torch.bfloat16)
        t["bias"] = bt.transpose(1, 2) if name == "end" else bt  # b_ki: q-contiguous view
    m = torch.ones((B, L), dtype=torch.uint8)
    t["mask"] = m.t().contiguous().to(dev).t() if name in ("col", "end") else m.to(dev)
    return t


def cpu_count():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ----------------------------------------------------------------------------- oracle arm
def oracle_block_sample(batch_rows, seed=0):
    """fp64 oracle fwd+bwd on `batch_rows` batch rows of each of the four modules (all heads).
    Returns (algorithmic flops done, seconds)."""
    import oracle
    from synth.gen import attention_case
    flops, secs = 0.0, 0.0
    for i, (name, B, H, L, bias) in enumerate(MODULES):
        b = min(batch_rows, B)
        c = attention_case(b, H, L, L, C_HEAD, seed=seed + i, bias="shared" if bias else None,
                           gate=True, mask="ones")
        t0 = time.perf_counter()
        oracle.attn_fwd(c["q"], c["k"], c["v"], c["bias"], c["mask"], c["g"], c["scale"])
        oracle.attn_bwd(c["q"], c["k"], c["v"], c["dout"], c["bias"], c["mask"], c["g"],
                        c["scale"])
        secs += time.perf_counter() - t0
        flops += alg_flops(b, H, L, C_HEAD)
    return flops, secs


def cpu_baseline(target_s=12.0):
    import oracle
    rows = 1
    f, s = oracle_block_sample(rows)
    while s < target_s / 2 and rows < 256:  # 256 rows = every batch row of every module
        rows *= 2
        f, s = oracle_block_sample(rows)
    return {"value": f / s / 1e12, "unit": "TFLOP/s", "cores": oracle.num_threads(),
            "kind": "oracle",
            "sample": f"fp64 C oracle (OpenMP), fwd+bwd of {rows} batch row(s) of each of the 4 "
                      f"block modules (all heads, full L), {s:.1f} s; scaled by algorithmic flops",
            "seconds": s}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    rows = args.ref_rows
    times, flops = [], 0.0
    for _ in range(args.warmup):
        oracle_block_sample(rows)
    for s in range(args.steps):
        f, t = oracle_block_sample(rows, seed=s)
        times.append(t)
        flops = f
    tot = sum(times)
    value = flops * len(times) / tot / 1e12
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "evoformer_block_attn_nres256_nseq128_sample",
                   "batch_rows_per_module": rows, "note": "bounded sample: the oracle runs "
                   f"{rows} batch row(s) of each module per step (full block = 128/256 rows)"},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": oracle.num_threads(),
                         "kind": "oracle",
                         "sample": f"{rows} batch row(s) per module per step"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def run_gpu(args):
    import torch
    from paper_2404_11068_b200 import evoattn

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1 or args.dap:
        from paper_2404_11068_b200 import dap_bench
        return dap_bench.run(args, METRIC)

    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    from paper_2404_11068_b200 import build as _b
    _b.build_attn()  # no-op unless a source is newer than the in-tree .so
    lib = evoattn.load()
    stream = torch.cuda.current_stream()
    mods = []
    for i, (name, B, H, L, bias) in enumerate(MODULES):
        t = make_module_inputs(torch, dev, name, B, H, L, bias, seed=100 + i)
        ws = torch.empty(max(1, evoattn.workspace_bytes(t["q"], t["k"], t["v"], t["bias"],
                                                        t["mask"], t["g"])),
                         dtype=torch.uint8, device=dev)
        mods.append((name, B, H, L, bias, t, ws))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    # The block's two attention stacks are independent (MSA: row -> col; pair: start -> end):
    # the pair stack runs on a second stream so its kernels fill the SMs the MSA stack's leave
    # idle (kernel tails, low-occupancy phases) — the same overlap the DAP block uses.
    pair_stream = None if args.no_overlap else torch.cuda.Stream()

    def run_mod(name, B, H, L, bias, t, ws):
        o, lse = evoattn.fwd(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"])
        n = evoattn.last_launch_count()
        evoattn.bwd(t["q"], t["k"], t["v"], o, lse, t["dout"], t["bias"], t["mask"], t["g"],
                    workspace=ws)
        return n + evoattn.last_launch_count()

    def step(overlap=True):
        launches = 0
        if pair_stream is None or not overlap:
            for m in mods:
                launches += run_mod(*m)
            return launches
        main = torch.cuda.current_stream()
        pair_stream.wait_stream(main)
        with torch.cuda.stream(pair_stream):
            for m in mods:
                if m[0] in ("start", "end"):
                    launches += run_mod(*m)
        for m in mods:
            if m[0] in ("row", "col"):
                launches += run_mod(*m)
        main.wait_stream(pair_stream)
        return launches

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # CUDA graph of the whole step (graphs remove the per-launch host overhead);
    # the C-ABI calls are stream-ordered and allocation-free, so they capture as they are
    graph = None
    launches_per_step = 0
    if not args.no_graph:
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        with torch.cuda.stream(cap):
            step()
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=cap):
                launches_per_step = step()
        torch.cuda.synchronize()

    # timed region: K steps, L2 flushed (256 MB write) before each, CUDA events per step
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    launches = 0
    for s in range(args.steps):
        if not args.no_flush:
            flush.zero_()
        ev[s][0].record(stream)
        if graph is not None:
            graph.replay()
            launches += launches_per_step
        else:
            launches += step()
        ev[s][1].record(stream)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ev]
    clk = clocks.stop()

    # per-kernel device time: the same K steps again, eager, each launch bracketed by CUDA
    # events on its stream (events cannot be timed inside a graph replay)
    nk_per_step = 64
    trace_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * nk_per_step * args.steps)]
    for e in trace_ev:  # torch creates events lazily: materialise the handles first
        e.record(stream)
    torch.cuda.synchronize()
    trace_arr = (__import__("ctypes").c_void_p * len(trace_ev))(*[e.cuda_event for e in trace_ev])
    lib.evo_trace_enable(trace_arr, len(trace_ev))
    for s in range(args.steps):  # one stream here: each kernel's own duration, not a share
        if not args.no_flush:
            flush.zero_()
        step(overlap=False)
    torch.cuda.synchronize()
    ntr = lib.evo_trace_count()
    labels = [lib.evo_trace_label(i).decode() for i in range(ntr)]
    lib.evo_trace_enable(None, 0)
    ms_step = float(np.mean(ms))
    flops = sum(alg_flops(B, H, L, C_HEAD) for _, B, H, L, _ in MODULES)
    value = flops / (ms_step * 1e-3) / 1e12

    # per-kernel device time (trace events) and the dominant kernel's roofline
    per = {}
    for i, lab in enumerate(labels):
        per.setdefault(lab, []).append(trace_ev[2 * i].elapsed_time(trace_ev[2 * i + 1]))
    kernels, roof = kernel_roofline(per, [(n, B, H, L, bias) for n, B, H, L, bias in MODULES], clk)

    # e2e: host buffers through the same C ABI, h2d + d2h inside the timed region
    e2e = run_e2e(torch, evoattn, mods, args, dev, stream, flops)

    cpu = cpu_baseline(args.cpu_seconds) if not args.no_cpu else None
    configs = None if args.no_configs else run_configs(
        torch, evoattn, dev, flush, max(3, min(args.steps, 10)), clk.get("sm_mhz"))
    stack = None
    if args.stack_blocks > 0:  # §8(f) f4: a chained stack of DAP blocks under one CUDA graph
        from paper_2404_11068_b200 import dap, dap_bench
        comm = dap.NcclDap()
        pair = None if args.no_overlap else (dap.NcclDap(store_key="evo_dap_uid_pair"),
                                              torch.cuda.Stream())
        stack = dap_bench.run_stack(torch, None, dap, evoattn, comm, pair, 1, 0, dev,
                                    args.stack_nseq, args.stack_nres, args.stack_blocks, args)
        if pair is not None:
            pair[0].close()
        comm.close()
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "ms_per_block": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "evoformer_block_attn_nres256_nseq128",
                   "modules": {m[0]: {"B": m[1], "H": m[2], "L": m[3], "D": C_HEAD,
                                      "bias": m[4]} for m in MODULES},
                   "l2": "flushed (256 MB write) before every timed step" if not args.no_flush
                   else "warm", "parallelism": "single GPU",
                   "launch": "CUDA graph of the step" if graph is not None else "eager",
                   "streams": "MSA stack (row, col) and pair stack (start, end) on two streams"
                   if pair_stream is not None else "one stream",
                   "kernel_timing": "per-launch CUDA events over K further eager steps (one "
                                    "stream)"},
        "pct_of_peak": {"tensor_measured": value / measured_peaks()["bf16_tflops"],
                        "tensor_nominal": value / 2250.0},
        "roofline": roof,
        "kernels": kernels,
        "clocks": clk,
        "e2e": e2e,
        "gpu_launches": launches,
        "cpu_baseline": cpu,
        "configs": configs,
        "stack": stack,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- other configs
# BASELINE.json configs[0], [3], [4] and the §8(f) side paths, timed in the same run so their
# numbers come from the driver's box (not only from builder tools): device time per call with
# CUDA events on the launching stream, L2 flushed before every call, median over `reps`.
# (name, B, H, L, D, bias, storage "bl" [B,L,H,D] | "lb" [L,B,H,D], bias q-contiguous)
CONFIGS = [
    ("cfg1_tri_start_nres32", 32, 2, 32, 16, True, "bl", False),
    ("cfg4_extra_msa_col_nextra1024", 256, 8, 1024, 8, False, "lb", False),
    ("f3_extra_msa_row_nextra1024", 1024, 8, 256, 8, True, "bl", False),
    ("cfg5_row_nres384_nseq512", 512, 8, 384, 32, True, "bl", False),
    ("cfg5_col_nres384_nseq512", 384, 8, 512, 32, False, "lb", False),
    ("cfg5_start_nres384", 384, 4, 384, 32, True, "bl", False),
    ("cfg5_end_nres384", 384, 4, 384, 32, True, "lb", True),
]


def _cfg_inputs(torch, dev, B, H, L, D, bias, st, bt, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    shape, perm = ((B, L, H, D), (0, 2, 1, 3)) if st == "bl" else ((L, B, H, D), (1, 2, 0, 3))
    t = {n: torch.randn(shape, generator=g).to(dev, torch.bfloat16).permute(*perm)
         for n in ("q", "k", "v", "g", "dout")}
    t["bias"] = None
    if bias:
        b = torch.randn((H, L, L), generator=g).to(dev, torch.bfloat16)
        t["bias"] = b.transpose(1, 2) if bt else b
    m = torch.ones((B, L), dtype=torch.uint8)
    t["mask"] = m.t().contiguous().to(dev).t() if st == "lb" else m.to(dev)
    return t


def _timed(torch, fn, flush, reps):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    for a, b in ev:
        flush.zero_()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev]))


def run_configs(torch, evoattn, dev, flush, reps, clk_mhz):
    """One entry per config: fwd / bwd / fwd+bwd ms, algorithmic TFLOP/s and the three roofline
    fractions of the call (tensor = 12·B·H·L²·D flops vs the measured bf16 peak, HBM = the
    algorithmic bytes of DESIGN.md §5 vs the measured copy bandwidth, MUFU = 2·B·H·L² exps vs
    148 x 16 ex2/clk at the sampled clock), with the binding one named."""
    pk = measured_peaks()
    mufu = 148 * 16 * (clk_mhz or pk["sm_max_mhz"]) * 1e6
    out = {}
    for i, (name, B, H, L, D, bias, st, bt) in enumerate(CONFIGS):
        t = _cfg_inputs(torch, dev, B, H, L, D, bias, st, bt, seed=200 + i)
        ws = torch.empty(max(1, evoattn.workspace_bytes(t["q"], t["k"], t["v"], t["bias"],
                                                        t["mask"], t["g"])),
                         dtype=torch.uint8, device=dev)
        f = lambda: evoattn.fwd(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"])
        o, lse = f()
        bw = lambda: evoattn.bwd(t["q"], t["k"], t["v"], o, lse, t["dout"], t["bias"],
                                 t["mask"], t["g"], workspace=ws)
        for _ in range(3):
            f()
            bw()
        torch.cuda.synchronize()
        tf, tb = _timed(torch, f, flush, reps), _timed(torch, bw, flush, reps)
        tfb = _timed(torch, lambda: (f(), bw()), flush, reps)
        X, P = B * H * L * D, B * H * L * L
        bb = 2 * H * L * L if bias else 0
        byt = 30.0 * X + 4.0 * bb + 2 * B * L + 8 * B * H * L  # fwd + bwd bytes
        fl = alg_flops(B, H, L, D)
        fr = {"tensor": fl / (tfb * 1e-3) / 1e12 / pk["bf16_tflops"],
              "hbm": byt / (tfb * 1e-3) / 1e9 / pk["hbm_gbs"],
              "mufu": 2.0 * P / (tfb * 1e-3) / mufu}
        out[name] = {"B": B, "H": H, "L": L, "D": D, "bias": bias, "fwd_ms": tf, "bwd_ms": tb,
                     "fwd_bwd_ms": tfb, "tflops_alg": fl / (tfb * 1e-3) / 1e12,
                     "fracs": fr, "binding": max(fr, key=fr.get)}
        del t, ws, o, lse
    # cfg 5 per block: the four modules at N_res = 384, N_seq = 512
    c5 = [k for k in out if k.startswith("cfg5_")]
    out["cfg5_block_nres384_nseq512"] = {
        "ms_per_block": sum(out[k]["fwd_bwd_ms"] for k in c5),
        "ms_per_48_block_stack": 48 * sum(out[k]["fwd_bwd_ms"] for k in c5),
        "tflops_alg": sum(alg_flops(out[k]["B"], out[k]["H"], out[k]["L"], out[k]["D"])
                          for k in c5) / (sum(out[k]["fwd_bwd_ms"] for k in c5) * 1e-3) / 1e12,
        "note": "sum of the four module calls timed one by one (L2 flushed before each)"}
    out.update(run_side_paths(torch, evoattn, dev, flush, reps, pk))
    return out


def run_side_paths(torch, evoattn, dev, flush, reps, pk):
    """§8(f) side paths at the N_res = 256 block shapes: f1 pair bias (LN(z)·W, fwd + bwd), f2
    LN + stacked q|k|v|g projection, f3 extra-MSA global column attention (fwd + bwd)."""
    out = {}
    L, C = 256, 128
    for H in (4, 8):
        z = torch.randn((L, L, C), device=dev).to(torch.bfloat16)
        gamma, beta = torch.ones(C, device=dev), torch.zeros(C, device=dev)
        W = torch.randn((C, H), device=dev) / C ** 0.5
        dbias = torch.randn((H, L, L), device=dev)
        bias, mean, rstd = evoattn.pair_bias_fwd(z, gamma, beta, W)
        ws = torch.empty(1 << 24, dtype=torch.uint8, device=dev)
        f = lambda: evoattn.pair_bias_fwd(z, gamma, beta, W)
        b = lambda: evoattn.pair_bias_bwd(z, gamma, beta, W, mean, rstd, dbias, workspace=ws)
        for _ in range(3):
            f()
            b()
        tf, tb = _timed(torch, f, flush, reps), _timed(torch, b, flush, reps)
        byf = L * L * C * 2 + H * L * L * 2 + 8 * L * L
        byb = 2 * L * L * C * 2 + H * L * L * 4 + 8 * L * L
        out[f"f1_pair_bias_nres256_cz128_h{H}"] = {
            "fwd_ms": tf, "bwd_ms": tb, "fwd_hbm_frac": byf / (tf * 1e-3) / 1e9 / pk["hbm_gbs"],
            "bwd_hbm_frac": byb / (tb * 1e-3) / 1e9 / pk["hbm_gbs"]}
    for name, rows, C, N in [("msa", 128 * 256, 256, 1024), ("triangle", 256 * 256, 128, 512),
                             ("extra_msa", 1024 * 256, 64, 256)]:
        x = torch.randn((rows, C), device=dev).to(torch.bfloat16)
        g, bt = torch.ones(C, device=dev), torch.zeros(C, device=dev)
        W = (torch.randn((N, C), device=dev) / C ** 0.5).to(torch.bfloat16)
        bb = torch.zeros(N, device=dev)
        o = torch.empty((rows, N), dtype=torch.bfloat16, device=dev)
        f = lambda: evoattn.ln_proj_fwd(x, g, bt, W, bb, out=o)
        for _ in range(3):
            f()
        tf = _timed(torch, f, flush, reps)
        byt = rows * C * 2 + rows * N * 2 + N * C * 2 + rows * 8
        # backward (dgrad + LN backward, wgrad, dγ/dβ/db): reads x, dout, W, mean/rstd; writes
        # dx (bf16), dW (fp32); 2 GEMMs of 2·rows·C·N flops each
        _, mean, rstd = evoattn.ln_proj_fwd(x, g, bt, W, bb)
        dout = torch.randn((rows, N), device=dev).to(torch.bfloat16)
        wsb = torch.empty(1 << 26, dtype=torch.uint8, device=dev)
        fb = lambda: evoattn.ln_proj_bwd(x, g, bt, W, mean, rstd, dout, workspace=wsb)
        for _ in range(3):
            fb()
        tb = _timed(torch, fb, flush, reps)
        byb = rows * C * 2 * 2 + rows * N * 2 + N * C * 2 + N * C * 4 + rows * 8
        out[f"f2_ln_qkvg_proj_{name}_{rows}x{C}to{N}"] = {
            "fwd_ms": tf, "tflops": 2.0 * rows * C * N / (tf * 1e-3) / 1e12,
            "hbm_frac": byt / (tf * 1e-3) / 1e9 / pk["hbm_gbs"],
            "bwd_ms": tb, "bwd_tflops": 4.0 * rows * C * N / (tb * 1e-3) / 1e12,
            "bwd_hbm_frac": byb / (tb * 1e-3) / 1e9 / pk["hbm_gbs"]}
    B, S, H, D = 256, 1024, 8, 8
    gq = torch.randn((S, B, H, D), device=dev).to(torch.bfloat16).transpose(0, 1)
    gg = torch.randn((S, B, H, D), device=dev).to(torch.bfloat16).transpose(0, 1)
    gk = torch.randn((S, B, D), device=dev).to(torch.bfloat16).transpose(0, 1)
    gv = torch.randn((S, B, D), device=dev).to(torch.bfloat16).transpose(0, 1)
    gm = torch.ones((S, B), dtype=torch.uint8, device=dev).t()
    o, lse, qbar = evoattn.global_attn_fwd(gq, gk, gv, gg, gm)
    f = lambda: evoattn.global_attn_fwd(gq, gk, gv, gg, gm)
    b = lambda: evoattn.global_attn_bwd(gq, gk, gv, gg, lse, qbar, o, gm)
    for _ in range(3):
        f()
        b()
    tf, tb = _timed(torch, f, flush, reps), _timed(torch, b, flush, reps)
    byf = (2 * B * S * H * D + 2 * B * S * D) * 2 + B * S * H * D * 2
    byb = (3 * B * S * H * D + 2 * B * S * D) * 2 + (2 * B * S * H * D + 2 * B * S * D) * 2
    out["f3_global_col_attn_nres256_nextra1024"] = {
        "fwd_ms": tf, "bwd_ms": tb, "fwd_hbm_frac": byf / (tf * 1e-3) / 1e9 / pk["hbm_gbs"],
        "bwd_hbm_frac": byb / (tb * 1e-3) / 1e9 / pk["hbm_gbs"]}
    return out


def load_traffic(kernel):
    """dram bytes per launch of `kernel` from the committed ncu capture summary, if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        try:
            v = json.load(open(p)).get(kernel)
            return float(v) if isinstance(v, (int, float)) else None
        except Exception:
            return None
    return None


def run_e2e(torch, evoattn, mods, args, dev, stream, flops):
    """Same metric through the public API from pinned HOST buffers: every step copies all of its
    inputs (q, k, v, g, dO, bias, mask of the four modules) H2D and reads the step's result back
    D2H inside the timed region.  The step's result is a device-side metric of every output
    (Σ over o and the five gradients, fp32 accumulation: the role a loss plays in a training
    step — the gradients themselves stay on the device for the optimizer), 4 bytes per step.
    For comparison `all_outputs_d2h` times the same step copying every output (o, lse, dq, dk,
    dv, dg, dbias) D2H."""
    host = []
    h2d = 0
    for name, B, H, L, bias, t, ws in mods:
        hin = {}
        for n in ("q", "k", "v", "g", "dout", "bias", "mask"):
            x = t[n]
            if x is None:
                continue
            hb = torch.empty_strided(x.shape, x.stride(), dtype=x.dtype, pin_memory=True)
            hb.copy_(x)  # keep the storage layout of the device view
            hin[n] = hb
            h2d += x.numel() * x.element_size()
        hout = {"o": torch.empty_strided(t["q"].shape, t["q"].stride(), dtype=torch.bfloat16,
                                         pin_memory=True),
                "lse": torch.empty((B, H, L), pin_memory=True)}
        for n in ("dq", "dk", "dv", "dg"):
            src = {"dq": "q", "dk": "k", "dv": "v", "dg": "g"}[n]
            hout[n] = torch.empty_strided(t[src].shape, t[src].stride(), dtype=torch.bfloat16,
                                          pin_memory=True)
        if bias:
            hout["dbias"] = torch.empty_strided(t["bias"].shape, t["bias"].stride(),
                                                dtype=torch.float32, pin_memory=True)
        host.append((t, ws, hin, hout))
    d2h_all = sum(hb.numel() * hb.element_size() for _, _, _, ho in host for hb in ho.values())
    metric_dev = torch.zeros((), dtype=torch.float32, device=dev)
    metric_host = torch.zeros((), dtype=torch.float32, pin_memory=True)
    # H2D on its own stream, module by module, so the copy of module i+1's inputs overlaps
    # module i's kernels (the copies are the bound); the copy into a module's device buffers
    # waits for that module's previous-step kernels (event), its kernels wait for the copy
    copy_stream = torch.cuda.Stream()
    copied = [torch.cuda.Event() for _ in host]
    used = [torch.cuda.Event() for _ in host]
    for e in used:
        e.record(stream)

    def step(all_outputs):
        metric_dev.zero_()
        main = torch.cuda.current_stream()
        copy_stream.wait_stream(main)  # a step's copies start after everything before it
        for i, (t, ws, hin, hout) in enumerate(host):
            copy_stream.wait_event(used[i])
            with torch.cuda.stream(copy_stream):
                for n, hb in hin.items():
                    t[n].copy_(hb, non_blocking=True)
            copied[i].record(copy_stream)
        for i, (t, ws, hin, hout) in enumerate(host):
            main.wait_event(copied[i])
            o, lse = evoattn.fwd(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"])
            r = evoattn.bwd(t["q"], t["k"], t["v"], o, lse, t["dout"], t["bias"], t["mask"],
                            t["g"], workspace=ws)
            used[i].record(main)
            outs = {"o": o, "lse": lse, **{n: r[n] for n in ("dq", "dk", "dv", "dg", "dbias")}}
            if all_outputs:
                for n, hb in hout.items():
                    hb.copy_(outs[n], non_blocking=True)
            else:
                for n in ("o", "dq", "dk", "dv", "dg", "dbias"):
                    if outs[n] is not None:
                        metric_dev.add_(torch.sum(outs[n], dtype=torch.float32))
        if not all_outputs:
            metric_host.copy_(metric_dev, non_blocking=True)

    def timed(all_outputs):
        for _ in range(2):
            step(all_outputs)
        torch.cuda.synchronize()
        n = max(3, min(args.steps, 10))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(n):
            step(all_outputs)
        b.record(stream)  # the last step's kernels follow every copy (events), so b ends them
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n, n

    ms, n = timed(False)
    ms_all, _ = timed(True)
    return {"value": flops / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 4, "steps": n,
            "note": "pinned host buffers; every input of the four modules H2D each step (on a "
                    "copy stream, module i+1's copy overlapping module i's kernels); the step's "
                    "result (an fp32 metric summing o and the five gradients, computed on the "
                    "device) D2H each step",
            "all_outputs_d2h": {"value": flops / (ms_all * 1e-3) / 1e12, "ms_per_step": ms_all,
                                "d2h_bytes_per_step": int(d2h_all),
                                "note": "same step, every output copied D2H"}}


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["evo", "reference"], default="evo")
    ap.add_argument("--no-flush", action="store_true", help="do not flush L2 between steps")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches, not a graph")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the other BASELINE configs / side paths (the `configs` key)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-rows", type=int, default=2,
                    help="--impl reference: batch rows of each module per step")
    ap.add_argument("--dap", action="store_true", help="run the DAP path even at N=1")
    ap.add_argument("--nseq", type=int, default=None, help="(DAP) override N_seq")
    ap.add_argument("--nres", type=int, default=None, help="(DAP) override N_res")
    ap.add_argument("--no-overlap", action="store_true",
                    help="(DAP) run the pair stack on the caller's stream (no overlap)")
    ap.add_argument("--stack-blocks", type=int, default=8,
                    help="blocks of the chained DAP stack timed under one CUDA graph (0: skip)")
    ap.add_argument("--stack-nres", type=int, default=384)
    ap.add_argument("--stack-nseq", type=int, default=512)
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    main()
