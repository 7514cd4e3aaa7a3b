"""Block step (4 modules fwd+bwd) eager vs captured in a CUDA graph: device time per step."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import bench
from paper_2404_11068_b200 import evoattn
dev = torch.device("cuda:0")
mods = []
for i, (name, B, H, L, bias) in enumerate(bench.MODULES):
    t = bench.make_module_inputs(torch, dev, name, B, H, L, bias, seed=100 + i)
    ws = torch.empty(max(1, evoattn.workspace_bytes(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"])), dtype=torch.uint8, device=dev)
    mods.append((t, ws))
def step():
    for t, ws in mods:
        o, lse = evoattn.fwd(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"])
        evoattn.bwd(t["q"], t["k"], t["v"], o, lse, t["dout"], t["bias"], t["mask"], t["g"], workspace=ws)
flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)
for _ in range(3): step()
torch.cuda.synchronize()
def timeit(fn, n=20):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        flush.zero_(); a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[n // 2]
print("eager ms", timeit(step))
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    step()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        step()
torch.cuda.synchronize()
print("graph ms", timeit(g.replay))
# per-kernel trace events captured as graph nodes
import ctypes
lib = evoattn.load()
trace_ev = [torch.cuda.Event(enable_timing=True) for _ in range(128)]
for e in trace_ev:
    e.record()
torch.cuda.synchronize()
arr = (ctypes.c_void_p * len(trace_ev))(*[e.cuda_event for e in trace_ev])
g2 = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    lib.evo_trace_enable(arr, len(trace_ev))
    with torch.cuda.graph(g2, stream=s):
        step()
    ntr = lib.evo_trace_count()
    labels = [lib.evo_trace_label(i).decode() for i in range(ntr)]
    lib.evo_trace_enable(None, 0)
torch.cuda.synchronize()
print("traced graph ms", timeit(g2.replay), "events", ntr)
g2.replay(); torch.cuda.synchronize()
for i, lab in enumerate(labels):
    print(lab, round(trace_ev[2 * i].elapsed_time(trace_ev[2 * i + 1]) * 1e3, 1))
