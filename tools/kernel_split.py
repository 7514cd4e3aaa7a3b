"""Per-kernel device time of one fwd + bwd call (C-ABI trace events) at a given shape.
python tools/kernel_split.py B H L D bias(0/1/t) [layout bl|lb] [--lib other.so]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2404_11068_b200 import evoattn  # noqa: E402

if "--lib" in sys.argv:  # A/B against another build of the library (e.g. a previous commit's)
    i = sys.argv.index("--lib")
    evoattn._LIB_PATH = os.path.abspath(sys.argv[i + 1])
    del sys.argv[i:i + 2]

Bn, H, L, D = (int(x) for x in sys.argv[1:5])
bias = sys.argv[5]
st = sys.argv[6] if len(sys.argv) > 6 else "bl"
dev = torch.device("cuda:0")
shape, perm = ((Bn, L, H, D), (0, 2, 1, 3)) if st == "bl" else ((L, Bn, H, D), (1, 2, 0, 3))
t = {n: torch.randn(shape, device=dev).to(torch.bfloat16).permute(*perm)
     for n in ("q", "k", "v", "g", "dout")}
t["bias"] = None
if bias != "0":
    bb = torch.randn((H, L, L), device=dev).to(torch.bfloat16)
    t["bias"] = bb.transpose(1, 2) if bias == "t" else bb
m = torch.ones((Bn, L), dtype=torch.uint8)
t["mask"] = m.t().contiguous().to(dev).t() if st == "lb" else m.to(dev)
lib = evoattn.load()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def step():
    o, lse = evoattn.fwd(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"])
    evoattn.bwd(t["q"], t["k"], t["v"], o, lse, t["dout"], t["bias"], t["mask"], t["g"])


for _ in range(3):
    step()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(256)]
for e in ev:
    e.record()
torch.cuda.synchronize()
arr = (ctypes.c_void_p * len(ev))(*[e.cuda_event for e in ev])
res = {}
for _ in range(5):
    flush.zero_()
    lib.evo_trace_enable(arr, len(ev))
    step()
    torch.cuda.synchronize()
    n = lib.evo_trace_count()
    for i in range(n):
        lab = lib.evo_trace_label(i).decode()
        res.setdefault(lab, []).append(ev[2 * i].elapsed_time(ev[2 * i + 1]) * 1e3)
    lib.evo_trace_enable(None, 0)
print(sys.argv[1:], {k: round(sorted(v)[len(v) // 2], 1) for k, v in res.items()})
