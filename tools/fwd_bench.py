"""Time the forward kernel alone per module (CUDA events, L2 warm): python tools/fwd_bench.py"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import bench
from paper_2404_11068_b200 import evoattn
dev = torch.device("cuda:0")
res = {}
for i, (name, B, H, L, bias) in enumerate(bench.MODULES):
    t = bench.make_module_inputs(torch, dev, name, B, H, L, bias, seed=100 + i)
    f = lambda: evoattn.fwd(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"])
    for _ in range(3): f()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): f()
    b.record(); torch.cuda.synchronize()
    res[name] = round(a.elapsed_time(b) / 20 * 1e3, 1)
print(os.environ.get("EVO_FWD_FLAGS", "0"), res, "sum_us", round(sum(res.values()), 1))
