"""Forward A/B at the row shape: with and without the bias, occ vs pp (EVO_FWD_IMPL)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import bench
from paper_2404_11068_b200 import evoattn
dev = torch.device("cuda:0")
name, B, H, L, bias = bench.MODULES[0]
t = bench.make_module_inputs(torch, dev, name, B, H, L, bias, seed=100)
def timeit(fn, n=20):
    for _ in range(3): fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3
r = {}
r["bias"] = timeit(lambda: evoattn.fwd(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"]))
r["nobias"] = timeit(lambda: evoattn.fwd(t["q"], t["k"], t["v"], None, t["mask"], t["g"]))
r["nobias_nomask"] = timeit(lambda: evoattn.fwd(t["q"], t["k"], t["v"], None, None, t["g"]))
r["nobias_nomask_nogate"] = timeit(lambda: evoattn.fwd(t["q"], t["k"], t["v"], None, None, None))
print(os.environ.get("EVO_FWD_IMPL", "occ"), {k: round(v, 1) for k, v in r.items()})
