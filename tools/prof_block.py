"""One Evoformer-block attention step (row, col, start, end; fwd+bwd) for ncu captures.
Usage: python tools/prof_block.py [iters]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2404_11068_b200 import evoattn  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dev = torch.device("cuda:0")
mods = []
for i, (name, B, H, L, bias) in enumerate(bench.MODULES):
    t = bench.make_module_inputs(torch, dev, name, B, H, L, bias, seed=100 + i)
    mods.append(t)
for _ in range(iters):
    for t in mods:
        o, lse = evoattn.fwd(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"])
        evoattn.bwd(t["q"], t["k"], t["v"], o, lse, t["dout"], t["bias"], t["mask"], t["g"])
torch.cuda.synchronize()
print("ok")
