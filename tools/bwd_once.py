"""fwd + bwd of one bench module shape through the C ABI, 3 times (for ncu captures of the
small kernels).  python tools/bwd_once.py [row|start|end|col]"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from paper_2404_11068_b200 import evoattn

kind = sys.argv[1] if len(sys.argv) > 1 else "row"
B, H, L, D, bias, st, bt = {"row": (128, 8, 256, 32, True, "bl", False),
                            "start": (256, 4, 256, 32, True, "bl", False),
                            "end": (256, 4, 256, 32, True, "lb", True),
                            "col": (256, 8, 128, 32, False, "lb", False)}[kind]
dev = torch.device("cuda:0")
shape, perm = ((B, L, H, D), (0, 2, 1, 3)) if st == "bl" else ((L, B, H, D), (1, 2, 0, 3))
t = {n: torch.randn(shape, device=dev).to(torch.bfloat16).permute(*perm)
     for n in ("q", "k", "v", "g", "dout")}
b = torch.randn((H, L, L), device=dev).to(torch.bfloat16) if bias else None
t["bias"] = (b.transpose(1, 2) if bt else b) if bias else None
m = torch.ones((B, L), dtype=torch.uint8)
t["mask"] = m.t().contiguous().to(dev).t() if st == "lb" else m.to(dev)
ws = torch.empty(max(1, evoattn.workspace_bytes(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"])),
                 dtype=torch.uint8, device=dev)
for _ in range(3):
    o, lse = evoattn.fwd(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"])
    evoattn.bwd(t["q"], t["k"], t["v"], o, lse, t["dout"], t["bias"], t["mask"], t["g"], workspace=ws)
torch.cuda.synchronize()
print("ok", kind)
