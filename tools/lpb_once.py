"""One f2 backward call at the MSA shape (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from paper_2404_11068_b200 import evoattn
dev = torch.device("cuda:0")
rows, C, N = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (32768, 256, 1024)))
x = torch.randn(rows, C, device=dev).to(torch.bfloat16)
g, b = torch.ones(C, device=dev), torch.zeros(C, device=dev)
W = (torch.randn(N, C, device=dev) / C ** 0.5).to(torch.bfloat16)
_, mean, rstd = evoattn.ln_proj_fwd(x, g, b, W)
dout = torch.randn(rows, N, device=dev).to(torch.bfloat16)
for _ in range(2):
    evoattn.ln_proj_bwd(x, g, b, W, mean, rstd, dout)
torch.cuda.synchronize()
print("ok")
