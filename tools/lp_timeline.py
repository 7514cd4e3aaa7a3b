"""Per-CTA timeline of the f2 kernel (LP_EXP=5 variant): µs since the earliest CTA start."""
import ctypes, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch
from paper_2404_11068_b200.evoattn import LnProjDesc

rows, C, N = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (32768, 256, 1024))]
dev = torch.device("cuda:0")
x = torch.randn((rows, C), device=dev).to(torch.bfloat16)
g, bt = torch.ones(C, device=dev), torch.zeros(C, device=dev)
W = (torch.randn((N, C), device=dev) / C ** 0.5).to(torch.bfloat16)
out = torch.empty((rows, N), dtype=torch.bfloat16, device=dev)
dbg = torch.zeros((148, 64), dtype=torch.int64, device=dev)
d = LnProjDesc()
d.rows, d.C, d.N, d.eps, d.x_ld, d.out_ld = rows, C, N, 1e-5, C, N
P = lambda t: ctypes.c_void_p(t.data_ptr())
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), os.environ.get("LPV", "lpvar/lp_tl.so")))
for _ in range(5):
    dbg.zero_()
    assert lib.evo_ln_proj_fwd(ctypes.byref(d), P(x), P(g), P(bt), P(W), None, P(out), P(dbg), None, None) == 0
torch.cuda.synchronize()
t = dbg.cpu().numpy().astype(np.float64)
t0 = t[:, 0][t[:, 0] > 0].min()
rel = np.where(t > 0, (t - t0) / 1e3, np.nan)
names = {0: "start", 1: "ln0 beg", 2: "ln1 beg", 5: "ln0 end", 6: "ln1 end", 9: "mma0 beg",
         10: "mma1 beg", 13: "mma0 end", 14: "mma1 end", 33: "epi0 beg", 34: "epi1 beg", 41: "end"}
for k, n in names.items():
    col = rel[:, k]
    col = col[~np.isnan(col)]
    if len(col):
        print(f"{n:9s} n={len(col):3d} min {col.min():6.2f} med {np.median(col):6.2f} max {col.max():6.2f} us")
