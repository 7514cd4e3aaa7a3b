"""f2 backward timing split: full call vs without db (python tools/lpb_split.py)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from paper_2404_11068_b200 import evoattn
if "--lib" in sys.argv:  # A/B against another build of the library
    evoattn._LIB_PATH = os.path.abspath(sys.argv[sys.argv.index("--lib") + 1])
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for rows, C, N in [(32768, 256, 1024), (65536, 128, 512), (262144, 64, 256)]:
    x = torch.randn(rows, C, device=dev).to(torch.bfloat16)
    g, b = torch.ones(C, device=dev), torch.zeros(C, device=dev)
    W = (torch.randn(N, C, device=dev) / C ** 0.5).to(torch.bfloat16)
    _, mean, rstd = evoattn.ln_proj_fwd(x, g, b, W)
    dout = torch.randn(rows, N, device=dev).to(torch.bfloat16)
    ws = torch.empty(1 << 26, dtype=torch.uint8, device=dev)
    res = {}
    for name, fn in (("full", lambda: evoattn.ln_proj_bwd(x, g, b, W, mean, rstd, dout, workspace=ws)),
                     ("no_db", lambda: evoattn.ln_proj_bwd(x, g, b, W, mean, rstd, dout, want_db=False, workspace=ws)),
                     ("linear_no_db", lambda: evoattn.linear_bwd(x, W, dout, want_db=False, workspace=ws))):
        for _ in range(3): fn()
        ts = []
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        res[name] = round(sorted(ts)[5], 1)
    print(rows, C, N, res, flush=True)
