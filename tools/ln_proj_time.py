"""Time evo_ln_proj_fwd (f2) at the AF2 module shapes; prints µs, GB/s and TFLOP/s per shape."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch

from paper_2404_11068_b200 import evoattn

dev = torch.device("cuda:0")
only = sys.argv[1] if len(sys.argv) > 1 else None
for name, rows, C, N in [("msa_row/col", 128 * 256, 256, 1024), ("triangle", 256 * 256, 128, 512),
                         ("extra_msa", 1024 * 256, 64, 256)]:
    if only and name != only:
        continue
    x = torch.randn((rows, C), device=dev).to(torch.bfloat16)
    g, bt = torch.ones(C, device=dev), torch.zeros(C, device=dev)
    W = (torch.randn((N, C), device=dev) / C ** 0.5).to(torch.bfloat16)
    b = torch.zeros(N, device=dev)
    out = torch.empty((rows, N), dtype=torch.bfloat16, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        evoattn.ln_proj_fwd(x, g, bt, W, b, out=out)
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        evoattn.ln_proj_fwd(x, g, bt, W, b, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    t = sorted(ts)[len(ts) // 2]
    byt = rows * C * 2 + rows * N * 2 + N * C * 2 + rows * 8
    fl = 2.0 * rows * C * N
    ref = torch.nn.functional.linear(torch.nn.functional.layer_norm(x.float(), (C,)), W.float())
    err = ((out.float() - ref).abs().max() / ref.abs().max()).item()
    print(f"{name:12s} rows={rows} C={C} N={N}: {t:7.1f} us  {byt / t / 1e3:7.0f} GB/s  "
          f"{fl / t / 1e6:6.0f} TFLOP/s  err={err:.2e}")
