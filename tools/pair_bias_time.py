"""Device time of the pair-bias side path at N_res=256, c_z=128 (H=4 triangle, H=8 MSA row)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from paper_2404_11068_b200 import evoattn
dev = torch.device("cuda:0")
flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)
for H in (4, 8):
    L, C = 256, 128
    z = torch.randn((L, L, C), device=dev).to(torch.bfloat16)
    gamma = torch.ones(C, device=dev); beta = torch.zeros(C, device=dev)
    W = torch.randn((C, H), device=dev) / C ** 0.5
    dbias = torch.randn((H, L, L), device=dev)
    bias, mean, rstd = evoattn.pair_bias_fwd(z, gamma, beta, W)
    ws = torch.empty(1 << 24, dtype=torch.uint8, device=dev)
    f = lambda: evoattn.pair_bias_fwd(z, gamma, beta, W)
    b = lambda: evoattn.pair_bias_bwd(z, gamma, beta, W, mean, rstd, dbias, workspace=ws)
    for fn, name, byts in ((f, "fwd", L * L * C * 2 + H * L * L * 2 + 8 * L * L),
                           (b, "bwd", 2 * L * L * C * 2 + H * L * L * 4 + 8 * L * L)):
        for _ in range(3): fn()
        ts = []
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        t = sorted(ts)[5]
        print(f"H={H} {name}: {t:.1f} us, {byts / t / 1e3:.0f} GB/s algorithmic")
