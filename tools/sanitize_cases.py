"""Small invocations of every hot kernel for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): python tools/sanitize_cases.py.  Shapes span several tiles and ragged tails and hit
each kernel variant: fwd_occ (no bias / k-contiguous bias / q-contiguous bias), bwd_pre,
bwd_fused (nk = 1, 2 reduce-add, 3 ordered parts; bias and none; D = 16 / 32), the two-pass
backward (L > 256 with a bias, D = 64, per-batch bias), dq_convert, dbias_reduce, the fp32
verification path, pair_bias fwd/bwd, ln_proj, global attention fwd/bwd, the DAP pack."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from gpu_harness import to_dev_bias, to_dev_mask, to_dev_x  # noqa: E402
from paper_2404_11068_b200 import dap, evoattn  # noqa: E402
from synth.gen import attention_case  # noqa: E402

dev = torch.device("cuda:0")
CASES = [  # B, H, L, D, bias, bias_t, layout, dtype
    (2, 2, 200, 32, "shared", False, "blhd", torch.bfloat16),
    (2, 2, 256, 32, "shared", True, "lbhd", torch.bfloat16),
    (3, 2, 130, 32, None, False, "lbhd", torch.bfloat16),
    (2, 1, 384, 16, None, False, "blhd", torch.bfloat16),
    (2, 1, 300, 32, "shared", False, "blhd", torch.bfloat16),
    (2, 1, 140, 64, "shared", False, "blhd", torch.bfloat16),
    (2, 1, 96, 32, "batch", False, "blhd", torch.bfloat16),
    (2, 1, 70, 16, "shared", False, "blhd", torch.float32),
]
for B, H, L, D, bias, bt, layout, dt in CASES:
    c = attention_case(B, H, L, L, D, seed=1, bias=bias, gate=True, mask="prefix_fm")
    t = {n: to_dev_x(c[n], dt, layout, dev) for n in ("q", "k", "v", "g", "dout")}
    b = to_dev_bias(c["bias"], dt, bt, dev) if c["bias"] is not None else None
    m = to_dev_mask(c["mask"], layout == "lbhd", dev)
    o, lse = evoattn.fwd(t["q"], t["k"], t["v"], b, m, t["g"], c["scale"])
    evoattn.bwd(t["q"], t["k"], t["v"], o, lse, t["dout"], b, m, t["g"], c["scale"])
    torch.cuda.synchronize()
    print("attn", (B, H, L, D, bias, bt, layout, str(dt)), "ok", flush=True)

L, C, H = 40, 32, 4
z = torch.randn((L, L, C), device=dev).to(torch.bfloat16)
gamma, beta = torch.ones(C, device=dev), torch.zeros(C, device=dev)
W = torch.randn((C, H), device=dev)
bias, mean, rstd = evoattn.pair_bias_fwd(z, gamma, beta, W)
evoattn.pair_bias_bwd(z, gamma, beta, W, mean, rstd, torch.randn((H, L, L), device=dev),
                      workspace=torch.empty(1 << 22, dtype=torch.uint8, device=dev))
torch.cuda.synchronize()
print("pair_bias ok", flush=True)

rows, C, N = 300, 64, 256
x = torch.randn((rows, C), device=dev).to(torch.bfloat16)
evoattn.ln_proj_fwd(x, torch.ones(C, device=dev), torch.zeros(C, device=dev),
                    torch.randn((N, C), device=dev).to(torch.bfloat16), torch.zeros(N, device=dev))
torch.cuda.synchronize()
print("ln_proj ok", flush=True)

B, S, H, D = 6, 50, 2, 8
gq = torch.randn((B, S, H, D), device=dev).to(torch.bfloat16)
gg = torch.randn((B, S, H, D), device=dev).to(torch.bfloat16)
gk = torch.randn((B, S, D), device=dev).to(torch.bfloat16)
gv = torch.randn((B, S, D), device=dev).to(torch.bfloat16)
gm = (torch.rand((B, S), device=dev) > 0.2).to(torch.uint8)
o, lse, qbar = evoattn.global_attn_fwd(gq, gk, gv, gg, gm)
evoattn.global_attn_bwd(gq, gk, gv, gg, lse, qbar, o, gm)
torch.cuda.synchronize()
print("global_attn ok", flush=True)

src = torch.randint(0, 255, (4 * 4 * 64,), dtype=torch.uint8, device=dev)
dap.pack(src, torch.empty_like(src), 4, 4, 4, 16, 0)
dap.pack(src, torch.empty_like(src), 4, 4, 4, 16, 1)
torch.cuda.synchronize()
print("dap_pack ok", flush=True)
