"""Per-config device time (fwd, bwd, fwd+bwd; L2 flushed) for BASELINE.json configs 1-5 through
the C ABI.  python tools/config_times.py"""
import os, sys, json
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from paper_2404_11068_b200 import evoattn

dev = torch.device("cuda:0")
flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)
CFG = [  # name, B, H, L, D, bias, storage ("bl": [B,L,H,D], "lb": [L,B,H,D]), bias transposed
    ("cfg1 tri-start N=32", 32, 2, 32, 16, True, "bl", False),
    ("cfg2 MSA row 128x256", 128, 8, 256, 32, True, "bl", False),
    ("cfg3 tri-start 256", 256, 4, 256, 32, True, "bl", False),
    ("cfg3 tri-end 256", 256, 4, 256, 32, True, "lb", True),
    ("block MSA col 256x128", 256, 8, 128, 32, False, "lb", False),
    ("cfg4 extra-MSA col 1024, 8x8", 256, 8, 1024, 8, False, "lb", False),
    ("f3 extra-MSA row 1024x256, 8x8", 1024, 8, 256, 8, True, "bl", False),
    ("cfg5 row 512x384", 512, 8, 384, 32, True, "bl", False),
    ("cfg5 col 384x512", 384, 8, 512, 32, False, "lb", False),
    ("cfg5 tri-start 384", 384, 4, 384, 32, True, "bl", False),
]


def mk(B, H, L, D, bias, st, bt, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    shape, perm = ((B, L, H, D), (0, 2, 1, 3)) if st == "bl" else ((L, B, H, D), (1, 2, 0, 3))
    t = {n: torch.randn(shape, generator=g).to(dev, torch.bfloat16).permute(*perm)
         for n in ("q", "k", "v", "g", "dout")}
    t["bias"] = None
    if bias:
        b = torch.randn((H, L, L), generator=g).to(dev, torch.bfloat16)
        t["bias"] = b.transpose(1, 2) if bt else b
    m = torch.ones((B, L), dtype=torch.uint8)
    t["mask"] = m.t().contiguous().to(dev).t() if st == "lb" else m.to(dev)
    return t


def timed(fn, n=10):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        flush.zero_(); a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[n // 2] * 1e3


res = []
for name, B, H, L, D, bias, st, bt in CFG:
    t = mk(B, H, L, D, bias, st, bt)
    ws = torch.empty(max(1, evoattn.workspace_bytes(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"])), dtype=torch.uint8, device=dev)
    f = lambda: evoattn.fwd(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"])
    o, lse = f()
    bw = lambda: evoattn.bwd(t["q"], t["k"], t["v"], o, lse, t["dout"], t["bias"], t["mask"], t["g"], workspace=ws)
    for _ in range(3): f(); bw()
    torch.cuda.synchronize()
    tf, tb = timed(f), timed(bw)
    tfb = timed(lambda: (f(), bw()))
    fl = 12.0 * B * H * L * L * D
    res.append({"config": name, "B": B, "H": H, "L": L, "D": D, "fwd_us": round(tf, 1),
                "bwd_us": round(tb, 1), "fwd_bwd_us": round(tfb, 1),
                "tflops_alg": round(fl / (tfb * 1e-6) / 1e12, 1)})
    print(json.dumps(res[-1]), flush=True)

# f3: extra-MSA global column attention core (AF2 Alg. 19) at N_extra=1024, N_res=256, 8x8
B, S, H, D = 256, 1024, 8, 8
gq = torch.randn((S, B, H, D), device=dev).to(torch.bfloat16).transpose(0, 1)
gg = torch.randn((S, B, H, D), device=dev).to(torch.bfloat16).transpose(0, 1)
gk = torch.randn((S, B, D), device=dev).to(torch.bfloat16).transpose(0, 1)
gv = torch.randn((S, B, D), device=dev).to(torch.bfloat16).transpose(0, 1)
gm = torch.ones((S, B), dtype=torch.uint8, device=dev).t()
o, lse, qbar = evoattn.global_attn_fwd(gq, gk, gv, gg, gm)
tf = timed(lambda: evoattn.global_attn_fwd(gq, gk, gv, gg, gm))
tb = timed(lambda: evoattn.global_attn_bwd(gq, gk, gv, gg, lse, qbar, o, gm))
by_f = (2 * B * S * H * D + 2 * B * S * D) * 2 + B * S * H * D * 2
by_b = (3 * B * S * H * D + 2 * B * S * D) * 2 + (2 * B * S * H * D + 2 * B * S * D) * 2
print(json.dumps({"config": "f3 extra-MSA global column attention 256x1024, 8x8", "fwd_us": round(tf, 1),
                  "bwd_us": round(tb, 1), "fwd_GBps": round(by_f / tf / 1e3), "bwd_GBps": round(by_b / tb / 1e3)}))
