"""Both compute groups + issuers of fused-backward CTA 0 (EVO_DEBUG_TIMING=1)."""
import ctypes, os, sys
os.environ["EVO_DEBUG_TIMING"] = "1"
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import bench
from paper_2404_11068_b200 import evoattn
dev = torch.device("cuda:0")
which = sys.argv[1] if len(sys.argv) > 1 else "row"
for i, (name, B, H, L, bias) in enumerate(bench.MODULES):
    if name != which: continue
    t = bench.make_module_inputs(torch, dev, name, B, H, L, bias, seed=100 + i)
    o, lse = evoattn.fwd(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"])
    for _ in range(3):
        evoattn.bwd(t["q"], t["k"], t["v"], o, lse, t["dout"], t["bias"], t["mask"], t["g"])
    torch.cuda.synchronize()
lib = evoattn.load()
buf = np.zeros(148 * 8 * 32 * 8 + 148 * 64 * 4, dtype=np.uint64)
lib.evo_debug_fwd_timing(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
d = buf[:4096].astype(np.int64)
t0 = d[8 * 16]
print(" j g | Sissue  spwait spdone  ldone compdone  waitdone psarr | ps_seen")
for j in range(16, 48):
    c = d[j * 8: j * 8 + 6] - t0
    m = d[2048 + j * 4: 2048 + j * 4 + 2] - t0
    print(f"{j:2d} {j & 1} | {m[0]:6d} {c[0]:6d} {c[1]:6d} {c[2]:6d} {c[3]:6d} {c[4]:6d} {c[5]:6d} | {m[1]:6d}")
