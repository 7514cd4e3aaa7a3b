"""Per-chunk timeline of the occupancy forward, thread 0 of CTAs 0..147 (EVO_DEBUG_TIMING=1)."""
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
    for _ in range(3):
        evoattn.fwd(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"])
    torch.cuda.synchronize()
lib = evoattn.load()
buf = np.zeros(148 * 8 * 32 * 8 + 148 * 64 * 4, dtype=np.uint64)
lib.evo_debug_fwd_timing(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
d = buf[:148 * 512].reshape(148, 512).astype(np.int64)
tma = d[:, :32].reshape(148, 8, 4)
sm = d[:, 256:288].reshape(148, 8, 4)
rows = []
for cta in range(148):
    t0 = tma[cta, 0, 1]
    for c in range(4):
        iss, rdy = tma[cta, c, 1], tma[cta, c, 2]
        s0_, s1_, s2_, s3_ = sm[cta, c]
        if not (iss and rdy and s0_): continue
        rows.append([rdy - iss, s1_ - s0_, s2_ - s1_, s3_ - s2_, s3_ - t0])
r = np.array(rows)
names = ["TMA lat", "S wait", "softmax", "sync", "t since start"]
for k, n in enumerate(names):
    print(f"{n:14s} median {np.median(r[:, k]):8.0f}  p90 {np.percentile(r[:, k], 90):8.0f}")
print("cta 3 timeline (rel start): ", [(int(sm[3, c, 0] - tma[3, 0, 1]), int(sm[3, c, 1] - tma[3, 0, 1]), int(sm[3, c, 3] - tma[3, 0, 1])) for c in range(4)], "tma ready", [int(tma[3, c, 2] - tma[3, 0, 1]) for c in range(4)])
for cta in (3, 50, 100):
    t0 = tma[cta, 0, 1]
    print(f"cta {cta}:")
    for c in range(4):
        print(f"  c{c}: issue {tma[cta,c,1]-t0} kvwait {tma[cta,c,0]-t0 if tma[cta,c,0] else '-'} kvready {tma[cta,c,2]-t0} Swait {sm[cta,c,0]-t0} Sdone {sm[cta,c,1]-t0} smx_end {sm[cta,c,2]-t0} sync_end {sm[cta,c,3]-t0}")
    print(f"  O done {d[cta,299]-t0} end {d[cta,300]-t0}")
