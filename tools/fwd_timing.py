"""Phase timing of the warp-specialised forward (EVO_DEBUG_TIMING=1)."""
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
buf = np.zeros(148 * 8 * 32 * 8, dtype=np.uint64)
lib.evo_debug_fwd_timing(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
d = buf.reshape(148, 8, 32, 8).astype(np.int64)
valid = (d[..., 1] > 0) & (d[..., 7] > 0)
names = ["wait_S", "ld_S", "bias+mask+max", "wait_turn", "exps", "waitO+stP", "stats/end"]
for k in range(7):
    x = (d[..., k + 1] - d[..., k])[valid]
    print(f"{names[k]:16s} median {np.median(x):7.0f} mean {x.mean():7.0f} p90 {np.percentile(x, 90):7.0f}")
gap = (d[:, :, 1:, 0] - d[:, :, :-1, 7])[valid[:, :, 1:] & valid[:, :, :-1]]
print(f"{'loop gap':16s} median {np.median(gap):7.0f} mean {gap.mean():7.0f}")
per = (d[:, :, 1:, 0] - d[:, :, :-1, 0])[valid[:, :, 1:] & valid[:, :, :-1]]
print("tile period median", np.median(per), "mean", per.mean())
