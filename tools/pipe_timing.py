"""Producer / MMA issue timing of the warp-specialised forward (EVO_DEBUG_TIMING=1)."""
import ctypes, os, sys
os.environ["EVO_DEBUG_TIMING"] = "1"
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import bench
from paper_2404_11068_b200 import evoattn
dev = torch.device("cuda:0")
which = sys.argv[1] if len(sys.argv) > 1 else "col"
for i, (name, B, H, L, bias) in enumerate(bench.MODULES):
    if name != which: continue
    t = bench.make_module_inputs(torch, dev, name, B, H, L, bias, seed=100 + i)
    for _ in range(3):
        evoattn.fwd(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"])
    torch.cuda.synchronize()
lib = evoattn.load()
n1 = 148 * 8 * 32 * 8
buf = np.zeros(n1 + 148 * 64 * 4, dtype=np.uint64)
lib.evo_debug_fwd_timing(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
d = buf[n1:].reshape(148, 64, 4).astype(np.int64)
c = d[5]
base = c[0, 0]
print("cta 5, per entry (cycles rel. to first): prod_wait_start, prod_issue, mma_S, mma_PV")
for e in range(min(28, 64)):
    if c[e, 0] == 0: break
    print(e, (c[e] - base).tolist(), " wait_empty", c[e, 1] - c[e, 0], " issue->S", c[e, 2] - c[e, 1], " S->PV", c[e, 3] - c[e, 2])
