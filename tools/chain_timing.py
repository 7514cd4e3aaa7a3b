"""S round-trip chain of the warp-specialised forward (EVO_DEBUG_TIMING=1), cycles on one SM."""
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
sm = buf[:n1].reshape(148, 8, 32, 8).astype(np.int64)
mm = buf[n1:].reshape(148, 64, 4).astype(np.int64)
cta = 7
print("slot tile: S_issue->S_full(wake)  wake->ld_done  ld_done->P_full  P_full->PV_issue  PV_issue->next S_full")
for t in range(8):
    for s in range(2):
        e = 2 * t + s
        w = 4 * s  # first warp of the slot
        si, pi = mm[cta, e, 2], mm[cta, e, 3]
        wake, ldd, pf = sm[cta, w, t, 1], sm[cta, w, t, 2], sm[cta, w, t, 6]
        nxt = sm[cta, w, t + 1, 1] if t + 1 < 32 else 0
        print(s, t, wake - si, ldd - wake, pf - ldd, pi - pf, nxt - pi if nxt else None)
print("per-warp P_full arrive times (rel. to warp 0) and wake times, slot 0 / slot 1")
for s in range(2):
    for t in range(6):
        ws = [4 * s + q for q in range(4)]
        pf = [sm[cta, w_, t, 6] - sm[cta, ws[0], t, 6] for w_ in ws]
        wk = [sm[cta, w_, t, 1] - sm[cta, ws[0], t, 1] for w_ in ws]
        ex = [sm[cta, w_, t, 5] - sm[cta, w_, t, 4] for w_ in ws]
        print(s, t, "P_full", pf, " wake", wk, " exps", ex)
