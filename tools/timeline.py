"""Per-sub-tile timeline of bwd_fused (clock64 stamps of CTAs 0/1) from a debug build compiled
with -DEVO_TIMELINE (never the product library).  python tools/timeline.py [row|start|end|col]
Prints per-group medians of: S wait (S issued -> landed), compute (landed -> hand-off),
hand-off -> next wait, and the grad-issuer / dQ timings."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2404_11068_b200 import build as B  # noqa: E402

out_dir = os.path.join(B.HERE, "build_tl")
os.makedirs(out_dir, exist_ok=True)
lib_tl = os.path.join(out_dir, "libevoattn_tl.so")
objs = []
procs = []
for s in B.ATTN_SRCS:
    o = os.path.join(out_dir, s.replace(".cu", ".o"))
    objs.append(o)
    procs.append(subprocess.Popen([B.NVCC, *B.ARCH, *B.FLAGS, "-DEVO_TIMELINE", "-c",
                                   os.path.join(B.CSRC, s), "-o", o]))
assert all(p.wait() == 0 for p in procs)
subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", lib_tl, *objs])

import torch  # noqa: E402
from paper_2404_11068_b200 import evoattn  # noqa: E402
evoattn._LIB_PATH = lib_tl
lib = evoattn.load()
lib.evo_debug_timeline_copy.argtypes = [ctypes.c_void_p, ctypes.c_size_t]

kind = sys.argv[1] if len(sys.argv) > 1 else "row"
Bn, H, L, D, bias, st, bt = {"row": (128, 8, 256, 32, True, "bl", False),
                             "start": (256, 4, 256, 32, True, "bl", False),
                             "end": (256, 4, 256, 32, True, "lb", True),
                             "col": (256, 8, 128, 32, False, "lb", False)}[kind]
dev = torch.device("cuda:0")
shape, perm = ((Bn, L, H, D), (0, 2, 1, 3)) if st == "bl" else ((L, Bn, H, D), (1, 2, 0, 3))
t = {n: torch.randn(shape, device=dev).to(torch.bfloat16).permute(*perm)
     for n in ("q", "k", "v", "g", "dout")}
b = torch.randn((H, L, L), device=dev).to(torch.bfloat16) if bias else None
t["bias"] = (b.transpose(1, 2) if bt else b) if bias else None
m = torch.ones((Bn, L), dtype=torch.uint8)
t["mask"] = m.t().contiguous().to(dev).t() if st == "lb" else m.to(dev)
for _ in range(3):
    o, lse = evoattn.fwd(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"])
    evoattn.bwd(t["q"], t["k"], t["v"], o, lse, t["dout"], t["bias"], t["mask"], t["g"])
torch.cuda.synchronize()
buf = np.zeros((2, 12, 512), dtype=np.uint64)
assert lib.evo_debug_timeline_copy(buf.ctypes.data, buf.nbytes) == 0
tl = buf[0].astype(np.int64)
J = int(np.max(np.nonzero(tl[3])[0])) + 1
t0 = tl[0][0]
rel = lambda x: x - t0
print(f"{kind}: J={J} sub-tiles on CTA 0, span {rel(tl[3][J - 1])} cycles, "
      f"{rel(tl[3][J - 1]) / J:.0f} per sub-tile")
for g in (0, 1):
    js = np.arange(g, J, 2)
    wait = tl[2][js] - tl[1][js]
    comp = tl[3][js] - tl[2][js]
    nxt = tl[1][js[1:]] - tl[3][js[:-1]]
    print(f"group {g}: S wait med {np.median(wait):.0f} mean {wait.mean():.0f} | compute med "
          f"{np.median(comp):.0f} mean {comp.mean():.0f} | hand-off->next wait med "
          f"{np.median(nxt):.0f} mean {nxt.mean():.0f}")
for g in (0, 1):
    js = np.arange(g, J, 2)
    ld = tl[11][js] - tl[2][js]
    math = tl[9][js] - tl[11][js]
    mmw = tl[10][js] - tl[9][js]
    st_ = tl[3][js] - tl[10][js]
    print(f"group {g} compute split (median): ldtm {np.median(ld):.0f} | math+Σ {np.median(math):.0f} "
          f"| wait Pᵀ slot/dS buf {np.median(mmw):.0f} (mean {mmw.mean():.0f}) | stores+fence "
          f"{np.median(st_):.0f}")
i = np.arange(J)
print(f"grad issuer: issue of dV/dK takes med {np.median(tl[8][i] - tl[5][i]):.0f} "
      f"mean {np.mean(tl[8][i] - tl[5][i]):.0f}")
js = np.arange(0, J, 2)
iss = tl[0][js]
land0 = tl[2][js]
print(f"S pair issue -> group0 landed: med {np.median(land0 - iss):.0f}; issue gaps med "
      f"{np.median(np.diff(iss)):.0f}")
i = np.arange(J)
print(f"hand-off -> grad issuer sees it: med {np.median(tl[4][i] - tl[3][i]):.0f}; "
      f"dkvfree wait med {np.median(tl[5][i] - tl[4][i]):.0f} max {np.max(tl[5][i] - tl[4][i])}")
nT = J // 4
T = np.arange(nT)
print(f"dQ issue -> landed (drain): med {np.median(tl[7][T] - tl[6][T]):.0f}")
print("first 12 sub-tiles (cycles from the first S issue): issue/wait/landed/handoff/grad")
for j in range(min(12, J)):
    print(j, rel(tl[0][j - (j & 1)]), rel(tl[1][j]), rel(tl[2][j]), rel(tl[3][j]), rel(tl[4][j]),
          rel(tl[5][j]))
