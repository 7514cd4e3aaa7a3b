"""Per-CTA timeline of fwd_occ (debug build with -DEVO_TIMELINE; never the product library).
python tools/fwd_timeline.py [row|start|end|col] — prints per-unit phase medians and how many
units overlap on one SM."""
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
objs, procs = [], []
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
lib.evo_debug_fwd_timeline_copy.argtypes = [ctypes.c_void_p, ctypes.c_size_t]

kind = sys.argv[1] if len(sys.argv) > 1 else "row"
Bn, H, L, D, bias, st, bt = {"row": (128, 8, 256, 32, True, "bl", False),
                             "start": (256, 4, 256, 32, True, "bl", False),
                             "end": (256, 4, 256, 32, True, "lb", True),
                             "col": (256, 8, 128, 32, False, "lb", False)}[kind]
dev = torch.device("cuda:0")
shape, perm = ((Bn, L, H, D), (0, 2, 1, 3)) if st == "bl" else ((L, Bn, H, D), (1, 2, 0, 3))
t = {n: torch.randn(shape, device=dev).to(torch.bfloat16).permute(*perm)
     for n in ("q", "k", "v", "g")}
b = torch.randn((H, L, L), device=dev).to(torch.bfloat16) if bias else None
t["bias"] = (b.transpose(1, 2) if bt else b) if bias else None
m = torch.ones((Bn, L), dtype=torch.uint8)
t["mask"] = m.t().contiguous().to(dev).t() if st == "lb" else m.to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(3):
    flush.zero_()
    evoattn.fwd(t["q"], t["k"], t["v"], t["bias"], t["mask"], t["g"])
torch.cuda.synchronize()
buf = np.zeros((4096, 20), dtype=np.uint64)
assert lib.evo_debug_fwd_timeline_copy(buf.ctypes.data, buf.nbytes) == 0
n = min(4096, Bn * H * ((L + 127) // 128))
tl = buf[:n].astype(np.int64)
nc = (L + 63) // 64
sm = tl[:, 19]
pro = tl[:, 1] - tl[:, 0]
first_s = tl[:, 2] - tl[:, 1]
sm_ph = [tl[:, 3 + 2 * c] - tl[:, 2 + 2 * c] for c in range(min(nc, 8))]
gap = [tl[:, 2 + 2 * (c + 1)] - tl[:, 3 + 2 * c] for c in range(min(nc, 8) - 1)]
epi = tl[:, 18] - tl[:, 3 + 2 * (min(nc, 8) - 1)]
tot = tl[:, 18] - tl[:, 0]
print(f"{kind}: {n} units, {nc} key chunks; per-unit medians (cycles): total {np.median(tot):.0f}, "
      f"prologue {np.median(pro):.0f}, first S {np.median(first_s):.0f}, "
      f"softmax per chunk {[int(np.median(x)) for x in sm_ph]}, "
      f"P_c -> S_c+1 landed {[int(np.median(x)) for x in gap]}, epilogue {np.median(epi):.0f}")
s0 = sm[0]
on = np.nonzero(sm == s0)[0]
st0 = tl[on, 0] - tl[on, 0].min()
en0 = tl[on, 18] - tl[on, 0].min()
order = np.argsort(st0)
print(f"SM {s0}: {len(on)} units, span {en0.max()} cycles ({en0.max() / len(on):.0f} per unit)")
for i in order[:12]:
    print(f"  unit {on[i]}: start {st0[i]} end {en0[i]} (len {en0[i] - st0[i]})")
