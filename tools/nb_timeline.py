"""Per-hand-off timeline of the no-bias backward (evo_bwd_nb.cu: col, cfg5col, cfg4) or the
pair-bias backward (evo_bwd_pb.cu: row, start, end) — clock64 stamps of CTA 0 — from a debug
build compiled with -DEVO_TIMELINE (never the product library).
python tools/nb_timeline.py [col|cfg5col|cfg4|row|start|end ...]"""
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
lib.evo_debug_nb_timeline_copy.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
lib.evo_debug_pb_timeline_copy.argtypes = [ctypes.c_void_p, ctypes.c_size_t]

for kind in sys.argv[1:] or ["col"]:
    Bn, H, L, D, bias, st = {"col": (256, 8, 128, 32, None, "lb"),
                             "cfg5col": (384, 8, 512, 32, None, "lb"),
                             "cfg4": (256, 8, 1024, 8, None, "lb"),
                             "row": (128, 8, 256, 32, "k", "bl"),
                             "start": (256, 4, 256, 32, "k", "bl"),
                             "end": (256, 4, 256, 32, "q", "lb")}[kind]
    dev = torch.device("cuda:0")
    shape, perm = ((Bn, L, H, D), (0, 2, 1, 3)) if st == "bl" else ((L, Bn, H, D), (1, 2, 0, 3))
    t = {n: torch.randn(shape, device=dev).to(torch.bfloat16).permute(*perm)
         for n in ("q", "k", "v", "g", "dout")}
    bb = None
    if bias:
        bb = torch.randn((H, L, L), device=dev).to(torch.bfloat16)
        bb = bb.transpose(1, 2) if bias == "q" else bb
    m = torch.ones((Bn, L), dtype=torch.uint8)
    m = m.t().contiguous().to(dev).t() if st == "lb" else m.to(dev)
    for _ in range(3):
        o, lse = evoattn.fwd(t["q"], t["k"], t["v"], bb, m, t["g"])
        evoattn.bwd(t["q"], t["k"], t["v"], o, lse, t["dout"], bb, m, t["g"])
    torch.cuda.synchronize()
    buf = np.zeros((2, 16 if bias else 14, 512), dtype=np.uint64)
    cp = lib.evo_debug_pb_timeline_copy if bias else lib.evo_debug_nb_timeline_copy
    assert cp(buf.ctypes.data, buf.nbytes) == 0
    tl = buf[0].astype(np.int64)
    J = int(np.max(np.nonzero(tl[5])[0])) + 1
    t0 = tl[11][0]
    i = np.arange(1, J)
    med = lambda x: float(np.median(x))
    print(f"{kind}: {J} hand-offs on CTA 0, span {tl[5][J - 1] - t0} cycles, "
          f"{(tl[5][J - 1] - tl[5][0]) / (J - 1):.0f} per hand-off")
    if bias:
        print(f"  compute: wait S {med(tl[2][i] - tl[1][i]):.0f} | math + Σ {med(tl[3][i] - tl[2][i]):.0f}"
              f" | wait Pᵀ/dS free {med(tl[4][i] - tl[3][i]):.0f} (mean {np.mean(tl[4][i] - tl[3][i]):.0f})"
              f" | stores + hand-off {med(tl[5][i] - tl[4][i]):.0f}")
        print(f"    math split: LDTM {med(tl[14][i] - tl[2][i]):.0f} | vec wait {med(tl[13][i] - tl[14][i]):.0f}"
              f" | math {med(tl[15][i] - tl[13][i]):.0f} | Σ store issue {med(tl[3][i] - tl[15][i]):.0f}")
    else:
        print(f"  compute: wait S {med(tl[2][i] - tl[1][i]):.0f} | batch0 math {med(tl[3][i] - tl[2][i]):.0f}"
              f" | wait Pᵀ/dS free {med(tl[4][i] - tl[3][i]):.0f} (mean {np.mean(tl[4][i] - tl[3][i]):.0f})"
              f" | batch1 math + wait {med(tl[13][i] - tl[4][i]):.0f} | stores + hand-off "
              f"{med(tl[5][i] - tl[13][i]):.0f}")
    print(f"  S issuer: ready after prev hand-off {med(tl[12][i] - tl[5][i - 1]):.0f}; "
          f"issued -> landed seen {med(tl[2][i] - tl[0][i]):.0f}; load issue -> S ready "
          f"{med(tl[12][i] - tl[11][i]):.0f}")
    print(f"  grad: hand-off seen {med(tl[6][i] - tl[5][i]):.0f} | dkvfree wait "
          f"{med(tl[7][i] - tl[6][i]):.0f} (max {np.max(tl[7][i] - tl[6][i])}) | dV/dK issue "
          f"{med(tl[8][i] - tl[7][i]):.0f} | dqfree + dQ issue {med(tl[9][i] - tl[8][i]):.0f} "
          f"(max {np.max(tl[9][i] - tl[8][i])})")
    last = [x for x in range(J) if tl[10][x] > 0]
    if last:
        lx = np.array(last)
        print(f"  drain: dV/dK issued -> landed {med(tl[10][lx] - tl[8][lx]):.0f}")
    if bias:
        t1 = buf[1].astype(np.int64)
        J1 = int(np.max(np.nonzero(t1[5])[0])) + 1
        print(f"  CTA 1: {(t1[5][J1 - 1] - t1[5][0]) / (J1 - 1):.0f} per hand-off")
        od = np.arange(1, J, 2)
        for nm, tt in (("CTA 0", tl), ("CTA 1", t1)):
            print(f"  {nm} drain per tile: dQ issued -> pulled qd0 {med(tt[13][od] - tt[9][od]):.0f} "
                  f"qd2 {med(tt[12][od] - tt[9][od]):.0f}; pulled -> exchange done qd0 "
                  f"{med(tt[11][od] - tt[13][od]):.0f} (max {np.max(tt[11][od] - tt[13][od])}) qd2 "
                  f"{med(tt[10][od - 1] - tt[12][od]):.0f} (max {np.max(tt[10][od - 1] - tt[12][od])})")
        if False:
            print(f"  dQ drain (pair): dQ issued -> rank 1 data in {med(tl[13][od] - tl[9][od]):.0f}"
                  f" -> stored {med(tl[11][od] - tl[13][od]):.0f}; rank 1 recvfree wait "
                  f"{med(t1[11][od] - t1[9][od]):.0f} after its dQ issue")
    print("  first tiles (cycles from the first load): load S-ready S-issued wait landed b0 free "
          "handoff seen dkvfree dVdK dQ")
    for x in range(min(10, J)):
        print("  ", x, *[int(tl[e][x] - t0) for e in (11, 12, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9)])
