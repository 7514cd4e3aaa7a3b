"""Step-by-step GPU bring-up: run fwd / bwd on small cases, sync and report after each call."""
import sys, os, traceback
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from gpu_harness import run_case

cases = [
    dict(B=1, H=1, Lq=128, Lk=128, D=32, bias=None, gate=False, mask="none", layout="bhld", bwd=False),
    dict(B=1, H=1, Lq=128, Lk=128, D=32, bias=None, gate=False, mask="none", layout="bhld", dtype=torch.float32, bwd=False),
    dict(B=2, H=2, Lq=256, Lk=256, D=32, bias="shared", gate=True, mask="prefix", layout="blhd", bwd=False),
    dict(B=1, H=1, Lq=128, Lk=128, D=32, bias=None, gate=False, mask="none", layout="bhld", bwd=True),
    dict(B=2, H=2, Lq=256, Lk=256, D=32, bias="shared", gate=True, mask="prefix", layout="blhd", bwd=True),
    dict(B=2, H=2, Lq=256, Lk=256, D=32, bias="shared", gate=True, mask="prefix", layout="blhd", dtype=torch.float32, bwd=True),
    dict(B=2, H=2, Lq=200, Lk=200, D=16, bias="shared", gate=True, mask="prefix", layout="blhd", bwd=True),
    dict(B=2, H=2, Lq=129, Lk=129, D=8, bias=None, gate=True, mask="prefix", layout="bhld", bwd=True),
    dict(B=2, H=2, Lq=300, Lk=300, D=64, bias="shared", gate=True, mask="prefix", layout="blhd", bwd=True),
]
for i, c in enumerate(cases):
    try:
        errs, _, _ = run_case(seed=1, **c)
        print(i, c, {k: f"{v:.2e}" for k, v in errs.items()}, flush=True)
    except Exception as e:
        print(i, c, "EXC", repr(e)[:400], flush=True)
        traceback.print_exc()
        if "illegal" in repr(e) or "CUDA" in repr(e) and "EvoError" not in repr(e):
            break
