"""One-off wide randomised parity sweep (GPU): N seeded random shapes over the ABI's space, every
output against the fp64 oracle at the bf16 tolerance — the same generator and check as
tests/test_gpu_parity.py::test_random_shapes_parity, more cases.
python tools/random_sweep.py [N] [seed]"""
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from gpu_harness import run_case  # noqa: E402
from test_gpu_parity import TOL, _random_cases  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 7
bad = 0
for i, case in enumerate(_random_cases(n, seed=seed)):
    B, H, L, D, bias, bias_t, gate, mask, mask_t, layout = case
    errs, _, _ = run_case(B, H, L, L, D, seed=L + 7 * D, bias=bias, bias_t=bias_t, gate=gate,
                          mask=mask, mask_t=mask_t, layout=layout)
    worst = max(errs.values())
    ok = worst <= TOL[torch.bfloat16]
    bad += not ok
    print(f"{i:4d} {'ok ' if ok else 'BAD'} {worst:.2e} {case}", flush=True)
print(f"{n - bad}/{n} within {TOL[torch.bfloat16]}")
