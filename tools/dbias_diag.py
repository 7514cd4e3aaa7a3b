"""dbias error by query region for a 256 < L <= 384 call (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import numpy as np
from gpu_harness import run_case
import oracle
cases = [(4, 2, 384, 32, "ones"), (4, 2, 384, 32, "prefix"), (16, 1, 320, 32, "ones")]
if len(sys.argv) > 1:
    cases = [(384, 4, 384, 32, "prefix"), (384, 4, 384, 32, "ones"), (384, 4, 256, 32, "prefix")]
for (B, H, L, D, mask) in cases:
    errs, out, c = run_case(B, H, L, L, D, seed=11, bias="shared", mask=mask)
    rg = oracle.attn_bwd(c["q"], c["k"], c["v"], c["dout"], c["bias"], c["mask"], c["g"], c["scale"])
    db = out["dbias"].double().cpu().numpy()
    ref = rg["dbias"]
    scale = np.max(np.abs(ref))
    for name, sl in (("q<128", slice(0, 128)), ("128-255", slice(128, 256)), ("q>=256", slice(256, L))):
        if sl.start >= L:
            continue
        d_ = np.abs(db[:, sl] - ref[:, sl])
        e = np.max(d_) / scale
        i = np.unravel_index(np.argmax(d_), d_.shape)
        print(B, H, L, mask, name, f"{e:.2e}", "at", i, "ref", ref[:, sl][i], "got", db[:, sl][i])
    print("errs", {k: f"{v:.1e}" for k, v in errs.items()})
