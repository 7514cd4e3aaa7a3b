"""The bench contract on CPU: the reference arm (`bench.py --impl reference`, the fp64 oracle on
the host cores) prints ONE JSON line with the contract's keys, and the algorithmic work model
of DESIGN.md §5 (`bench.kernel_alg`, `bench.alg_flops`) matches its closed forms."""
import json
import os
import subprocess
import sys

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "3", "--ref-rows", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["metric"] == bench.METRIC
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


def test_work_model_closed_forms():
    B, H, L, D = 128, 8, 256, 32
    X, P = B * H * L * D, B * H * L * L
    assert bench.alg_flops(B, H, L, D) == 12.0 * P * D
    f, by, ex = bench.kernel_alg("fwd_bf16", B, H, L, D, True)
    assert f == 4.0 * P * D and ex == P
    assert by == 10.0 * X + 2 * H * L * L + B * L + 4 * B * H * L
    f, by, ex = bench.kernel_alg("bwd_fused", B, H, L, D, True)
    assert f == 8.0 * P * D and by == 14.0 * X + 8.0 * B * H * L + 3.0 * 2 * H * L * L + B * L
    # the block's four modules: 90.2 GFLOP
    tot = sum(bench.alg_flops(b, h, l, 32) for _, b, h, l, _ in bench.MODULES)
    assert abs(tot - 90.19e9) / 90.19e9 < 1e-3
