python - <<'PY'
import torch, sys
sys.path.insert(0, '.')
import bench
from paper_2404_11068_b200 import evoattn
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
r = bench.run_side_paths(torch, evoattn, dev, flush, 10, bench.measured_peaks())
for k, v in r.items(): print(k, {a: round(b, 4) for a, b in v.items()})
PY
