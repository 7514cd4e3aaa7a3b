import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2404_11068_b200 import dap, dap_bench, evoattn
class A: steps=3
dev = torch.device("cuda:0")
comm = dap.NcclDap()
pair = (dap.NcclDap(store_key="evo_dap_uid_pair"), torch.cuda.Stream()) if sys.argv[1] == "1" else None
t0 = time.time()
print("start", flush=True)
r = dap_bench.run_stack(torch, None, dap, evoattn, comm, pair, 1, 0, dev, int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[2]), A)
print(r, time.time() - t0, flush=True)
