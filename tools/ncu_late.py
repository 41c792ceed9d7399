"""ncu target late in a config-2 solve: run to iteration K0 (rank 20 after
24118), then profile ONE per-step launch of the iteration kernel between
cudaProfilerStart/Stop (ncu --profile-from-start off)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200 import workloads
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
K0 = int(sys.argv[2]) if len(sys.argv) > 2 else 29000
prob, cfg = workloads.config(idx)
res = pk.solve_lr_pd_sdp(prob, pk.SolverConfig(**{**cfg.__dict__, "max_iter": K0}))
b = prob._device_cache["batch"]
r = res.rank_path[-1][1]
ypar = K0 & 1
o = b.iterate([0], [r], [ypar])[0]
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
o = b.iterate([0], [r], [ypar ^ 1])[0]
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("rank", r, "passes", o[4], "matvecs", o[5])
