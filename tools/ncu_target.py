"""Short config-2 solve (first N iterations) used as the ncu target: the
launch list and one --set full capture of the iteration kernel."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200 import workloads
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
N = int(sys.argv[2]) if len(sys.argv) > 2 else 400
prob, cfg = workloads.config(idx)
res = pk.solve_lr_pd_sdp(prob, pk.SolverConfig(**{**cfg.__dict__, "max_iter": N}))
print(res.status, res.iterations, res.rank_path, res.final_residuals)
