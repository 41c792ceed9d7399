"""Diagnostic: config 3 (equipartition n=5000) residual/rank trajectory on the GPU."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200 import workloads
prob, cfg = workloads.config(2)
every = int(sys.argv[1]) if len(sys.argv) > 1 else 100
cfg = pk.SolverConfig(**{**cfg.__dict__, "progress_every": every})
t = time.perf_counter()
try:
    res = pk.solve_lr_pd_sdp(prob, cfg, callback=lambda i: print(f"k={i[0]} ep={i[1]:.4e} ed={i[2]:.4e} ec={i[3]:.4e} r={i[4]} obj={i[5]:.6f} t={time.perf_counter()-t:.1f}", flush=True))
    print(res.status, res.iterations, res.rank_path)
except Exception as e:
    print("EXC", e, time.perf_counter() - t)
