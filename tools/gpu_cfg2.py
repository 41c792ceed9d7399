"""Ad-hoc: config-2 solve with progress, for sizing bench.py."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200 import workloads
prob, cfg = workloads.config(1)
cfg = pk.SolverConfig(**{**cfg.__dict__, "progress_every": 1000, "max_iter": int(sys.argv[1]) if len(sys.argv) > 1 else 100000})
st = {}
t = time.perf_counter()
res = pk.solve_lr_pd_sdp(prob, cfg, callback=lambda i: print("   ", i, f"{time.perf_counter()-t:.1f}s", flush=True), stats=st)
dt = time.perf_counter() - t
print(f"cfg2: {res.status} iters={res.iterations} obj={res.primal_objective:.10f} dobj={res.dual_objective:.10f} rank_path={res.rank_path} res={res.final_residuals} wall={dt:.2f}s it/s={res.iterations/dt:.1f} stats={st}", flush=True)
