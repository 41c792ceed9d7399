"""Ad-hoc: full solves of configs 2/4/5 (one instance) on the GPU, with timing."""
import sys, os, time, logging
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200 import workloads
which = [int(a) for a in sys.argv[1:]] or [1, 4, 3]
for idx in which:
    prob, cfg = workloads.config(idx)
    st = {}
    hist = []
    t = time.perf_counter()
    cfg = pk.SolverConfig(**{**cfg.__dict__, "progress_every": 5000})
    res = pk.solve_lr_pd_sdp(prob, cfg, callback=lambda i: (hist.append(i), print("   ", i, flush=True)), stats=st)
    dt = time.perf_counter() - t
    print(f"cfg{idx+1}: {res.status} iters={res.iterations} obj={res.primal_objective:.10f} dobj={res.dual_objective:.10f} "
          f"rank_path={res.rank_path} res={res.final_residuals} wall={dt:.2f}s it/s={res.iterations/dt:.1f} stats={st}", flush=True)
