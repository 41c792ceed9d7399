"""Target of tools/gpu_sanitize.sh: short solves that exercise every cluster
path of lrpdhg_iterate_kernel (multicast all-gather with several row groups,
cluster reductions, rank doubling, inequality rows) and the dense path."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200 import workloads

which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "cluster"):
    prob = workloads.maxcut_problem(300, 0.05, 3, signed=True)      # cluster of 4 CTAs
    res = pk.solve_lr_pd_sdp(prob, pk.SolverConfig(eps_tol=1e-4, max_iter=12, initial_rank=5, window_ell=5))
    print("maxcut n=300:", res.status.value, res.iterations, res.rank_path, res.final_residuals)
if which in ("all", "cfg1"):
    prob, cfg = workloads.config(0)
    res = pk.solve_lr_pd_sdp(prob, pk.SolverConfig(**{**cfg.__dict__, "max_iter": 25}))
    print("config 1:", res.status.value, res.iterations, res.final_residuals)
if which in ("all", "dense"):
    rng = np.random.default_rng(5)
    R = rng.standard_normal((70, 70))
    P, lam = pk.aproj_psd(pk.SymMatrix.from_dense(0.5 * (R + R.T)), 70)
    print("dense aproj n=70:", lam, float(np.linalg.norm(P.data)))
