"""Diagnostic: spectrum of S = X - alpha (C + M^T y) along config 3 (torch eigvalsh, test-only)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200 import workloads
from paper_1810_05231_b200.layout import smat
prob, cfg = workloads.config(2)
last = [0]
def cb(i):
    last[0] = i[0]
    print(f"k={i[0]} ec={i[3]:.5e} r={i[4]} obj={i[5]:.6f}", flush=True)
for K in [int(a) for a in sys.argv[1:]]:
    c = pk.SolverConfig(**{**cfg.__dict__, "max_iter": K, "progress_every": 250})
    try:
        st = {}
        res = pk.solve_lr_pd_sdp(prob, c, callback=cb, stats=st)
    except Exception as e:
        print("EXC at", last[0], e); continue
    import scipy.sparse as sp
    ip, ix, vv = prob.stacked_arrays()
    M = sp.csr_matrix((vv, ix, ip), shape=(ip.size - 1, prob.n * (prob.n + 1) // 2))
    alpha = st["alpha"]
    adj = M.T @ res.y
    S = res.X.data - alpha * (adj + prob.C.data)
    Sd = torch.tensor(smat(S), device="cuda")
    ev = torch.linalg.eigvalsh(Sd).cpu().numpy()[::-1]
    Xd = torch.tensor(res.X.to_dense(), device="cuda")
    xe = torch.linalg.eigvalsh(Xd).cpu().numpy()[::-1]
    print(f"K={K} rank_path={res.rank_path} npos(S)={int((ev > 0).sum())} rank(X)={int((xe > 1e-12 * xe[0]).sum())} "
          f"top={ev[:3]} ev[60:70]={ev[60:70]}", flush=True)
