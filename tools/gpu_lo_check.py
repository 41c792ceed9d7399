"""How conservative is the Gershgorin lower bound of S = X_k - alpha Z_k that
sets the Chebyshev interval?  Solve config 2 to iteration K0 on the device,
then compare -alpha * Gershgorin(Z) with the true lambda_min(S) (scipy)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as sla
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200 import workloads
from paper_1810_05231_b200.layout import smat
idx = int(sys.argv[1]); K0s = [int(a) for a in sys.argv[2:]]
prob, cfg = workloads.config(idx)
for K0 in K0s:
    res = pk.solve_lr_pd_sdp(prob, pk.SolverConfig(**{**cfg.__dict__, "max_iter": K0}))
    alpha = pk.step_size(prob, cfg)
    Z = smat(prob.C.data if hasattr(prob.C, "data") else prob.C) + smat(pk.apply_M_adjoint(prob, res.y).data)
    X = smat(res.X.data)
    g = np.max(np.sum(np.abs(Z), axis=1))
    zmax = sla.eigsh(sp.csr_matrix(Z), k=1, which="LA", return_eigenvectors=False)[0]
    smin = np.linalg.eigvalsh(X - alpha * Z)[0]
    print(f"K0={K0} r={res.rank_path[-1][1]}: Gershgorin lo={-alpha*g:.4f}  -alpha*lmax(Z)={-alpha*zmax:.4f}  lambda_min(S)={smin:.4f}")
