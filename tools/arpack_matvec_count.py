"""Matvec count of the reference's ARPACK call (symmat.py:189-199) on the
projection argument S = X - alpha (C + M^T y) at the END of a solve, from a
reference-to-tolerance fixture (tests/golden/cfgN_full.npz): the number the
device eigensolver's operator applications per iteration compare with.
CPU only; uses the oracle's restatement of the eigsh call."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from scipy.sparse.linalg import LinearOperator, eigsh
from oracle import lrpdhg_oracle as orc
from paper_1810_05231_b200 import workloads

name = sys.argv[1]                      # e.g. cfg4
idx = int(name[3]) - 1
seed = int(name.split("s")[1]) if "s" in name[4:] else 0
d = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", f"{name}_full.npz"))
prob, cfg = workloads.config(idx, seed)
n = prob.n
M = orc.stacked_csr(prob)
alpha = cfg.alpha_safety / orc.op_norm(M, cfg.seed)
X = orc.pack((d["X_V"] * d["X_lam"]) @ d["X_V"].T)
S = orc.unpack(X - alpha * (M.T @ d["y_final"] + prob.C.data), n)
r = int(d["rank_path"][-1][1])
k = min(r + 1, n)
c = float(np.abs(S).sum(axis=1).max())
A = S + c * np.eye(n)
count = [0]
def mv(x):
    count[0] += 1
    return A @ x
v0 = np.random.default_rng(orc.KRYLOV_SEED).standard_normal(n)
v0 /= np.linalg.norm(v0)
w, V = eigsh(LinearOperator((n, n), matvec=mv, dtype=float), k=k, which="LA", v0=v0,
             ncv=min(n, max(2 * k + 1, 20)), maxiter=orc.KRYLOV_MAXITER, tol=orc.KRYLOV_TOL)
print(f"{name}: n={n} r={r} k={k} ncv={min(n, max(2 * k + 1, 20))} ARPACK matvecs {count[0]} "
      f"(one n x n dgemv each); top eigenvalues {np.sort(w)[::-1] - c}")
