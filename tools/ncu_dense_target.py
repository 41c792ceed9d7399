"""ncu target for the dense-iterate path: one full projection (aproj_psd with
r = n) of a seeded n x n symmetric matrix -> dense_arg / jacobi_round /
eig_finalize / recon launches."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_05231_b200 as pk

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
rng = np.random.default_rng(3)
R = rng.standard_normal((n, n))
S = pk.SymMatrix.from_dense(0.5 * (R + R.T) / np.sqrt(n))
P, lam = pk.aproj_psd(S, n)
print("n", n, "lambda_min", lam, "||P||", float(np.linalg.norm(P.data)))
