"""Time of one full projection (dense-iterate path: full device
eigendecomposition) of a seeded n x n symmetric matrix."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_05231_b200 as pk
for n in [int(a) for a in sys.argv[1:]] or [1024, 2048]:
    rng = np.random.default_rng(3)
    R = rng.standard_normal((n, n))
    Sd = 0.5 * (R + R.T) / np.sqrt(n)
    S = pk.SymMatrix.from_dense(Sd)
    t = time.perf_counter()
    P, lam = pk.aproj_psd(S, n)
    dt = time.perf_counter() - t
    w = np.linalg.eigvalsh(Sd)
    ref = np.sqrt(np.sum(np.maximum(w, 0.0) ** 2))
    iu = np.triu_indices(n)
    print(f"n={n}: {dt:.3f} s (upload, re-indexing, eigendecomposition, download); lambda_min {lam:.12f} vs {w[0]:.12f}; "
          f"||P||_F rel err {abs(np.linalg.norm(P.data) - ref) / ref:.2e}", flush=True)
