"""Time of one dense-path iteration (full device eigendecomposition +
reconstruction + residuals) on a seeded n x n symmetric matrix, setup
excluded; sweeps = Jacobi sweeps of the eigendecomposition."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200.device import DeviceBatch, OUT_PASSES, OUT_LAMBDA
for n in [int(a) for a in sys.argv[1:]] or [1024, 2048]:
    rng = np.random.default_rng(3)
    R = rng.standard_normal((n, n))
    Sd = 0.5 * (R + R.T) / np.sqrt(n)
    prob = pk.SdpProblem(n=n, C=pk.SymMatrix.from_dense(-Sd), A=[pk.SparseRow(np.array([0]), np.array([0.0]))], b=np.zeros(1))   # a null row: the model wants one constraint
    batch = DeviceBatch([prob])
    batch.set_alpha(0, 1.0)
    batch.reset(0, 0.0)
    batch.dense_begin(0, False)
    t = time.perf_counter()
    out = batch.iterate_dense(0, n, 0)
    dt = time.perf_counter() - t
    w0 = np.linalg.eigvalsh(Sd)[0]
    print(f"n={n}: dense iteration {dt:.3f} s, {int(out[OUT_PASSES])} sweeps, lambda_min {out[OUT_LAMBDA]:.12f} vs {w0:.12f}", flush=True)
    batch.close()
