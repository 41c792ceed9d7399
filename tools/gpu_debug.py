"""Ad-hoc GPU diagnostics (not a test): op parity + config-1 iterate parity."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from conftest import problem_from_golden
from oracle import lrpdhg_oracle as orc
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200 import device, workloads
from paper_1810_05231_b200.solver import _device_batch

d = np.load("tests/golden/ops_small.npz")
for ci in range(5):
    pre = f"c{ci}_"
    prob = problem_from_golden(d, pre)
    n = prob.n
    try:
        mx = pk.apply_M(prob, pk.SymMatrix(n, d[pre + "X"]))
        mty = pk.apply_M_adjoint(prob, d[pre + "y"]).data
        on = pk.estimate_operator_norm(prob, 0)
        print(ci, "apply_M err", np.abs(mx - d[pre + "MX"]).max(), "adj err", np.abs(mty - d[pre + "MTy"]).max(),
              "opnorm", on, float(d[pre + "opnorm"]))
    except Exception as e:
        print(ci, "ops failed", repr(e))
    for r in (1, 3, n // 2, n):
        try:
            P, lam = pk.aproj_psd(pk.SymMatrix(n, d[pre + "S"]), r)
            print(f"   aproj n={n} r={r} err={np.abs(P.data - d[pre + f'aproj{r}']).max():.3e} lam={lam:.10f} ref={float(d[pre + f'aproj{r}_lam']):.10f}")
        except Exception as e:
            print("   aproj failed", r, repr(e))
sys.stdout.flush()
g = np.load("tests/golden/cfg1.npz")
prob, cfg = workloads.config(0)
for K in (1, 10, 100):
    c2 = pk.SolverConfig(**{**cfg.__dict__, "max_iter": K})
    st = {}
    t = time.perf_counter()
    res = pk.solve_lr_pd_sdp(prob, c2, stats=st)
    dt = time.perf_counter() - t
    X = res.X.data
    print(f"K={K} relX={np.linalg.norm(X - g[f'X{K}'])/np.linalg.norm(g[f'X{K}']):.3e} rely={np.linalg.norm(res.y - g[f'y{K}'])/np.linalg.norm(g[f'y{K}']):.3e} "
          f"res={res.final_residuals} ref={g[f'res{K}']} t={dt:.3f}s stats={st}")
    sys.stdout.flush()
st = {}
t = time.perf_counter()
res = pk.solve_lr_pd_sdp(prob, cfg, stats=st)
dt = time.perf_counter() - t
print("full:", res.status, res.iterations, res.primal_objective, float(g["pobj"]), res.rank_path, dt, st)
print("relX final", np.linalg.norm(res.X.data - g["X_final"]) / np.linalg.norm(g["X_final"]))
