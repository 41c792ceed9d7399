"""How predictable is the eigenvector block from one iteration to the next?
Runs config idx to k0, k0+1, k0+2 (three solves, same trajectory), takes the
kept eigenvectors V of each iterate and compares the subspace angle between
span(V_k) and (a) span(V_{k-1}) -- the warm start the kernel uses -- with
(b) span(2 V_{k-1} - V_{k-2}), a linear extrapolation."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200 import workloads, SolverConfig

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
k0s = [int(a) for a in sys.argv[2:]] or [5000, 20000, 28000]
prob, cfg = workloads.config(idx)
n = prob.n
iu, ju = np.triu_indices(n)

def dense(Xp):
    w = np.array(Xp, dtype=float)
    w[iu != ju] /= np.sqrt(2.0)
    S = np.zeros((n, n)); S[iu, ju] = w; S[ju, iu] = w
    return S

def top(X, r):
    w, V = np.linalg.eigh(X)
    return w[::-1][:r], V[:, ::-1][:, :r]

def sin_angle(A, B):      # largest principal angle between span(A) and span(B)
    Qa, _ = np.linalg.qr(A); Qb, _ = np.linalg.qr(B)
    return np.linalg.norm(Qb - Qa @ (Qa.T @ Qb), 2)

for k0 in k0s:
    Vs, r = [], None
    for k in (k0, k0 + 1, k0 + 2):
        c = SolverConfig(**{**cfg.__dict__, "max_iter": k})
        res = pk.solve_lr_pd_sdp(prob, c)
        r = res.rank_path[-1][1]
        lam, V = top(dense(res.X.data), r)
        if Vs:
            V = V * np.sign(np.sum(V * Vs[-1], axis=0))
        Vs.append(V)
    a = sin_angle(Vs[1], Vs[2]); b = sin_angle(2 * Vs[1] - Vs[0], Vs[2])
    pc = [np.linalg.norm(Vs[2][:, j] - Vs[1][:, j]) for j in range(r)]
    pe = [np.linalg.norm(Vs[2][:, j] - 2 * Vs[1][:, j] + Vs[0][:, j]) for j in range(r)]
    print(f"k0={k0} r={r} sin(angle) warm start {a:.3e}  extrapolated {b:.3e}  ratio {a / b:.2f}")
    print("   per column |dV|   :", " ".join(f"{x:.1e}" for x in pc))
    print("   per column |d2V|  :", " ".join(f"{x:.1e}" for x in pe), flush=True)
