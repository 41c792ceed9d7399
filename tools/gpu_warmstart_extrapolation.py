"""How predictable is the eigenvector block from one iteration to the next?
Runs config idx to k0, k0+1, k0+2 (three solves, same trajectory), takes the
kept eigenvectors V of each iterate and compares the subspace angle between
span(V_k) and (a) span(V_{k-1}) -- the plain warm start -- with (b)
span(2 V_{k-1} - V_{k-2}), the linear extrapolation the kernel starts from,
and (c) the quadratic one, 3 V_{k-1} - 3 V_{k-2} + V_{k-3}."""
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
    for k in (k0, k0 + 1, k0 + 2, k0 + 3):
        c = SolverConfig(**{**cfg.__dict__, "max_iter": k})
        res = pk.solve_lr_pd_sdp(prob, c)
        r = res.rank_path[-1][1]
        lam, V = top(dense(res.X.data), r)
        if Vs:
            V = V * np.sign(np.sum(V * Vs[-1], axis=0))
        Vs.append(V)
    npos = int(np.sum(np.linalg.norm(Vs[3] - Vs[2], axis=0) < 0.5))      # columns tracked from step to step
    W = [V[:, :npos] for V in Vs]
    a = sin_angle(W[2], W[3]); b = sin_angle(2 * W[2] - W[1], W[3]); c = sin_angle(3 * W[2] - 3 * W[1] + W[0], W[3])
    pc = [np.linalg.norm(W[3][:, j] - W[2][:, j]) for j in range(npos)]
    pe = [np.linalg.norm(W[3][:, j] - 2 * W[2][:, j] + W[1][:, j]) for j in range(npos)]
    pq = [np.linalg.norm(W[3][:, j] - 3 * W[2][:, j] + 3 * W[1][:, j] - W[0][:, j]) for j in range(npos)]
    print(f"k0={k0} r={r} ({npos} tracked) sin(angle) warm start {a:.3e}  linear {b:.3e}  quadratic {c:.3e}")
    print("   per column |dV|   :", " ".join(f"{x:.1e}" for x in pc))
    print("   per column |d2V|  :", " ".join(f"{x:.1e}" for x in pe))
    print("   per column |d3V|  :", " ".join(f"{x:.1e}" for x in pq), flush=True)
