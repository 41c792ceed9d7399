"""Per-step timeline of CTA 0 (flag bit 5 trace): run a config to iteration
K0, then trace one iteration and print (label, delta us) in order."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200 import workloads
idx, K0 = int(sys.argv[1]), int(sys.argv[2])
NT = int(sys.argv[3]) if len(sys.argv) > 3 else 1
prob, cfg = workloads.config(idx)
res = pk.solve_lr_pd_sdp(prob, pk.SolverConfig(**{**cfg.__dict__, "max_iter": K0}))
b = prob._device_cache["batch"]
r = res.rank_path[-1][1]
ypar = K0 & 1
names = {0: "prologue", 1: "op gram", 2: "op sync+issue+T", 3: "op apply/next", 4: "R2/R3 reduce", 5: "rotate",
         6: "dual", 7: "adjoint", 8: "G reduce", 9: "chol", 10: "tri_inv/M1", 11: "DHD+gemm", 12: "jacobi",
         13: "mbar wait", 14: "group compute", 20: "  cluster.sync done", 21: "  T read done", 24: "  epilogue done",
         25: "  fence+sync done", 26: "  gram_next done", 31: "plan done", 50: "dual: block red done",
         51: "P gram done", 53: "F_perp done", 54: "adjoint partials", 55: "G gram done", 57: "dense done", 99: "end"}
for t in range(NT):
    o = b.iterate([0], [r], [ypar], flags=[32])[0]; ypar ^= 1
    raw = b.debug(0)["raw"]
    tr = raw[400:400 + 4104]
    cnt = int(tr[4103])
    ev = tr[:2 * cnt].reshape(cnt, 2)
    print(f"iteration K0+{t}: r={r} passes {o[4]:.0f} matvecs {o[5]:.0f} block {o[11]:.0f} events {cnt}")
    t0 = ev[0, 1]
    prev = t0
    for lab, cyc in ev:
        print(f"  {1e-3*(cyc-t0)/1.965:8.2f} us  +{1e-3*(cyc-prev)/1.965:7.2f}  [{int(lab):2d}] {names.get(int(lab), '')}")
        prev = cyc
