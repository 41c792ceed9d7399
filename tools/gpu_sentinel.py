"""Diagnostic: effective-rank (sentinel) blocks on a small equipartition problem."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
np.set_printoptions(linewidth=200, precision=4)
from paper_1810_05231_b200 import workloads
from paper_1810_05231_b200.device import DeviceBatch
from paper_1810_05231_b200.solver import operator_norm_on_device
prob = workloads.equipartition_problem(150, 0.05, 2)
b = DeviceBatch([prob])
alpha = 0.99 / operator_norm_on_device(b, 0, 0)
b.set_alpha(0, alpha); b.reset(0, 0.0)
ypar = 0
for k in range(40):
    try:
        o = b.iterate([0], [150], [ypar])[0]
    except Exception as e:
        print("EXC", k, e)
        dbg = b.debug(0)
        for row in dbg["passes"]:
            if row[0] == 0 and row[1] == 0: continue
            print("  pass m=%d maxres=%.3e last_bad=%d r=%d c0=%d b=%d bc=%d lo=%.3e cut=%.3e" % (
                row[0], row[1], row[2], row[3] // 1000, row[3] % 1000, row[4] // 1000, row[4] % 1000, row[5], row[6]))
        print("  theta", dbg["theta"][:20]); print("  res", dbg["res"][:20])
        break
    ypar ^= 1
    dbg = b.debug(0)
    print(k, "passes", o[4], "mv", o[5], "conv", o[6], "lam", o[2], "blk", o[11], "eps", o[0], o[1], "theta", dbg["theta"][:4], "res", dbg["res"][:4])

print("---- through the solver")
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200.config import SolverConfig
for r0, K in ((100, 60), (150, 40), (70, 300)):
    cfg = SolverConfig(eps_tol=1e-4, max_iter=K, initial_rank=r0, window_ell=50, progress_every=1)
    hist = []
    try:
        res = pk.solve_lr_pd_sdp(prob, cfg, callback=lambda i: hist.append(i))
        print(r0, K, "ok", res.rank_path)
    except Exception as e:
        print(r0, K, "EXC after", len(hist), e)
        bb = prob._device_cache["batch"]
        dbg = bb.debug(0)
        for row in dbg["passes"]:
            if row[0] == 0 and row[1] == 0: continue
            print("  pass m=%d maxres=%.3e last_bad=%d r=%d c0=%d b=%d bc=%d lo=%.3e cut=%.3e" % (
                row[0], row[1], row[2], row[3] // 1000, row[3] % 1000, row[4] // 1000, row[4] % 1000, row[5], row[6]))
        print("  theta", dbg["theta"][:66]); print("  res", dbg["res"][:66])
