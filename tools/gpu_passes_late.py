"""Pass plans (degree, active columns, residuals) late in a solve."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
np.set_printoptions(linewidth=220, precision=3)
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200 import workloads
idx, K0, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
prob, cfg = workloads.config(idx)
res = pk.solve_lr_pd_sdp(prob, pk.SolverConfig(**{**cfg.__dict__, "max_iter": K0}))
b = prob._device_cache["batch"]
r = res.rank_path[-1][1]
ypar = K0 & 1
for k in range(K):
    o = b.iterate([0], [r], [ypar])[0]; ypar ^= 1
    dbg = b.debug(0)
    if os.environ.get("COMPACT"):
        rows = dbg["passes"][: int(o[4])]
        print(f"it {k}: passes {o[4]:.0f} mv {o[5]:.0f} plans", [(int(row[0]), int(row[4] % 1000), f"{row[1]:.1e}") for row in rows],
              "kept res max %.1e tail res %.1e" % (dbg["res"][:r].max(), dbg["res"][r]))
        continue
    print(f"it {k}: passes {o[4]:.0f} mv {o[5]:.0f} conv {o[6]:.0f} blk {o[11]:.0f} lam {o[2]:.4e}")
    for row in dbg["passes"][: int(o[4]) + 1]:
        print("   m=%d maxres=%.2e last_bad=%d r=%d c0=%d b=%d bc=%d lo=%.3e cut=%.3e" % (
            row[0], row[1], row[2], row[3] // 1000, row[3] % 1000, row[4] // 1000, row[4] % 1000, row[5], row[6]))
    print("   theta", dbg["theta"][:int(o[11])])
    print("   res  ", dbg["res"][:int(o[11])])
