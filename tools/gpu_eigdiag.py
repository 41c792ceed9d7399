"""Ad-hoc: per-iteration eigensolver diagnostics for a config."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
np.set_printoptions(linewidth=200, precision=3)
from paper_1810_05231_b200 import workloads
from paper_1810_05231_b200.device import DeviceBatch
from paper_1810_05231_b200.solver import operator_norm_on_device
from paper_1810_05231_b200.config import RankController
idx = int(sys.argv[1]); K = int(sys.argv[2]); r = int(sys.argv[3]) if len(sys.argv) > 3 else None
prob, cfg = workloads.config(idx)
b = DeviceBatch([prob])
alpha = cfg.alpha_safety / operator_norm_on_device(b, 0, 0)
b.set_alpha(0, alpha); b.reset(0, 0.0)
r = r or cfg.initial_rank
ypar = 0
t = time.perf_counter()
for k in range(1, K + 1):
    o = b.iterate([0], [r], [ypar])[0]; ypar ^= 1
    if k <= 5 or k % max(1, K // 12) == 0:
        d = b.debug(0)
        npass = int(o[4])
        print(f"k={k} eps=({o[0]:.4e},{o[1]:.4e}) lam={o[2]:.4e} passes={npass} matvecs={int(o[5])} conv={int(o[6])} blk={int(o[11])}")
        for p in range(32):
            if not d["passes"][p].any(): break
            print("    pass", p, d["passes"][p])
        bb = int(o[11])
        print("    theta", d["theta"][:bb]); print("    res", d["res"][:bb])
print("time", time.perf_counter() - t)
