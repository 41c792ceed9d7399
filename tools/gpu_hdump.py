"""Dump projected RR matrices for offline Jacobi analysis."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1810_05231_b200 import workloads
from paper_1810_05231_b200.device import DeviceBatch
from paper_1810_05231_b200.solver import operator_norm_on_device
idx = int(sys.argv[1]); K = int(sys.argv[2])
prob, cfg = workloads.config(idx)
b = DeviceBatch([prob])
alpha = cfg.alpha_safety / operator_norm_on_device(b, 0, 0)
b.set_alpha(0, alpha); b.reset(0, 0.0)
ypar = 0; Hs = []
for k in range(K):
    fl = 16 if k >= K - 5 else 0
    b.iterate([0], [cfg.initial_rank], [ypar], [fl]); ypar ^= 1
    if fl: Hs.append(b.debug(0)["H"])
np.save("gpurun_out/hdump_cfg%d.npy" % (idx + 1), np.array(Hs))
print("saved", np.array(Hs).shape)
