"""Per-iteration time breakdown on a config (kernel CUDA events vs loop wall time)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1810_05231_b200 import workloads
from paper_1810_05231_b200.device import DeviceBatch
from paper_1810_05231_b200.solver import operator_norm_on_device
idx = int(sys.argv[1]); K = int(sys.argv[2]); r = int(sys.argv[3]) if len(sys.argv) > 3 else None
prob, cfg = workloads.config(idx)
b = DeviceBatch([prob])
print(b.info(0))
alpha = cfg.alpha_safety / operator_norm_on_device(b, 0, 0)
b.set_alpha(0, alpha); b.reset(0, 0.0)
r = r or cfg.initial_rank
ypar = 0
for k in range(20):
    b.iterate([0], [r], [ypar]); ypar ^= 1
b.set_timing(True)
t = time.perf_counter()
mv = ps = 0
pc = np.zeros(16)
for k in range(K):
    o = b.iterate([0], [r], [ypar])[0]; ypar ^= 1
    mv += o[5]; ps += o[4]
    pc += b.debug(0)["prof_cycles"]
dt = time.perf_counter() - t
kt = b.kernel_times()
print(f"n={prob.n} r={r} K={K}: loop {1e6*dt/K:.1f} us/iter; iterate kernel {1e3*kt['iterate_ms']/max(1,kt['iterations']):.1f} us; "
      f"residual kernel {1e3*kt['residual_ms']/K:.1f} us; matvecs/iter {mv/K:.2f} passes/iter {ps/K:.2f}")
names = ["prologue/epilogue", "op gram", "op cluster-reduce", "op apply", "R2 reduce, R3+assess+plan", "rotations+R2 gram", "dual step", "adjoint+epilogue",
         "chol", "tri_inv+M1", "DHD+gemms", "jacobi", "sort+B", "apply: staging issue", "apply: staging wait", "jacobi sweeps (count)"]
tot = pc[:15].sum()
for nm, c in zip(names[:15], pc[:15]):
    print(f"   {nm:22s} {c/K/1.9e3:8.1f} us/iter ({c/tot:.2f})")
print(f"   jacobi sweeps/iter {pc[15]/K:.2f}")
