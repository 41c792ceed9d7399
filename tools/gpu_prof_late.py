"""Phase breakdown late in a solve: run the solver to iteration K0, then profile K more iterations."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200 import workloads
idx, K0, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
prob, cfg = workloads.config(idx)
res = pk.solve_lr_pd_sdp(prob, pk.SolverConfig(**{**cfg.__dict__, "max_iter": K0}))
b = prob._device_cache["batch"]
r = res.rank_path[-1][1]
ypar = K0 & 1
print("rank_path", res.rank_path, "residuals", res.final_residuals)
b.set_timing(True)
t = time.perf_counter()
mv = ps = 0
pc = np.zeros(16)
b.debug(0)
for k in range(K):
    o = b.iterate([0], [r], [ypar])[0]; ypar ^= 1
    mv += o[5]; ps += o[4]
    pc += b.debug(0)["prof_cycles"]
dt = time.perf_counter() - t
kt = b.kernel_times()
print(f"n={prob.n} r={r} K0={K0} K={K}: loop {1e6*dt/K:.1f} us/iter; iterate kernel {1e3*kt['iterate_ms']/max(1,kt['iterations']):.1f} us; "
      f"residual kernel {1e3*kt['residual_ms']/K:.1f} us; matvecs/iter {mv/K:.2f} passes/iter {ps/K:.2f} block {o[11]}")
names = ["prologue/epilogue", "op gram", "op cluster-reduce", "op apply", "R2 reduce, R3+assess+plan", "rotations+R2 gram", "dual step", "adjoint+epilogue",
         "chol", "tri_inv+M1", "DHD+gemms", "jacobi", "sort+B", "apply: staging issue", "apply: staging wait", "jacobi sweeps (count)"]
tot = pc[:15].sum()
for nm, c in zip(names[:15], pc[:15]):
    print(f"   {nm:22s} {c/K/1.965e3:8.1f} us/iter ({c/tot:.2f})")
print(f"   jacobi sweeps/iter {pc[15]/K:.2f}")
