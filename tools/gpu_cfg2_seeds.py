"""Config-2-shaped instances at other seeds (the replicas of bench.py --gpus N):
time to tolerance, iterations, rank path."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200 import workloads
for seed in [int(a) for a in sys.argv[1:]] or [1, 2, 3]:
    prob, cfg = workloads.config(1, seed)
    t = time.perf_counter()
    res = pk.solve_lr_pd_sdp(prob, cfg)
    dt = time.perf_counter() - t
    print(f"seed {seed}: {res.status.value} iterations {res.iterations} rank path {res.rank_path} "
          f"pobj {res.primal_objective:.6f} wall {dt:.2f} s ({res.iterations / dt:.0f} it/s)", flush=True)
    prob._device_cache["batch"].close()
