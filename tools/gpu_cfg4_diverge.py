"""Where does the GPU trajectory of config 4 leave the reference's?  Compares
the combined residual every 100 iterations with the reference-to-tolerance
fixture's history (tests/golden/cfg4_full.npz)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200 import workloads
d = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "cfg4_full.npz"))
ref = {int(r[0]): r for r in d["history"]}
prob, cfg = workloads.config(3)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 3300
hist = []
res = pk.solve_lr_pd_sdp(prob, pk.SolverConfig(**{**cfg.__dict__, "max_iter": K, "progress_every": 100}),
                         callback=lambda i: hist.append(tuple(i)))
print("rank path", res.rank_path)
for h in hist:
    k = int(h[0])
    if k in ref:
        r = ref[k]
        print(f"k={k:5d} r={int(h[4])}/{int(r[4])} eps_c gpu {h[3]:.10e} ref {r[3]:.10e} rel diff {abs(h[3]-r[3])/r[3]:.2e}  obj rel diff {abs(h[5]-r[5])/max(abs(r[5]),1e-300):.2e}")
