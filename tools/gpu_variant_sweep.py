"""Config-2 solve to tolerance with one library variant (PDSDP_B200_LIB):
one warm-up solve, one timed solve (CUDA events), iterations, passes and
matvecs per iteration, objective.  Used to compare eigensolver heuristics."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_05231_b200 import workloads
from paper_1810_05231_b200.device import DeviceBatch
from paper_1810_05231_b200.solver import operator_norm_on_device, run_lr_loop
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prob, cfg = workloads.config(idx)
if len(sys.argv) > 2:      # optional iteration cap (bounded sweeps of long configs)
    from paper_1810_05231_b200 import SolverConfig
    cfg = SolverConfig(**{**cfg.__dict__, "max_iter": int(sys.argv[2])})
batch = DeviceBatch([prob])
alpha = cfg.alpha_safety / operator_norm_on_device(batch, 0, cfg.seed)
stream = torch.cuda.ExternalStream(batch.stream_handle())
if len(sys.argv) <= 3:
    o = run_lr_loop(batch, 0, prob, cfg, alpha)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(stream)
o = run_lr_loop(batch, 0, prob, cfg, alpha)
e1.record(stream)
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 1e3
print(json.dumps({"lib": os.path.basename(os.environ.get("PDSDP_B200_LIB", "default")), "iters": o.it.k,
                  "time_s": round(t, 3), "it_per_s": round(o.it.k / t, 1), "status": o.status.value,
                  "rank_path": o.rank_path, "passes_per_it": round(o.eig_passes / o.it.k, 3),
                  "mv_per_it": round(o.eig_matvecs / o.it.k, 3), "res": o.res}))
