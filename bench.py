#!/usr/bin/env python
"""bench.py — PDHG iterations/s and time-to-1e-4 residual on BASELINE.json
configs[1]: n=2000 Max-Cut SDP (G(2000, 0.01), +-1 weights, seed 0), FP64.

A step is one complete LR-PD-SDP solve to the reference's relative 1e-4 rule
(lowrank.py:153-161).  `value` = PDHG iterations / device time of the solve
loop with the problem already resident in HBM (CUDA events on the library's
stream, L2 flushed between steps).  `e2e` = the same metric through the
public drop-in API `solve_lr_pd_sdp(prob, config)` from host data: problem
upload and re-indexing, operator-norm estimate, the loop, the final X / y
download (host wall clock around synchronised calls).

--impl reference times the reference algorithm's CPU implementation (the
numpy/scipy oracle port, oracle/lrpdhg_oracle.py; the reference itself is pure
Python and cannot travel to the GPU box) on this host's cores, each step a
bounded sample of iterations of the same workload.

Multi-GPU (one process per GPU; `--gpus N` re-executes itself under
torch.distributed.run when no launcher set WORLD_SIZE): every rank solves its
own seeded instance of the workload (seed = rank; instances are independent,
no data-path collective, "scaling": "weak"); per-instance results are gathered
with NCCL all_gather and the time is the max over ranks.  Every run also
measures, once, BASELINE config 5 as a batch (`"batch"` in the JSON line):
`--batch-instances` independent n=1000 Max-Cut SDPs sharded over the N ranks
(strong scaling), per-instance results gathered with one NCCL all_gather.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PDHG iterations/s and time-to-1e-4 residual, n=2000 Max-Cut SDP, FP64"
WORKLOADS = {
    "cfg1": (0, "maxcut_n100_p0.1_unit_r5"),
    "cfg2": (1, "maxcut_n2000_p0.01_pm1_r10"),
    "cfg4": (3, "sensor_n1002_d2_r0.1"),
    "cfg5": (4, "maxcut_n1000_p0.02_pm1_r1"),
}
FP64_DMMA_TFLOPS = 37.1   # measured on this pool's B200 (profiles/r01_fp64_cluster_probe.txt)
# dram__bytes_read.sum + dram__bytes_write.sum of one iteration at rank 20 from the
# last committed `ncu --set full` capture of the iteration kernel (archived, per commit)
ARCHIVED_TRAFFIC = (3558656, "profiles/r02_iterate_kernel_ncu_raw_r20.csv (archived capture)")


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# Share of a config-2 solve's iterations spent at each target rank (rank path
# [(0, 10), (k1, 20)] of the solve to tolerance; tests/golden/cfg2_full.npz when
# the reference-to-tolerance fixture is present, else the GPU solve's own path).
# rank paths of the solves to tolerance measured on the B200 (used by the
# reference arm when the reference-to-tolerance fixture is not in the tree)
MEASURED_RANK_PATHS = {1: ([(0, 10), (24118, 20)], 30920)}


def rank_shares(idx: int, fallback=None):
    path = os.path.join(ROOT, "tests", "golden", f"cfg{idx + 1}_full.npz")
    try:
        d = np.load(path)
        rp, iters = d["rank_path"], int(d["iters"])
    except (OSError, KeyError, ValueError):
        if fallback is None:
            fallback = MEASURED_RANK_PATHS.get(idx)
        if fallback is None:
            return None
        rp, iters = np.asarray(fallback[0]), int(fallback[1])
    shares = {}
    for q in range(len(rp)):
        k0 = int(rp[q][0])
        k1 = int(rp[q + 1][0]) if q + 1 < len(rp) else iters
        shares[int(rp[q][1])] = shares.get(int(rp[q][1]), 0.0) + (k1 - k0) / max(1, iters)
    return shares


def oracle_stamps(prob, cfg, iters: int, alpha: float | None = None, initial_rank: int | None = None):
    """Per-iteration completion times of `iters` iterations of the CPU oracle
    (the reference algorithm): callback with progress_every=1."""
    from oracle import lrpdhg_oracle as orc
    from paper_1810_05231_b200.config import SolverConfig
    stamps = [time.perf_counter()]
    over = {"progress_every": 1, "max_iter": iters, "time_limit_s": 1e9}
    if initial_rank is not None:
        over["initial_rank"] = initial_rank
    c = SolverConfig(**{**cfg.__dict__, **over})
    orc.solve_lr(prob, c, progress=lambda info: stamps.append(time.perf_counter()),
                 alpha=alpha, stop_after=iters)
    return np.diff(np.asarray(stamps))


def cpu_reference(prob, cfg, shares, alpha=None, span=(100, 200), span_hi=(20, 50), with_cfg1=True):
    """The CPU baseline of SURVEY 8(d) on this host: setup time (stacked CSR +
    operator norm), median s/iteration over iterations span[0]..span[1] of the
    solve at its initial rank, the same over span_hi of a solve started at each
    later rank of the workload's rank path, the rank-weighted iterations/s, and
    the config-1 time to tolerance."""
    from oracle import lrpdhg_oracle as orc
    from paper_1810_05231_b200 import workloads
    t = time.perf_counter()
    M = orc.stacked_csr(prob)
    t_csr = time.perf_counter() - t
    t = time.perf_counter()
    sigma = orc.op_norm(M, cfg.seed)
    t_norm = time.perf_counter() - t
    if alpha is None:
        alpha = cfg.alpha_safety / sigma
    ranks = sorted(shares) if shares else [cfg.initial_rank]
    per_rank = {}
    for q, r in enumerate(ranks):
        lo, hi = span if q == 0 else span_hi
        dt = oracle_stamps(prob, cfg, hi, alpha=alpha, initial_rank=r)
        per_rank[r] = float(np.median(dt[lo:hi]))
    w = shares or {ranks[0]: 1.0}
    s_per_it = sum(w[r] * per_rank[r] for r in ranks)
    out = {"value": 1.0 / s_per_it, "unit": "iterations/s", "cores": os.cpu_count(), "kind": "port",
           "cpu_model": cpu_model(), "setup_s": {"stacked_csr": t_csr, "operator_norm": t_norm},
           "median_s_per_iteration": {str(r): per_rank[r] for r in ranks},
           "rank_shares": {str(r): w[r] for r in ranks},
           "sample": (f"numpy/scipy oracle port (OpenBLAS, ARPACK) on all host threads: median s/iteration "
                      f"over iterations {span[0]}-{span[1]} at the initial rank and over {span_hi[0]}-{span_hi[1]} "
                      f"of a solve started at each later rank of the rank path, weighted by the share of the "
                      f"solve's iterations at each rank")}
    if with_cfg1:
        p1, c1 = workloads.config(0)
        t = time.perf_counter()
        r1 = orc.solve_lr(p1, c1)
        out["cfg1_time_to_tol_s"] = time.perf_counter() - t
        out["cfg1_iterations"] = int(r1.iterations)
    return out


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm's CPU implementation (oracle
    port) on this host's cores.  A step = ref-iters-per-step iterations of the
    continuing solve at the initial rank plus the same number at each later
    rank of the workload's rank path; value = rank-weighted iterations/s over
    the timed steps (the GPU arm's value averages over the same rank mix)."""
    if rank != 0:
        return 0
    from paper_1810_05231_b200 import workloads
    idx, wname = WORKLOADS[args.workload]
    prob, cfg = workloads.config(idx, seed=0)
    shares = rank_shares(idx) or {cfg.initial_rank: 1.0}
    ranks = sorted(shares)
    per_step = args.ref_iters_per_step
    burn = max(args.warmup * per_step, args.ref_burn_in)
    total = burn + args.steps * per_step
    t_rank = {}
    for q, r in enumerate(ranks):
        b = burn if q == 0 else max(args.warmup * per_step, args.ref_burn_in // 5)
        dt = oracle_stamps(prob, cfg, b + args.steps * per_step, initial_rank=r)
        t_rank[r] = float(np.median(dt[b:]))
    s_per_it = sum(shares[r] * t_rank[r] for r in ranks)
    value = 1.0 / s_per_it
    cores = os.cpu_count()
    its = args.steps * per_step
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "iterations/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * s_per_it * per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE recipe)",
        "config": {"workload": wname,
                   "steps_are": f"{per_step} PDHG iterations of a continuing solve at each rank of the rank path",
                   "threads": cores, "cpu_model": cpu_model(), "burn_in_iterations": burn,
                   "s_per_iteration_by_rank": {str(r): t_rank[r] for r in ranks},
                   "rank_shares": {str(r): shares[r] for r in ranks}},
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": cores, "kind": "port",
                         "sample": f"median s/iteration over {its} timed LR-PDHG iterations per rank (after {burn} burn-in "
                                   f"iterations at the initial rank) of {wname} with numpy/scipy (OpenBLAS, ARPACK) on "
                                   f"all host threads, weighted by the solve's iteration share at each rank"},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def flush_l2(torch, stream):
    buf = getattr(flush_l2, "buf", None)
    if buf is None:
        buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > 126 MB L2
        flush_l2.buf = buf
    with torch.cuda.stream(stream):
        buf.fill_(1.0)


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1810_05231_b200 import SolverConfig, solve_lr_pd_sdp, workloads
    from paper_1810_05231_b200.device import DeviceBatch
    from paper_1810_05231_b200.layout import packed_length
    from paper_1810_05231_b200.solver import operator_norm_on_device, run_lr_loop

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    idx, wname = WORKLOADS[args.workload]
    prob, cfg = workloads.config(idx, seed=rank)
    batch = DeviceBatch([prob])
    alpha = cfg.alpha_safety / operator_norm_on_device(batch, 0, cfg.seed)
    stream = torch.cuda.ExternalStream(batch.stream_handle())

    def one_solve():
        return run_lr_loop(batch, 0, prob, cfg, alpha)

    for _ in range(args.warmup):
        o = one_solve()
    # ---- timed region: device-resident solves ----
    batch.set_timing(True)
    times, iters, outcomes = [], [], []
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            flush_l2(torch, stream)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            o = one_solve()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
            iters.append(o.it.k)
            outcomes.append(o)
    ktimes = batch.kernel_times()
    batch.set_timing(False)
    t_loop = sum(times)
    it_tot = sum(iters)
    # max over ranks, iterations summed
    t_all, it_all = t_loop, it_tot
    gathered = None
    o = outcomes[-1]
    final = torch.tensor([float(o.it.k), o.res[0], o.res[1], o.res[2], float(o.controller.r),
                          1.0 if o.status.value == "optimal" else 0.0], dtype=torch.float64,
                         device="cuda")
    if world > 1:
        tt = torch.tensor([t_loop, float(it_tot)], dtype=torch.float64, device="cuda")
        lst = [torch.zeros_like(tt) for _ in range(world)]
        dist.all_gather(lst, tt)
        t_all = max(float(x[0]) for x in lst)
        it_all = sum(float(x[1]) for x in lst)
        glist = [torch.zeros_like(final) for _ in range(world)]
        dist.all_gather(glist, final)          # per-instance results over NCCL
        gathered = [g.tolist() for g in glist]
    value = it_all / t_all * (args.steps and 1)
    # ---- e2e: public API from host data ----
    e2e_times, e2e_iters = [], []
    h2d = d2h = 0
    for _ in range(args.steps):
        p2, c2 = workloads.config(idx, seed=rank)
        indptr, ridx, rval = p2.stacked_arrays()
        torch.cuda.synchronize()
        t = time.perf_counter()
        res = solve_lr_pd_sdp(p2, c2)
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t)
        e2e_iters.append(res.iterations)
        b2 = p2._device_cache["batch"]
        nT = b2.info(0)["t_space"]
        h2d = (p2.C.data.nbytes + indptr.nbytes + ridx.nbytes + rval.nbytes + p2.b.nbytes +
               p2.h.nbytes + 8 * nT + res.iterations * 16 * 2)
        d2h = (8 * packed_length(p2.n) * (1 + len(res.checkpoints)) + res.y.nbytes *
               (1 + len(res.checkpoints)) + res.iterations * 16 * 8)
        b2.close()
        p2._device_cache.clear()
    e2e_rate = sum(e2e_iters) / sum(e2e_times)
    if world > 1:
        tt = torch.tensor([sum(e2e_times), float(sum(e2e_iters))], dtype=torch.float64, device="cuda")
        lst = [torch.zeros_like(tt) for _ in range(world)]
        dist.all_gather(lst, tt)
        e2e_rate = sum(float(x[1]) for x in lst) / max(float(x[0]) for x in lst)
    # ---- roofline: algorithmic bytes/flops of one iteration
    #      of the reference's dense formulation, per iteration's launches ----
    n = prob.n
    r = o.controller.r
    it_ms = ktimes["iterate_ms"] / max(1, ktimes["iterations"])
    t_it = it_ms * 1e-3
    mv = sum(x.eig_matvecs for x in outcomes) / max(1, it_tot)
    kb = min(r + 1, n)
    b = min(n, 64, ((kb + 1 + 1) // 2) * 2)   # block_for(): one guard column, rounded to 2
    ip, _, _ = prob.stacked_arrays()
    nnz, mp = int(ip[-1]), prob.m + prob.p
    B = 6551.7
    try:
        B = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except (OSError, ValueError, KeyError):
        pass
    B *= 1e9
    P = FP64_DMMA_TFLOPS * 1e12
    nn = 8.0 * n * n
    phases = [(3 * nn, 0.0),                                       # K2: read X, C; write S
              (mv * (nn + 16.0 * n * b), mv * 2.0 * n * n * b),     # K3: p_pass x S.V
              (0.0, 6.0 * mv * n * b * b),                          # K4/K6: Gram / rotations
              (2 * nn, 2.0 * n * n * r),                            # K7/K10: write X+, read X_k
              (12.0 * nnz + 32.0 * mp, 0.0)]                        # K8/K9: dual step
    algo_bytes = sum(ph[0] for ph in phases)
    algo_flops = sum(ph[1] for ph in phases)
    t_roof = sum(max(by / B, fl / P) for by, fl in phases)
    achieved = algo_bytes / t_it / 1e9
    roof = {"kernel": "lrpdhg_iterate_kernel (one launch = one PDHG iteration, residuals included)",
            "bound": "hbm", "achieved": achieved, "peak": B / 1e9, "unit": "GB/s", "frac": achieved / (B / 1e9),
            # dram__bytes_read.sum + dram__bytes_write.sum of one iteration-kernel
            # launch = one iteration at the final rank (ncu --set full; 2067456 at
            # rank 10): the iterate stays L2-resident, the kernel is latency-bound
            # archived figure of that capture (not re-measured by this run)
            "traffic": ARCHIVED_TRAFFIC[0], "traffic_source": ARCHIVED_TRAFFIC[1],
            "limiter": "latency: cross-CTA synchronisation inside one cluster (the factored iterate stays in "
                       "L2/shared memory, so measured DRAM traffic is ~1% of the dense formulation's bytes)",
            "peak_source": "MEASURED_PEAKS.json hbm_gbs",
            "algorithmic_bytes_per_iteration": algo_bytes, "algorithmic_flops_per_iteration": algo_flops,
            "basis": f"SURVEY 8(d) dense formulation, n={n}, b={b}, p_pass={mv:.2f}, r={r}",
            "t_roof_us": 1e6 * t_roof, "frac_sum_phase": t_roof / t_it,
            "fp64_achieved_tflops": algo_flops / t_it / 1e12, "fp64_peak_tflops": FP64_DMMA_TFLOPS}
    roof.update({"iterate_kernel_us": 1e3 * it_ms,
                 "loop_us_per_iteration": 1e6 * t_loop / max(1, it_tot)})
    # ---- CPU baseline (rank 0, N = 1) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # in a fresh interpreter (no CUDA context, no torch thread pools): the
        # same environment as the --impl reference arm
        leg = subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-leg", "--workload", args.workload,
                              "--cpu-iters", str(args.cpu_iters)], capture_output=True, text=True)
        try:
            cpu = json.loads([ln for ln in leg.stdout.splitlines() if ln.startswith("{")][-1])
        except (IndexError, ValueError):
            cpu = {"error": (leg.stderr or leg.stdout)[-400:]}
    # ---- BASELINE config 5 as one batch over the ranks, measured once ----
    batch.close()
    brec = None
    if args.batch_instances > 0:
        brec = batch_record(args, rank, world, local_rank, args.batch_instances, steps=1, warmup=0)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "iterations/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE recipe; each rank its own instance, seed = rank)",
            "config": {"workload": wname, "step": "one full LR-PD-SDP solve to eps_tol=1e-4 (relative)",
                       "iterations_per_solve": iters, "time_to_tol_s": times,
                       "l2": "flushed (256 MB write) before every timed step",
                       "parallelism": f"replicas x{world}", "final_rank": r,
                       "eig_matvecs_per_iter": sum(x.eig_matvecs for x in outcomes) / max(1, it_tot),
                       "eig_passes_per_iter": sum(x.eig_passes for x in outcomes) / max(1, it_tot),
                       "status": o.status.value},
            "e2e": {"value": e2e_rate, "unit": "iterations/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "time_to_tol_s": e2e_times},
            "gpu_launches": int(ktimes["launches"]),
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        if gathered is not None:
            line["per_instance"] = gathered
        if brec is not None:
            line["batch"] = brec
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def batch_record(args, rank, world, local_rank, count, steps, warmup):
    """BASELINE config 5: `count` independent Max-Cut instances (n=1000,
    p=0.02, +-1, seeds 0..count-1) sharded over the ranks, each rank solving
    its block as one resident batch; per-instance results gathered with one
    NCCL all_gather.  Returns the record (rank 0) -- value = instance-iterations
    of all ranks / max rank time.  The process group must exist when world > 1."""
    import torch
    import torch.distributed as dist
    from paper_1810_05231_b200 import workloads
    from paper_1810_05231_b200.device import DeviceBatch
    from paper_1810_05231_b200.distributed import gather_summaries, shard, summarize
    from paper_1810_05231_b200.solver import _result, operator_norm_on_device, run_lr_batch

    mine = shard(count, rank, world)
    probs, cfg = [], None
    for i in mine:
        p, cfg = workloads.config(4, seed=i)
        probs.append(p)
    if cfg is None:
        _, cfg = workloads.config(4, seed=0)
    times, iters, launches, results = [], [], 0, []
    clk = None
    if probs:
        batch = DeviceBatch(probs)
        alphas = [cfg.alpha_safety / operator_norm_on_device(batch, j, cfg.seed) for j in range(len(probs))]
        stream = torch.cuda.ExternalStream(batch.stream_handle())
        for _ in range(warmup):
            run_lr_batch(batch, list(range(len(probs))), cfg, alphas)
        batch.set_timing(True)
    with ClockSampler(local_rank) as clk:
        for _ in range(steps):
            if probs:
                flush_l2(torch, stream)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            if not probs:
                times.append(0.0)
                iters.append(0)
                continue
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            outs = run_lr_batch(batch, list(range(len(probs))), cfg, alphas)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
            iters.append(sum(o.it.k for o in outs))
    if probs:
        launches = batch.kernel_times()["launches"]
        batch.set_timing(False)
        results = [_result(p, cfg, o, a, 0.0) for p, o, a in zip(probs, outs, alphas)]
        batch.close()
    local = summarize(results)
    t_local, it_local = sum(times), float(sum(iters))
    if world > 1:
        full = gather_summaries(local, count, rank, world, device=torch.device("cuda", local_rank))
        tt = torch.tensor([t_local, it_local], dtype=torch.float64, device="cuda")
        lst = [torch.zeros_like(tt) for _ in range(world)]
        dist.all_gather(lst, tt)
        t_ranks = [float(x[0]) for x in lst]
        t_all = max(t_ranks)
        it_all = sum(float(x[1]) for x in lst)
    else:
        full, t_all, it_all, t_ranks = local, t_local, it_local, [t_local]
    if rank != 0:
        return None
    ok = int(np.sum(full[:, 7] == 0))
    return {
        "metric": "PDHG instance-iterations/s, batched n=1000 Max-Cut SDPs (BASELINE config 5), FP64",
        "value": it_all / t_all, "unit": "instance-iterations/s", "n_gpus": world,
        "steps": steps, "warmup": warmup, "ms_per_step": 1e3 * t_all / steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE recipe, seeds 0..count-1)",
        "config": {"workload": f"maxcut_n1000_p0.02_pm1_x{count}", "instances": count,
                   "parallelism": f"instances sharded over {world} GPU(s), NCCL all_gather of results",
                   "optimal": ok, "mean_iterations": float(np.mean(full[:, 5])),
                   "max_iterations": float(np.max(full[:, 5])),
                   "seconds_per_rank": t_ranks,
                   "objective_sum": float(np.sum(full[:, 0])),
                   "l2": "flushed (256 MB write) before every timed step"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }


def run_batch(args, rank, world, local_rank):
    """--workload cfg5: the config-5 batch as the benchmark's own steps."""
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = batch_record(args, rank, world, local_rank, args.instances, args.steps, args.warmup)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def launcher_check(rank, world):
    """Hidden self-test of the `--gpus N` launcher (CPU, gloo): every rank
    joins the group and rank 0 prints one JSON line with n_gpus = world."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([float(rank)], dtype=torch.float64)
    got = [t.clone()]
    if world > 1:
        got = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(got, t)
    if rank == 0:
        print(json.dumps({"launcher_check": True, "n_gpus": world, "ranks": [int(g.item()) for g in got]}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def spawn_ranks(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: re-execute under
    torch.distributed.run, one process per GPU, rendezvous on 127.0.0.1."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg2")
    ap.add_argument("--cpu-iters", type=int, default=100,
                    help="cpu_baseline: iterations in the median window after 100 burn-in iterations")
    ap.add_argument("--ref-iters-per-step", type=int, default=4)
    ap.add_argument("--ref-burn-in", type=int, default=100)
    ap.add_argument("--batch-instances", type=int, default=32,
                    help="config-5 instances of the once-per-run batch record (0 = skip)")
    ap.add_argument("--launcher-check", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--cpu-leg", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--instances", type=int, default=256, help="cfg5: number of instances")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        return spawn_ranks(args.gpus)
    if args.cpu_leg:      # the cpu_baseline leg of the GPU arm, in its own process
        from paper_1810_05231_b200 import workloads
        idx, _ = WORKLOADS[args.workload]
        prob, cfg = workloads.config(idx, seed=0)
        print(json.dumps(cpu_reference(prob, cfg, rank_shares(idx), span=(100, 100 + args.cpu_iters),
                                       span_hi=(20, 20 + max(10, args.cpu_iters // 3)))), flush=True)
        return 0
    rank, world, local_rank = env_rank()
    if args.launcher_check:
        return launcher_check(rank, world)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.workload == "cfg5":
        return run_batch(args, rank, world, local_rank)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
