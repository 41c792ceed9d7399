"""Per-CTA timelines of one iteration (flag bit 6): segment durations
between consecutive marks for every CTA of the cluster, with the slowest CTA."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200 import workloads
idx, K0 = int(sys.argv[1]), int(sys.argv[2])
nshow = int(sys.argv[3]) if len(sys.argv) > 3 else 60
prob, cfg = workloads.config(idx)
res = pk.solve_lr_pd_sdp(prob, pk.SolverConfig(**{**cfg.__dict__, "max_iter": K0}))
b = prob._device_cache["batch"]
C = b.info(0)["cluster"]
r = res.rank_path[-1][1]
o = b.iterate([0], [r], [K0 & 1], flags=[64])[0]
raw = b.debug(0)["raw"][4504:]
evs = []
for c in range(C):
    t = raw[c * 2048:(c + 1) * 2048]
    cnt = int(t[2047])
    evs.append(t[:2 * cnt].reshape(cnt, 2))
n = min(len(e) for e in evs)
print(f"r={r} C={C} events per CTA {[len(e) for e in evs]} passes {o[4]:.0f} matvecs {o[5]:.0f}")
labels = evs[0][:, 0]
print("first events (label, us from CTA start):", [(int(l), round((c - evs[0][0, 1]) / 1965.0, 2)) for l, c in evs[0][:4]])
same = all(np.array_equal(e[:n, 0], labels[:n]) for e in evs)
print("identical label sequences:", same)
tot = np.array([(e[n - 1, 1] - e[0, 1]) / 1965.0 for e in evs])
print("total us per CTA:", np.round(tot, 1))
lo = int(sys.argv[4]) if len(sys.argv) > 4 else 1
for i in range(max(1, lo), min(n, nshow)):
    d = np.array([(e[i, 1] - e[i - 1, 1]) / 1965.0 for e in evs])
    print(f"{i:3d} [{int(labels[i-1]):2d}->{int(labels[i]):2d}]  min {d.min():6.2f}  med {np.median(d):6.2f}  max {d.max():6.2f} (cta {d.argmax():2d})  cta0 {d[0]:6.2f}")

# aggregate: total CTA-0 time per transition (label_prev -> label)
import collections
agg = collections.defaultdict(lambda: [0, 0.0])
for i in range(1, n):
    key = (int(labels[i - 1]), int(labels[i]))
    dmax = max((e[i, 1] - e[i - 1, 1]) / 1965.0 for e in evs)
    agg[key][0] += 1
    agg[key][1] += (evs[0][i, 1] - evs[0][i - 1, 1]) / 1965.0
print("transition totals (CTA 0):")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k[0]:3d}->{k[1]:3d}  count {c:4d}  total {t:8.1f} us  mean {t / c:6.2f} us")
