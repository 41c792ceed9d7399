"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launch count, total time and share of the listed GPU time."""
import collections, csv, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID"]
per = collections.defaultdict(list)
for r in rows:
    per[r[4].split("(")[0]].append(float(r[-1]))
tot = sum(sum(v) for v in per.values())
print(f"{len(rows)} launches, {tot / 1e6:.3f} ms GPU time")
for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:45s} n={len(v):5d} total={sum(v) / 1e3:10.1f} us  mean={sum(v) / len(v) / 1e3:8.1f} us  share={sum(v) / tot:.3f}")
