"""Per-kernel achieved DRAM GB/s from an ncu csv with gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum (dense-path kernels)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "ID")
iname, imet, ival, iunit = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
per = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for r in rows:
    if len(r) <= ival or r[0] == "ID" or not r[0].isdigit():
        continue
    v = float(r[ival].replace(",", ""))
    u = r[iunit]
    if r[imet].startswith("dram__bytes"):
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    else:
        v *= {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}.get(u, 1e-9)
    k = r[iname].split("(")[0]
    per[k][r[imet]] += v
    if r[imet].startswith("gpu__time"):
        cnt[k] += 1
print(f"{'kernel':32s} {'launches':>8s} {'time ms':>10s} {'DRAM MB':>10s} {'GB/s':>8s}")
for k, m in sorted(per.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
    t = m["gpu__time_duration.sum"]
    b = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    print(f"{k:32s} {cnt[k]:8d} {1e3 * t:10.3f} {b / 1e6:10.1f} {b / t / 1e9 if t else 0:8.1f}")
