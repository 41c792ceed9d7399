"""Summarise an ncu source page (cuda,sass) by CUDA line with stall breakdown."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None; cur = None; data = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split('/')[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr and len(r) > 5 and r[0] not in ("",) and r[2] == "-":
        try: smp = int(r[4])
        except ValueError: continue
        st = {hdr[i]: int(r[i]) for i in range(32, 49) if r[i].isdigit() and int(r[i]) > 0}
        data.append((smp, cur, r[0], r[1][:70], st))
tot = sum(d[0] for d in data)
print("total samples", tot)
for smp, f, l, src, st in sorted(data, key=lambda d: -d[0])[:top]:
    top3 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{smp:5d} {100*smp/tot:5.1f}% {f}:{l:5s} {src:70s} {' '.join(f'{k[6:]}={v}' for k, v in top3)}")
