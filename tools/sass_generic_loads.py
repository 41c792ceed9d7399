"""Count generic (LD.E / ST.E) vs shared (LDS/STS) and global (LDG/STG)
accesses per source line of one kernel in `nvdisasm -g` output."""
import collections, re, sys
path, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cur = None; inside = False
cnt = collections.Counter(); tot = collections.Counter()
for l in open(path):
    if l.startswith("\t.text.") or l.startswith(".text."):
        inside = kern in l
    if re.match(r"^\s*\.section\s+\.text\.", l):
        inside = kern in l
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2))); continue
    for op in ("LD.E", "ST.E", "LDS", "STS", "LDG", "STG"):
        if re.search(r"\b" + re.escape(op) + r"\b", l):
            tot[op] += 1
            if op in ("LD.E", "ST.E"):
                cnt[(cur, op)] += 1
print(dict(tot))
for k, v in sorted(cnt.items(), key=lambda kv: -kv[1])[:top]:
    print(k, v)
