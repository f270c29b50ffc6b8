"""Group a kernel's SASS (ncu source page CSV) by execution count: shows how many instructions
run at each frequency (loop bodies) and their total share.   python tools/ncu_blocks.py src.csv [section]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
sec = int(sys.argv[2]) if len(sys.argv) > 2 else -1
secs, cur, hdr = [], None, None
for r in rows:
    if "Source" in r and "Instructions Executed" in r:
        hdr, cur = r, []
        secs.append((hdr, cur))
        continue
    if cur is not None and len(r) == len(hdr):
        cur.append(dict(zip(hdr, r)))
hdr, data = secs[sec]
groups = collections.defaultdict(list)
for d in data:
    try:
        groups[int(d["Instructions Executed"] or 0)].append(d)
    except ValueError:
        pass
tot = sum(k * len(v) for k, v in groups.items())
for k, v in sorted(groups.items(), key=lambda kv: -kv[0] * len(kv[1]))[:14]:
    ops = collections.Counter()
    for d in v:
        t = d["Source"].split()
        op = t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "?")
        ops[op.split(".")[0]] += 1
    print(f"exec {k:>10d} x {len(v):4d} instr = {100 * k * len(v) / tot:5.1f}%  " +
          " ".join(f"{o}:{c}" for o, c in ops.most_common(12)))
