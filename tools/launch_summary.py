"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv): per-kernel share of time.
    python tools/launch_summary.py gpurun_out/launches.csv
"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"]
    m = re.search(r"(\w+)(<|\()", name.replace("void ", ""))
    k = m.group(1) if m else name[:40]
    agg[k][0] += 1
    agg[k][1] += float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':32s} {'launches':>8s} {'total_us':>12s} {'mean_us':>10s} {'share':>7s}")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:32s} {n:8d} {t:12.1f} {t / n:10.2f} {100 * t / tot:6.1f}%")
