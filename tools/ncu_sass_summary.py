"""Summarise an ncu source page (SASS view): instructions executed and stall samples by opcode,
and the hottest instruction addresses, per kernel section of the CSV.

    ncu -i prof.ncu-rep --page source --csv --print-source sass > src.csv
    python tools/ncu_sass_summary.py src.csv [top_n]
"""
import collections
import csv
import sys


def summarise(hdr, data, top):
    by_op = collections.defaultdict(lambda: [0, 0])
    tot_i = tot_s = 0
    data = [d for d in data if d.get("Address", "") not in ("-", "")]  # (cuda,sass exports: SASS rows only)
    for d in data:
        try:
            ie = int(d.get("Instructions Executed") or 0)
            ss = int(d.get("Warp Stall Sampling (All Samples)") or 0)
        except ValueError:
            continue
        toks = d["Source"].split()
        op = toks[0] if toks else "?"
        if op.startswith("@") and len(toks) > 1:
            op = toks[1]
        op = op.split(".")[0]
        by_op[op][0] += ie
        by_op[op][1] += ss
        tot_i += ie
        tot_s += ss
    if tot_i == 0:
        return
    print(f"total warp instructions {tot_i:.4g}, stall samples {tot_s}")
    for op, (i, s) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:25]:
        print(f"{op:12s} inst {i:14d} ({100 * i / tot_i:5.1f}%)  samples {100 * s / max(tot_s, 1):5.1f}%")
    print("\nhottest instructions by samples:")
    def key(d):
        try:
            return -int(d.get("Warp Stall Sampling (All Samples)") or 0)
        except ValueError:
            return 0
    for d in sorted(data, key=key)[:top]:
        print(f"{d.get('Address', '?'):>8} {d.get('Warp Stall Sampling (All Samples)', ''):>6} "
              f"{d.get('Instructions Executed', ''):>12}  {d['Source'][:70]}")


def main(path, top=30):
    rows = list(csv.reader(open(path, errors="replace")))
    sections, cur, hdr = [], None, None
    for r in rows:
        if "Source" in r and "Instructions Executed" in r:
            hdr = r
            cur = []
            sections.append((hdr, cur))
            continue
        if cur is not None and len(r) == len(hdr):
            cur.append(dict(zip(hdr, r)))
    for i, (h, data) in enumerate(sections):
        print(f"===== kernel section {i}")
        summarise(h, data, top)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
