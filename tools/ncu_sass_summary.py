"""Summarise an ncu source page (SASS view): instructions executed and stall samples by opcode,
and the hottest instruction addresses.

    ncu -i prof.ncu-rep --page source --csv > src.csv
    python tools/ncu_sass_summary.py src.csv [top_n]
"""
import collections
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    by_op = collections.defaultdict(lambda: [0, 0])
    tot_i = tot_s = 0
    for d in data:
        op = d["Source"].split()[0] if d["Source"].split() else "?"
        if op.startswith("@"):
            op = d["Source"].split()[1]
        op = op.split(".")[0]
        ie = int(d["Instructions Executed"] or 0)
        sm = int(d["Warp Stall Sampling (All Samples)"] or 0)
        by_op[op][0] += ie
        by_op[op][1] += sm
        tot_i += ie
        tot_s += sm
    print(f"total warp instructions {tot_i:.4g}, stall samples {tot_s}")
    for op, (ie, sm) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:25]:
        print(f"{op:12s} inst {ie:14d} ({100 * ie / max(tot_i, 1):5.1f}%)  samples {100 * sm / max(tot_s, 1):5.1f}%")
    print("\nhottest instructions by samples:")
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    for d in sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:top]:
        st = sorted(((int(d[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
        print(f'{d["Address"][-5:]} {int(d["Warp Stall Sampling (All Samples)"] or 0):7d} '
              f'{int(d["Instructions Executed"] or 0):12d}  {d["Source"][:60]:60s} {st}')


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
