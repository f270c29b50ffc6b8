"""Per-CUDA-source-line totals (instructions executed, stall samples) from an ncu source page
exported with --print-source cuda,sass (SASS rows follow their source line).

    ncu -i prof.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top_n]
"""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path, errors="replace")))
    hdr = None
    cur_file, cur_line, cur_src = "", None, ""
    acc = {}
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        if r[0] != "":
            cur_line, cur_src = r[0], r[1]
            continue
        try:
            ie = int(r[hdr.index("Instructions Executed")] or 0)
            ss = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        k = (cur_file, cur_line)
        a = acc.setdefault(k, [0, 0, cur_src])
        a[0] += ie
        a[1] += ss
    ti = sum(v[0] for v in acc.values()) or 1
    ts = sum(v[1] for v in acc.values()) or 1
    print(f"total warp instructions {ti:.4g}, samples {ts}")
    for (f, ln), (i, s, src) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{f}:{ln:>5} inst {100 * i / ti:5.1f}%  samples {100 * s / ts:5.1f}%  {src.strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
