"""Copy the evidence of one ncu --set full capture into profiles/: the key metrics (JSON, the file
bench.py reads for roofline.traffic), the details page (CSV) and the SASS opcode summary.

    python tools/save_profile.py gpurun_out/prof.ncu-rep profiles/r01/ncu_full_bm_box_c5
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__cycles_elapsed.avg.per_second"]


def main(rep, out, kernel_regex=None):
    """rep: an .ncu-rep, or the prefix of CSV exports made on the GPU box by tools/prof_f.sh
    (<prefix>_raw.csv, <prefix>_details.csv, <prefix>_src.csv[.gz] with --print-source cuda,sass)."""
    if not rep.endswith(".ncu-rep"):
        return main_csv(rep, out, kernel_regex)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    sel = [r for r in rows[2:] if kernel_regex is None or kernel_regex in r[hdr.index("Kernel Name")]]
    vals = sel[-1]
    m = {"kernel": vals[hdr.index("Kernel Name")]}
    for k in KEYS:
        if k in hdr:
            m[k] = {"value": vals[hdr.index(k)], "unit": units[hdr.index(k)]}
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(vals[i])
            except ValueError:
                pass
    m["stalls_per_issue_active"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:10])
    json.dump(m, open(out + "_metrics.json", "w"), indent=1)
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    open(out + "_details.csv", "w").write(det)
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    open("/tmp/_src.csv", "w").write(src)
    summ = subprocess.run([sys.executable, "tools/ncu_sass_summary.py", "/tmp/_src.csv", "30"],
                          capture_output=True, text=True).stdout
    blocks = subprocess.run([sys.executable, "tools/ncu_blocks.py", "/tmp/_src.csv"], capture_output=True, text=True).stdout
    open(out + "_sass_summary.txt", "w").write(summ + "\n\nby execution count (loop bodies):\n" + blocks)
    print(json.dumps(m, indent=1)[:1500])


def main_csv(prefix, out, kernel_regex=None):
    import gzip
    import os
    raw = open(prefix + "_raw.csv").read()
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    sel = [r for r in rows[2:] if kernel_regex is None or kernel_regex in r[hdr.index("Kernel Name")]]
    vals = sel[-1]
    m = {"kernel": vals[hdr.index("Kernel Name")]}
    for k in KEYS:
        if k in hdr:
            m[k] = {"value": vals[hdr.index(k)], "unit": units[hdr.index(k)]}
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(vals[i])
            except ValueError:
                pass
    m["stalls_per_issue_active"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:10])
    json.dump(m, open(out + "_metrics.json", "w"), indent=1)
    if os.path.exists(prefix + "_details.csv"):
        open(out + "_details.csv", "w").write(open(prefix + "_details.csv").read())
    src = prefix + "_src.csv"
    if os.path.exists(src + ".gz"):
        open("/tmp/_src.csv", "w").write(gzip.open(src + ".gz", "rt").read())
        src = "/tmp/_src.csv"
    if os.path.exists(src):
        summ = subprocess.run([sys.executable, "tools/ncu_sass_summary.py", src, "30"], capture_output=True,
                              text=True).stdout
        lines = subprocess.run([sys.executable, "tools/ncu_lines.py", src, "40"], capture_output=True, text=True).stdout
        open(out + "_sass_summary.txt", "w").write(summ + "\n\nby CUDA source line:\n" + lines)
    print(json.dumps(m, indent=1)[:1500])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
