"""Summarise ncu reports / launch lists into profiles/ (markdown + json)."""
import csv
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"]


def report_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        res.append({"kernel": d["Kernel Name"], **{k: (d.get(k), u.get(k)) for k in KEYS}})
    return res


def launch_shares(csvfile):
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(csvfile) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rdr = csv.reader(lines)
    hdr = next(rdr)
    ki = hdr.index("Kernel Name")
    mi = hdr.index("Metric Name")
    vi = hdr.index("Metric Value")
    for r in rdr:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    s = sum(tot.values())
    return {k: {"launches": cnt[k], "total": tot[k], "share": tot[k] / s} for k in sorted(tot, key=lambda k: -tot[k])}


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "report":
        print(json.dumps(report_rows(sys.argv[2]), indent=1))
    else:
        print(json.dumps(launch_shares(sys.argv[2]), indent=1))
