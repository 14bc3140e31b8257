"""Summaries of an `ncu --page source --csv --print-source cuda,sass` export and a `--page raw --csv`
export: headline metrics, stall reasons per issue, and the CUDA source lines with the most warp-stall
samples (mapped to the current source tree).

    python tools/ncu_lines.py raw.csv[.gz] src.csv[.gz] [top]"""
import csv
import gzip
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def opener(p):
    return gzip.open(p, "rt") if p.endswith(".gz") else open(p)


def raw_summary(path):
    rows = list(csv.reader(opener(path)))
    hdr = rows[0]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__block_size", "smsp__inst_executed.sum"]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(d["Kernel Name"][:90])
        print("  ", {k.split("__")[1][:28]: d.get(k) for k in keys})
        st = {h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(d[h])
              for h in hdr if re.match(r"smsp__average_warps_issue_stalled_.*_per_issue_active.ratio", h) and d[h]}
        print("   stalls/issue", {k: round(v, 2) for k, v in sorted(st.items(), key=lambda x: -x[1]) if v > 0.1})


def line_summary(path, top):
    res, fpath, hdr = [], None, None
    for row in csv.reader(opener(path)):
        if not row:
            continue
        if row[0] == "File Path":
            fpath, hdr = row[1], None
            continue
        if row[0] == "Function Name":
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr and fpath:
            d = dict(zip(hdr, row))
            try:
                smp = int(d.get("Warp Stall Sampling (All Samples)") or 0)
                ln = int(d["Line No"])
            except ValueError:
                continue
            res.append((smp, fpath, ln))
    tot = max(1, sum(r[0] for r in res))
    for smp, fpath, ln in sorted(res, reverse=True)[:top]:
        local = os.path.join(ROOT, "paper_1905_12725_b200", "csrc", os.path.basename(fpath))
        text = ""
        if os.path.exists(local):
            with open(local) as f:
                lines = f.readlines()
            text = lines[ln - 1].strip()[:100] if ln <= len(lines) else ""
        print(f"{100 * smp / tot:5.1f}%  {os.path.basename(fpath)}:{ln}  {text}")


if __name__ == "__main__":
    raw_summary(sys.argv[1])
    line_summary(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
