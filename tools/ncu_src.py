"""Summarise an ncu source page (cuda,sass) by CUDA source line: stall samples per line."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kfilter = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
agg = defaultdict(lambda: [0, 0, ""])
cur_file = None
cur_fn = None
hdr = None
for row in csv.reader(lines):
    if not row:
        continue
    if row[0] == "File Path":
        cur_file = row[1].split("/")[-1]
        continue
    if row[0] == "Function Name":
        cur_fn = row[1]
        continue
    if kfilter and kfilter not in (cur_fn or ""):
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < 6:
        continue
    try:
        ln = int(row[0])
    except ValueError:
        continue
    src = row[1]
    try:
        s_all = int(row[4] or 0)
        s_ni = int(row[5] or 0)
    except ValueError:
        continue
    key = (cur_file, ln)
    agg[key][0] += s_all
    agg[key][1] += s_ni
    if src:
        agg[key][2] = src.strip()[:90]
tot = sum(v[0] for v in agg.values()) or 1
for (f, ln), (a, ni, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*a/tot:5.1f}% {f}:{ln:4d}  {src}")
