"""Registers / spills per kernel instantiation from a build log (build/obj*/passes.cu.log).

    python tools/ptxas_summary.py LOG [substring]"""
import re
import subprocess
import sys

log = open(sys.argv[1]).read().splitlines()
pat = sys.argv[2] if len(sys.argv) > 2 else "x_pass_kernel"
cur = None
rows = {}
for ln in log:
    m = re.search(r"Function properties for (\S+)", ln)
    if m:
        cur = m.group(1)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m:
        rows.setdefault(cur, {})["spill"] = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", ln)
    if m:
        rows.setdefault(cur, {})["regs"] = int(m.group(1))
names = list(rows)
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
for n, d in zip(names, dem):
    if pat in d:
        r = rows[n]
        print(f"{d[:90]:90s} regs={r.get('regs')} spill={r.get('spill')}")
