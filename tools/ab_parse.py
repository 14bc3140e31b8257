"""Summarise tools/ab_multi.sh output: apply_K and pass_X per build and config."""
import json
import re
import sys

for ln in open(sys.argv[1]):
    m = re.match(r"(\S+) (.*?): (\{.*)", ln.strip())
    if not m:
        print(ln.strip()[:200])
        continue
    d = json.loads(m.group(3))
    p = d["passes"]
    other = " ".join(f"{k[5:]}={v['ms']:.3f}" for k, v in p.items() if k != "pass_X")
    print(f"{m.group(1):22s} {m.group(2):16s} apply={d['apply_ms']:.3f} X={p['pass_X']['ms']:.4f} ({p['pass_X']['GBps']})  {other}")
