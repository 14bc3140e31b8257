"""Preconditioner variants on one GPU: iteration counts and solve time per variant.

    python tools/precond_variants.py            -> one JSON line per (config, variant)

* refresh policy of the mean tangent (P:263 per increment / every Newton iteration / "once in a
  while"; P:341 initial tangent) on c4 (256^3 neo-Hookean, first K increments) and on the c5 twin
  c5s (128^3, 31 grains, J2);
* reference medium of linear phases (P:255 arithmetic; P:394 harmonic / Hill) on c2 (64^3, equal
  nu: every medium is a multiple of <C>, identical PCG path) and c3 (128^3 cubic polycrystal)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from paper_1905_12725_b200 import dbfft  # noqa: E402
from synth import configs  # noqa: E402


def run(name, cfg, incs, opts):
    n = cfg["n"]
    ctx = dbfft.DBFFT(n, kinematics="finite" if cfg["kin"] == "finite" else "small")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(ctx.stream)
    cg = newton = 0
    per_inc = []
    for L in cfg["loads"][:incs]:
        rep = ctx.solve_increment(L["target"], L["mask"], dt=cfg["dt"], check_every=8, **opts)
        cg += rep["cg_iters"]
        newton += rep["newton_iters"]
        per_inc.append(rep["cg_iters"])
    ev1.record(ctx.stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    out = dict(config=name, grid=list(n), increments=incs, opts=opts, cg_iters=cg, newton_iters=newton,
               cg_per_increment=per_inc, solve_s=ms / 1e3,
               macro_stress=[round(v, 10) for v in rep["macro_stress"].ravel().tolist()])
    ctx.close()
    return out


def main():
    refresh = [dict(precond_refresh=0), dict(precond_refresh=1), dict(precond_refresh=2),
               dict(precond_refresh=3, precond_period=3)]
    t0 = time.time()
    cfg = configs.c4()
    for o in refresh:
        print(json.dumps(run("c4", cfg, 4, o)), flush=True)
    cfg = configs.c5s()
    for o in refresh:
        print(json.dumps(run("c5s", cfg, 6, o)), flush=True)
    for name, cfg in (("c2", configs.c2()), ("c3", configs.c3())):
        for m in (0, 1, 2):
            print(json.dumps(run(name, cfg, 1, dict(precond_medium=m))), flush=True)
    print(json.dumps(dict(total_s=time.time() - t0)), file=sys.stderr)


if __name__ == "__main__":
    main()
