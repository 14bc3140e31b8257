"""Time-to-solution of the BASELINE configs c1..c5 on one GPU (solve only; setup separate).

usage: python tools/run_configs.py [c1 c2 c3 c4 c5] [--incs K] [--noprof] [--warm]  -> one JSON line per config"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1905_12725_b200 import dbfft  # noqa: E402
from synth import configs  # noqa: E402

incs = None
if "--incs" in sys.argv:
    incs = int(sys.argv[sys.argv.index("--incs") + 1])
names = [a for a in sys.argv[1:] if not a.startswith("--") and a != str(incs)] or ["c1", "c2", "c3", "c4", "c5"]
for name in names:
    t0 = time.perf_counter()
    cfg = configs.CONFIGS[name]()
    t_gen = time.perf_counter() - t0
    n = cfg["n"]
    N = n[0] * n[1] * n[2]
    t0 = time.perf_counter()
    ctx = dbfft.DBFFT(n, kinematics="finite" if cfg["kin"] == "finite" else "small")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    loads = cfg["loads"][: incs or len(cfg["loads"])]
    if "--noprof" not in sys.argv:  # the per-kernel profiler disables the CUDA-graph PCG rounds
        ctx.profile(True)

    def walk():
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(ctx.stream)
        iters = newton = 0
        reps = []
        for L in loads:
            rep = ctx.solve_increment(L["target"], L["mask"], dt=cfg["dt"], check_every=8)
            iters += rep["cg_iters"]
            newton += rep["newton_iters"]
            reps.append(rep)
        ev1.record(ctx.stream)
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) / 1e3, iters, newton, reps

    # cold: the first walk builds the device-side PCG loop graphs; warm: the same walk again after
    # set_phases (buffers and graphs reused), what a repeated / batched analysis pays
    t, iters, newton, reps = walk()
    t_warm = None
    if "--warm" in sys.argv:
        ctx.set_phases(cfg["phase"], cfg["materials"])
        t_warm = walk()[0]
    prof = ctx.profile_read()
    last = reps[-1]
    ctx.profile(False)
    res = ctx.residuals(loads[-1]["target"], loads[-1]["mask"])  # P:270-290 monitors, final state
    print(json.dumps({"config": name, "grid": list(n), "increments": len(loads), "cg_iters": iters,
                      "newton_iters": newton, "time_to_solution_s": t, "time_to_solution_warm_s": t_warm,
                      "ms_per_cg_iter_warm": (1e3 * t_warm / max(iters, 1)) if t_warm else None,
                      "setup_s": t_setup, "gen_s": t_gen,
                      "voxel_iter_per_s": N * iters / t,
                      "ms_per_cg_iter": 1e3 * t / max(iters, 1),
                      "macro_strain": np.round(last["macro_strain"], 10).tolist(),
                      "macro_stress": np.round(last["macro_stress"], 10).tolist(),
                      "eps_eq": last["eps_eq"],
                      "residuals_final": res,
                      "kernel_ms": {k: round(v[0], 3) for k, v in prof.items()}}), flush=True)
    ctx.close()
    del ctx
    torch.cuda.empty_cache()
