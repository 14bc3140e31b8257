"""The paper's SS3.1 / SS3.2 study on its own 63^3 grid: centred spherical inclusion
(vf 0.2), E_m = 70 MPa, nu = 0.3, inclusion E = k E_m for k = 1e-5 ... 1e4; uniaxial strain 0.1 %
(SS3.1, full strain control) and uniaxial stress (SS3.2, every component stress-controlled,
sigma_xx = 0.07 MPa, the others 0).  Tolerances as the paper: equilibrium 1e-8, loading
1e-10, at most 1e4 iterations.  One JSON line per (control, k): PCG iterations, device time and
the three residuals of the converged state.

    python tools/contrast_sweep.py [n]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1905_12725_b200 import dbfft  # noqa: E402
from synth import configs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 63
CONTRASTS = [1e-5, 1e-4, 1e-3, 1e-2, 1e-1, 1e1, 1e2, 1e3, 1e4]
for control in ("strain", "stress"):
    for k in CONTRASTS:
        cfg = configs.s31(n=n, contrast=k)
        if control == "strain":
            target, mask = cfg["loads"][0]["target"], cfg["loads"][0]["mask"]
        else:
            target = np.zeros((3, 3)); target[0, 0] = 0.07
            mask = np.ones((3, 3), bool)
        ctx = dbfft.DBFFT(cfg["n"], kinematics="small")
        ctx.set_phases(cfg["phase"], cfg["materials"])
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(ctx.stream)
        rep = ctx.solve_increment(target, mask, raise_on_error=False, tol_eq=1e-8, tol_load=1e-10,
                                  max_cg=10000, check_every=8)
        ev1.record(ctx.stream)
        torch.cuda.synchronize()
        res = ctx.residuals(target, mask)
        trace = ctx.trace()[:, 0]  # eps_eq per PCG iteration (the paper's Fig. div)
        print(json.dumps(dict(section="3.1" if control == "strain" else "3.2", control=control, contrast=k,
                              grid=list(cfg["n"]), status=rep["status"], cg_iters=rep["cg_iters"],
                              solve_ms=ev0.elapsed_time(ev1), residuals=res,
                              macro_strain_xx=float(rep["macro_strain"][0, 0]),
                              macro_stress_xx=float(rep["macro_stress"][0, 0]),
                              eps_eq_trace_every_10=[float(v) for v in trace[::10]])), flush=True)
        ctx.close()
