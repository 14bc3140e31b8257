"""Where the e2e leg's time goes: K increments of c4's load walk through the C ABI, timed on the
host (wall) and on the device (CUDA events), with / without get_field(U) and with the PCG
rounds replayed from CUDA graphs or launched directly (DBFFT_GRAPHS=0 in a second process).

    python tools/e2e_probe.py [K]"""
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

K = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = configs.c4()
stream = torch.cuda.current_stream()
ctx = dbfft.DBFFT(cfg["n"], kinematics="finite", stream=stream)
phase_host = torch.from_numpy(cfg["phase"].view(np.int16)).pin_memory().numpy().view(np.uint16)
u_host = torch.empty((3,) + cfg["phase"].shape, dtype=torch.float64, pin_memory=True).numpy()
for fetch in (True, False, True):
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    ev0.record(stream)
    ctx.set_phases(phase_host, cfg["materials"])
    t_set = time.perf_counter() - t0
    its, t_solve, t_get = 0, 0.0, 0.0
    for k in range(K):
        L = cfg["loads"][k]
        a = time.perf_counter()
        rep = ctx.solve_increment(L["target"], L["mask"])
        b = time.perf_counter()
        if fetch:
            ctx.get_field(dbfft.FIELD_U, out=u_host)
        t_solve += b - a
        t_get += time.perf_counter() - b
        its += rep["cg_iters"]
    ev1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    dev = ev0.elapsed_time(ev1) / 1e3
    N = np.prod(cfg["n"])
    print(json.dumps(dict(graphs=os.environ.get("DBFFT_GRAPHS", "1"), fetch=fetch, cg_iters=its, wall_s=wall, device_s=dev,
                          set_phases_s=t_set, solve_s=t_solve, get_field_s=t_get,
                          wall_rate=N * its / wall, device_rate=N * its / dev)), flush=True)
