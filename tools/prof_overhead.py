"""Overhead of the per-kernel CUDA-event profiler (and of CUDA-graph rounds) on a c4 increment."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_1905_12725_b200 import dbfft  # noqa: E402
from synth import configs  # noqa: E402
cfg = configs.c4()
ctx = dbfft.DBFFT(cfg["n"], kinematics="finite")
ctx.set_phases(cfg["phase"], cfg["materials"])
L = cfg["loads"]
for k in range(3):
    ctx.solve_increment(L[k]["target"], L[k]["mask"], check_every=8)
for prof in (True, False, True, False):
    ctx.profile(prof)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(s)
    it = 0
    for k in range(3, 5):
        it += ctx.solve_increment(L[k]["target"], L[k]["mask"], check_every=8)["cg_iters"]
    e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print("profile" if prof else "plain  ", it, "%.1f ms" % ms, "%.3f ms/iter" % (ms / it), "%.3e voxel*it/s" % (256 ** 3 * it / ms * 1e3))
    ctx.set_phases(cfg["phase"], cfg["materials"])
    for k in range(3):
        ctx.solve_increment(L[k]["target"], L[k]["mask"], check_every=8)
