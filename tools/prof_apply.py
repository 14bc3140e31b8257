"""Profiling driver: c4-size operator applications (for ncu).  Usage: python tools/prof_apply.py [n] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1905_12725_b200 import dbfft  # noqa: E402
from synth import configs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = configs.c4(n=n, radius_vox=max(1, round(10 * n / 256)))
ctx = dbfft.DBFFT(cfg["n"], kinematics="finite")
ctx.set_phases(cfg["phase"], cfg["materials"])
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn((3, n, n, n), dtype=torch.float64, device="cuda", generator=g)
u = (torch.fft.rfftn(x, dim=(1, 2, 3)) / x[0].numel()).permute(0, 2, 1, 3).contiguous()
del x
f = ctx.empty_spectral()
for _ in range(reps):
    ctx.apply_K(u, f)
torch.cuda.synchronize()
print("ok", float(f.abs().max()))
