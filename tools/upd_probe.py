"""A few PCG iterations of c4 256^3 (first increment) — a target for ncu on the PCG kernels
(e.g. DBFFT_FUSED_UPDATE=1 ncu -k regex:'col_tma_kernel<256, 7, 1' ...)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_1905_12725_b200 import dbfft  # noqa: E402
from synth import configs  # noqa: E402

cfg = configs.c4()
ctx = dbfft.DBFFT(cfg["n"], kinematics="finite")
ctx.set_phases(cfg["phase"], cfg["materials"])
L = cfg["loads"][0]
ctx.solve_increment(L["target"], L["mask"], raise_on_error=False, max_cg=int(os.environ.get("MAXCG", "12")), max_newton=1)
torch.cuda.synchronize()
print("ok")
