"""Kernel-level timing of the operator passes (library CUDA-event profiler, no ncu).

    python tools/kbench.py [n] [reps] [small|finite|j2]

Prints per-pass average ms and GB/s against the SURVEY 8(d) model bytes of each pass."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_1905_12725_b200 import dbfft  # noqa: E402
from synth import configs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
kin = sys.argv[3] if len(sys.argv) > 3 else "finite"
if kin == "finite":
    cfg = configs.c4(n=n, radius_vox=max(1, round(10 * n / 256)))
elif kin == "j2":  # c5's J2-Perzyna polycrystal (elastic tangent right after set_phases)
    cfg = configs.c5(n=n)
else:
    cfg = configs.c3(n=n)
ctx = dbfft.DBFFT(cfg["n"], kinematics="finite" if kin == "finite" else "small")
ctx.set_phases(cfg["phase"], cfg["materials"])
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn((3, n, n, n), dtype=torch.float64, device="cuda", generator=g)
u = (torch.fft.rfftn(x, dim=(1, 2, 3)) / x[0].numel()).permute(0, 2, 1, 3).contiguous()
del x
f = ctx.empty_spectral()
for _ in range(3):
    ctx.apply_K(u, f)
torch.cuda.synchronize()
ctx.profile(True)
for _ in range(reps):
    ctx.apply_K(u, f)
torch.cuda.synchronize()
prof = ctx.profile_read()
H = (n // 2 + 1) * n * n
N = n ** 3
c = 9 if kin == "finite" else 6
fields = {"pass_I1": 3 + 6, "pass_I2": 6 + c, "pass_X": 2 * c, "pass_F2": c + 6, "pass_F3": 6 + 3}
# per-voxel material bytes: compact neo-Hookean (F^-1, c1) + phase id; J2 compact tangent (theta,
# thetabar, n) + phase id; linear: phase id only
mat = 82 * N if kin == "finite" else 66 * N if kin == "j2" else 2 * N
res = {}
for k, (ms, cnt) in prof.items():
    if cnt == 0:
        continue
    avg = ms / cnt
    b = 16 * fields.get(k, 0) * H + (mat if k == "pass_X" else 0)
    res[k] = {"ms": round(avg, 4), "GBps": round(b / avg / 1e6, 1) if b else None}
tot = sum(v["ms"] for v in res.values())
print(json.dumps({"n": n, "kin": kin, "apply_ms": round(tot, 4), "passes": res}))
