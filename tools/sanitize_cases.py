"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck): every kernel family of the
hot path once — register and TMA column passes (incl. the N = 512 named-barrier columns), pass_X
(incl. n1 = 512 pair FFTs across two warps), the fused F3 + PCG update, the device-side PCG loop,
the constitutive kinds (neo-Hookean, J2), loopback slabs and the residual monitors.

    python tools/sanitize_cases.py [case ...]      (default: all)"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_1905_12725_b200 import dbfft  # noqa: E402
from synth import configs, microstructure as ms  # noqa: E402


def spec(ctx, seed):
    n = ctx.n
    x = torch.from_numpy(ms.random_field((3, n[2], n[1], n[0]), seed)).cuda()
    return (torch.fft.rfftn(x, dim=(1, 2, 3)) / x[0].numel()).permute(0, 2, 1, 3).contiguous()


def two_phase(n, seed):
    return (ms.SplitMix64(seed).uniform(n[0] * n[1] * n[2]).reshape(n[2], n[1], n[0]) < 0.3).astype(np.uint16)


ISO2 = [dict(kind="iso", E=1.0, nu=0.3), dict(kind="iso", E=10.0, nu=0.25)]
NH2 = [dict(kind="neohooke", mu=1.0, kappa=2.5), dict(kind="neohooke", mu=10.0, kappa=25.0)]


def c1():
    cfg = configs.c1()
    ctx = dbfft.DBFFT(cfg["n"], kinematics="small")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    L = cfg["loads"][0]
    ctx.solve_increment(L["target"], L["mask"])
    ctx.residuals(L["target"], L["mask"])
    ctx.get_field(dbfft.FIELD_STRESS)


def finite16():
    cfg = configs.c4(n=16, radius_vox=2)
    ctx = dbfft.DBFFT(cfg["n"], kinematics="finite")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    L = cfg["loads"][0]
    ctx.solve_increment(L["target"], L["mask"])
    ctx.get_field(dbfft.FIELD_TANGENT)


def j2_16():
    cfg = configs.c5(n=16, grains=4, increments=2)
    ctx = dbfft.DBFFT(cfg["n"], kinematics="small")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    for L in cfg["loads"]:
        ctx.solve_increment(L["target"], L["mask"], dt=1.0)


def tma():
    """TMA column passes (N = 128, 256 on z / y), both kinematics, and a fused-update PCG solve."""
    n = (16, 128, 256)
    for kin, mats in (("small", ISO2), ("finite", NH2)):
        ctx = dbfft.DBFFT(n, kinematics=kin)
        ctx.set_phases(two_phase(n, 71), mats)
        ctx.apply_K(spec(ctx, 72))
        t = np.eye(3) + np.diag([0.0, 0.0, 1e-3]) if kin == "finite" else np.diag([0.0, 0.0, 1e-3])
        ctx.solve_increment(t, np.zeros((3, 3), bool), max_cg=30, raise_on_error=False)


def n512():
    """N = 512 columns (z: TMA tiles of 4 columns, 64 threads per column on two warps) and n1 = 512
    pair FFTs (named barriers), small and finite."""
    for n in ((16, 8, 512), (512, 8, 8)):
        for kin, mats in (("small", ISO2), ("finite", NH2)):
            ctx = dbfft.DBFFT(n, kinematics=kin)
            ctx.set_phases(two_phase(n, 73), mats)
            ctx.apply_K(spec(ctx, 74))


def loopback():
    n = (16, 32, 64)
    for transport in ("nccl", "peer"):
        ctx = dbfft.DBFFT(n, kinematics="small", world=2, loopback=True, transport=transport)
        ctx.set_phases(two_phase(n, 75), ISO2)
        ctx.apply_K(spec(ctx, 76))
        ctx.solve_increment(np.diag([1e-3, 0, 0]), np.zeros((3, 3), bool), max_cg=20, raise_on_error=False)


CASES = dict(c1=c1, finite16=finite16, j2_16=j2_16, tma=tma, n512=n512, loopback=loopback)

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
        torch.cuda.synchronize()
        print("case", name, "ok", flush=True)
