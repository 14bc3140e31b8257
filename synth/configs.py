"""The five BASELINE.json configurations (c1..c5) as raw, seeded inputs.

Every number here is a *parameter* (moduli, geometry, load targets), never a
derived quantity of the method: Lame constants, stiffness tensors, rotations
of tensors etc. are computed separately by the oracle and by the product.
Readings R14-R21 of SURVEY section 8(c) are applied here.

Material records: dict(kind=..., params...) with kinds
  'iso'      : E, nu                       (linear isotropic)
  'cubic'    : C11, C12, C44, R (3x3)      (crystal frame stiffness + rotation)
  'neohooke' : mu, kappa                   (R14)
  'j2'       : E, nu, sigma_y, n, edot0    (R16)
  'svk'      : E, nu                       (Saint Venant-Kirchhoff)
Load: target (3x3), mask (3x3 bool, True = stress-controlled).
"""
import numpy as np
from . import microstructure as ms

SMALL, FINITE = "small", "finite"


def _load(target, mask):
    return dict(target=np.asarray(target, dtype=np.float64), mask=np.asarray(mask, dtype=bool))


def c1(n=8):
    """8^3, centred sphere r=0.25, E=1/10, nu=0.3, eps_xx=1e-3 strain control (BJ configs[0])."""
    phase = ms.centred_sphere((n, n, n), 0.25)
    mats = [dict(kind="iso", E=1.0, nu=0.3), dict(kind="iso", E=10.0, nu=0.3)]
    t = np.zeros((3, 3)); t[0, 0] = 1e-3
    return dict(name="c1", n=(n, n, n), kin=SMALL, phase=phase, materials=mats,
                loads=[_load(t, np.zeros((3, 3), bool))], dt=1.0)


def c2(n=64, radius_vox=6, count=None, seed=2):
    """64^3, RSA spheres r=6 (vf~0.2), E 100/1, mixed control (R18, BJ configs[1])."""
    if count is None:
        count = int(round(0.2 * n ** 3 / (4.0 / 3.0 * np.pi * radius_vox ** 3)))
    phase, _ = ms.rsa_spheres((n, n, n), count, radius_vox, seed)
    mats = [dict(kind="iso", E=1.0, nu=0.3), dict(kind="iso", E=100.0, nu=0.3)]
    t = np.zeros((3, 3)); t[2, 2] = 1e-3
    mask = np.ones((3, 3), bool); mask[2, 2] = False
    return dict(name="c2", n=(n, n, n), kin=SMALL, phase=phase, materials=mats,
                loads=[_load(t, mask)], dt=1.0)


def c3(n=128, grains=200, seed=3):
    """128^3 Voronoi polycrystal, rotated cubic Cu (GPa), pure shear xy (R19, BJ configs[2])."""
    phase, _ = ms.voronoi((n, n, n), grains, seed)
    R = ms.random_rotations(grains, seed + 1000)
    mats = [dict(kind="cubic", C11=168.4, C12=121.4, C44=75.4, R=R[g]) for g in range(grains)]
    t = np.zeros((3, 3)); t[0, 1] = t[1, 0] = 1e-3
    return dict(name="c3", n=(n, n, n), kin=SMALL, phase=phase, materials=mats,
                loads=[_load(t, np.zeros((3, 3), bool))], dt=1.0)


def c4(n=256, radius_vox=10, count=None, seed=4, increments=10):
    """256^3 finite-strain neo-Hookean, 30% spheres, F_zz -> 1.10 in 10 increments,
    P_xx = P_yy = 0 (R14, R15, BJ configs[3])."""
    if count is None:
        count = int(round(0.3 * n ** 3 / (4.0 / 3.0 * np.pi * radius_vox ** 3)))
    phase, _ = ms.rsa_spheres((n, n, n), count, radius_vox, seed)
    mats = [dict(kind="neohooke", mu=1.0, kappa=2.5), dict(kind="neohooke", mu=10.0, kappa=25.0)]
    mask = np.zeros((3, 3), bool); mask[0, 0] = mask[1, 1] = True
    loads = []
    for k in range(1, increments + 1):
        t = np.eye(3); t[2, 2] = 1.0 + 0.1 * k / increments
        t[0, 0] = t[1, 1] = 0.0          # stress-controlled targets P_xx = P_yy = 0
        loads.append(_load(t, mask))
    return dict(name="c4", n=(n, n, n), kin=FINITE, phase=phase, materials=mats, loads=loads, dt=1.0)


def c5(n=512, grains=2000, seed=5, increments=20):
    """512^3 J2-Perzyna polycrystal (R16, R17, BJ configs[4]); eps = 1e-3 t diag(-1/2,-1/2,1)."""
    phase, _ = ms.voronoi((n, n, n), grains, seed)
    sy = ms.lognormal(grains, seed + 1000, 300.0, 0.2)
    mats = [dict(kind="j2", E=2.0e5, nu=0.3, sigma_y=float(sy[g]), n=20.0, edot0=1e-3) for g in range(grains)]
    loads = []
    for k in range(1, increments + 1):
        t = 1e-3 * k * np.diag([-0.5, -0.5, 1.0])
        loads.append(_load(t, np.zeros((3, 3), bool)))
    return dict(name="c5", n=(n, n, n), kin=SMALL, phase=phase, materials=mats, loads=loads, dt=1.0)


def c5s(n=128, grains=31, seed=5, increments=20):
    """Downscaled c5 twin: same grain volume, all else identical."""
    d = c5(n=n, grains=grains, seed=seed, increments=increments)
    d["name"] = "c5s"
    return d


def s31(n=63, contrast=10.0, vf=0.2):
    """The paper's SS3.1 cell: one centred spherical inclusion of volume fraction
    `vf` in an n^3 cell (63^3 in the paper), matrix E = 70 MPa, nu = 0.3, inclusion E = k E_m;
    uniaxial strain 0.1 % (full strain control, other components 0)."""
    r = (3.0 * vf / (4.0 * np.pi)) ** (1.0 / 3.0)
    phase = ms.centred_sphere((n, n, n), r)
    mats = [dict(kind="iso", E=70.0, nu=0.3), dict(kind="iso", E=70.0 * contrast, nu=0.3)]
    t = np.zeros((3, 3)); t[0, 0] = 1e-3
    return dict(name="s31", n=(n, n, n), kin=SMALL, phase=phase, materials=mats,
                loads=[_load(t, np.zeros((3, 3), bool))], dt=1.0)


def p33(n=64, pores=5, vf=0.2, seed=33, increments=5, stretch=2.0):
    """The paper's own finite-strain benchmark (SS3.3), synthetic stand-in:
    SVK matrix E = 70 MPa, nu = 0.3 with `pores` non-overlapping spherical voids of total volume
    fraction `vf` modelled as 100x more compliant SVK inclusions; uniaxial elongation
    lambda = L/L0 -> `stretch` along z with the other directions held (full deformation control),
    in `increments` equal steps.  The paper's cell is 63^3 (odd grids: SURVEY 8(f1)); n = 64 here."""
    radius = (vf * n ** 3 / pores * 3.0 / (4.0 * np.pi)) ** (1.0 / 3.0)
    phase, _ = ms.rsa_spheres((n, n, n), pores, radius, seed)
    mats = [dict(kind="svk", E=70.0, nu=0.3), dict(kind="svk", E=0.7, nu=0.3)]
    loads = []
    for k in range(1, increments + 1):
        loads.append(_load(np.diag([1.0, 1.0, 1.0 + (stretch - 1.0) * k / increments]), np.zeros((3, 3), bool)))
    return dict(name="p33", n=(n, n, n), kin=FINITE, phase=phase, materials=mats, loads=loads, dt=1.0)


CONFIGS = dict(c1=c1, c2=c2, c3=c3, c4=c4, c5=c5, c5s=c5s, p33=p33, s31=s31)
