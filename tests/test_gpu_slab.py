"""Slab-decomposed (multi-rank) DBFFT through the C ABI in loopback mode: P virtual ranks in one
process on one GPU run the exact distributed data path (rank-chunked z/y passes, the two
exchanges per operator, per-rank partial sums + all-reduce) with device copies standing in for
NCCL.  Compared against the oracle and against P = 1.  Marked `gpu`."""
import numpy as np
import pytest

from oracle import dbfft_oracle as O
from synth import configs, microstructure as ms

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dbf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1905_12725_b200 import dbfft
    dbfft.load_library()
    return dbfft


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def two_phase(n, seed, frac=0.3):
    u = ms.SplitMix64(seed).uniform(n[0] * n[1] * n[2]).reshape(n[2], n[1], n[0])
    return (u < frac).astype(np.uint16)


ISO2 = [dict(kind="iso", E=1.0, nu=0.3), dict(kind="iso", E=10.0, nu=0.25)]


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("n", [(16, 8, 32), (32, 32, 16), (32, 128, 256), (16, 32, 512)])
def test_apply_K_small_loopback(dbf, n, P):
    if n[1] % P or n[2] % P:
        pytest.skip("P must divide n2 and n3")
    ph = two_phase(n, 21)
    ctx = dbf.DBFFT(n, kinematics="small", world=P, loopback=True)
    ctx.set_phases(ph, ISO2)
    u = ms.random_field((3, n[2], n[1], n[0]), 22)
    f = ctx.apply_K(torch.from_numpy(dbf.half_spectrum(u)).cuda())
    ref, _ = O.apply_K(O.fft(u), O.stiffness_field(ph, ISO2), O.frequency_grid(n))
    assert rel(dbf.full_from_half(f.cpu().numpy(), n[0]), ref) <= 1e-12
    # preconditioner with the rank-local ky offsets of xi_y
    z = ctx.precond(torch.from_numpy(dbf.half_spectrum(u)).cuda())
    zref = O.precondition(O.fft(u), O.volume_average(O.stiffness_field(ph, ISO2)), O.frequency_grid(n))
    assert rel(dbf.full_from_half(z.cpu().numpy(), n[0]), zref) <= 1e-12


@pytest.mark.parametrize("P", [2, 4])
def test_apply_K_finite_loopback(dbf, P):
    n = (16, 16, 32)
    ph = two_phase(n, 23)
    mats = [dict(kind="neohooke", mu=1.0, kappa=2.5), dict(kind="neohooke", mu=10.0, kappa=25.0)]
    F = np.eye(3).reshape(3, 3, 1, 1, 1) + 0.1 * ms.random_field((3, 3, n[2], n[1], n[0]), 24)
    ctx = dbf.DBFFT(n, kinematics="finite", world=P, loopback=True)
    ctx.set_phases(ph, mats)
    ctx.eval_state(F.reshape(9, n[2], n[1], n[0]))
    u = ms.random_field((3, n[2], n[1], n[0]), 25)
    f = ctx.apply_K(torch.from_numpy(dbf.half_spectrum(u)).cuda())
    _, K = O.neo_hookean(F, np.array([1.0, 10.0])[ph], np.array([2.5, 25.0])[ph])
    ref, _ = O.apply_K(O.fft(u), K, O.frequency_grid(n), finite=True)
    assert rel(dbf.full_from_half(f.cpu().numpy(), n[0]), ref) <= 1e-12


@pytest.mark.parametrize("P", [2, 8])
def test_solve_c1_loopback(dbf, P):
    cfg = configs.c1()
    L = cfg["loads"][0]
    ref = O.solve_small_strain(cfg["phase"], cfg["materials"], L, tol=1e-10)
    ctx = dbf.DBFFT(cfg["n"], kinematics="small", world=P, loopback=True)
    ctx.set_phases(cfg["phase"], cfg["materials"])
    rep = ctx.solve_increment(L["target"], L["mask"])
    assert rep["converged"] and abs(rep["cg_iters"] - ref["iters"]) <= 1
    assert rel(rep["macro_stress"], ref["mean_sig"]) <= 1e-9
    assert rel(ctx.get_field(dbf.FIELD_STRESS), ref["sig"]) <= 1e-8
    assert rel(ctx.get_field(dbf.FIELD_U), O.displacement(ref["u_hat"])) <= 1e-8


def test_solve_c2_mixed_loopback_matches_single(dbf):
    cfg = configs.c2(n=32, radius_vox=3)
    L = cfg["loads"][0]
    out = {}
    for P in (1, 4):
        ctx = dbf.DBFFT(cfg["n"], kinematics="small", world=P, loopback=P > 1)
        ctx.set_phases(cfg["phase"], cfg["materials"])
        rep = ctx.solve_increment(L["target"], L["mask"])
        out[P] = (rep, ctx.get_field(dbf.FIELD_STRESS))
    assert out[1][0]["cg_iters"] == out[4][0]["cg_iters"]
    assert rel(out[4][0]["macro_stress"], out[1][0]["macro_stress"]) <= 1e-12
    assert rel(out[4][1], out[1][1]) <= 1e-11


def test_solve_c4_twin_loopback(dbf):
    cfg = configs.c4(n=32, radius_vox=3)
    st = O.FiniteStrainState(cfg["n"])
    ctx = dbf.DBFFT(cfg["n"], kinematics="finite", world=2, loopback=True)
    ctx.set_phases(cfg["phase"], cfg["materials"])
    for L in cfg["loads"][:2]:
        ref = O.solve_finite_increment(st, cfg["phase"], cfg["materials"], L, tol=1e-10)
        rep = ctx.solve_increment(L["target"], L["mask"])
        assert rep["converged"] and rep["newton_iters"] == ref["newton_iters"]
        assert rel(rep["macro_stress"], ref["mean_P"]) <= 1e-9
        assert rel(ctx.get_field(dbf.FIELD_STRESS), ref["P"]) <= 1e-8


def test_solve_c5_twin_loopback(dbf):
    cfg = configs.c5(n=16, grains=6, increments=3)
    st = O.J2State(cfg["n"])
    ctx = dbf.DBFFT(cfg["n"], kinematics="small", world=4, loopback=True)
    ctx.set_phases(cfg["phase"], cfg["materials"])
    for L in cfg["loads"]:
        ref = O.solve_j2_increment(st, cfg["phase"], cfg["materials"], L, 1.0, tol=1e-10)
        rep = ctx.solve_increment(L["target"], L["mask"], dt=1.0)
        assert rep["converged"]
        assert rel(rep["macro_stress"], ref["mean_sig"]) <= 1e-9
        assert rel(ctx.get_field(dbf.FIELD_STRESS), ref["sig"]) <= 1e-8
