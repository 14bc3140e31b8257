"""2-D pencil decomposition (include/dbfft.h dbfft_env.pencil_rows) through the C ABI in
loopback mode: P = Py x Pz virtual ranks in one process on one GPU run the exact distributed data path
— kx-blocked spectra, the column-group exchanges around the z passes, the row-group exchanges of the
x-line layout after the y-inverse and the x pass, per-rank partial sums + all-reduce — with device
copies standing in for NCCL.  Operator outputs are compared with P = 1 (to round-off: a kx block
narrower than a TMA tile takes the register-pipelined column kernel, whose twiddles are products of
table entries) and with the oracle; solves with the oracle.  Marked `gpu`."""
import numpy as np
import pytest

from oracle import dbfft_oracle as O
from spectra import full_from_half, half_spectrum
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
NH2 = [dict(kind="neohooke", mu=1.0, kappa=2.5), dict(kind="neohooke", mu=10.0, kappa=25.0)]

# (grid, (Py, Pz)): register-pipelined column kernels (8..32), TMA column passes (64..256; kx
# blocks of 8 / 16 / 32 columns), the n1 = 512 x pass (two-warp pair FFTs) and Py = n1/2
GRIDS = [((16, 8, 32), (2, 2)), ((16, 8, 32), (8, 1)), ((32, 32, 16), (4, 2)), ((32, 32, 16), (2, 4)),
         ((64, 64, 64), (2, 2)), ((256, 16, 64), (2, 2)), ((32, 128, 256), (4, 2)), ((512, 8, 16), (2, 4)),
         ((128, 64, 32), (4, 1)), ((256, 128, 128), (2, 2))]


def ctx_of(dbf, n, kin, py, pz):
    P = py * pz
    return dbf.DBFFT(n, kinematics=kin, world=P, loopback=P > 1, pencil_rows=py)


@pytest.mark.parametrize("n,grid", GRIDS)
def test_apply_K_small_pencil(dbf, n, grid):
    py, pz = grid
    ph = two_phase(n, 41)
    u = torch.from_numpy(half_spectrum(ms.random_field((3, n[2], n[1], n[0]), 42))).cuda()
    out = {}
    for g in [(1, 1), grid]:
        ctx = ctx_of(dbf, n, "small", *g)
        ctx.set_phases(ph, ISO2)
        assert ("pencils" in ctx.info()["decomposition"]) == (g[0] > 1)
        out[g] = (ctx.apply_K(u).cpu().numpy(), ctx.precond(u).cpu().numpy())
        ctx.close()
    assert rel(out[grid][0], out[(1, 1)][0]) <= 1e-14
    assert rel(out[grid][1], out[(1, 1)][1]) <= 1e-15
    if n[0] * n[1] * n[2] <= 64 ** 3:
        ur = ms.random_field((3, n[2], n[1], n[0]), 42)
        ref, _ = O.apply_K(O.fft(ur), O.stiffness_field(ph, ISO2), O.frequency_grid(n))
        assert rel(full_from_half(out[grid][0], n[0]), ref) <= 1e-12


@pytest.mark.parametrize("n,grid", [((16, 16, 32), (2, 2)), ((16, 16, 32), (4, 1)), ((64, 32, 32), (2, 4)),
                                    ((256, 16, 16), (4, 2))])
def test_apply_K_finite_pencil(dbf, n, grid):
    ph = two_phase(n, 43)
    F = np.eye(3).reshape(3, 3, 1, 1, 1) + 0.1 * ms.random_field((3, 3, n[2], n[1], n[0]), 44)
    ur = ms.random_field((3, n[2], n[1], n[0]), 45)
    u = torch.from_numpy(half_spectrum(ur)).cuda()
    out = {}
    for g in [(1, 1), grid]:
        ctx = ctx_of(dbf, n, "finite", *g)
        ctx.set_phases(ph, NH2)
        ctx.eval_state(F.reshape(9, n[2], n[1], n[0]))
        out[g] = ctx.apply_K(u).cpu().numpy()
        # the per-voxel tangent comes back in the global layout
        if g == grid:
            tan = ctx.get_field(dbf.FIELD_TANGENT)
        ctx.close()
    assert rel(out[grid], out[(1, 1)]) <= 1e-14
    _, K = O.neo_hookean(F, np.array([1.0, 10.0])[ph], np.array([2.5, 25.0])[ph])
    if n[0] * n[1] * n[2] <= 32 ** 3:
        ref, _ = O.apply_K(O.fft(ur), K, O.frequency_grid(n), finite=True)
        assert rel(full_from_half(out[grid], n[0]), ref) <= 1e-12
    assert rel(tan, K) <= 1e-13


def test_apply_K_aug_pencil(dbf):
    n = (32, 16, 16)
    ph = two_phase(n, 46)
    mask = np.array([1, 0, 0, 0, 1, 0, 0, 0, 0], np.uint8)
    e = 0.01 * np.arange(1, 10, dtype=np.float64)
    e = 0.5 * (e.reshape(3, 3) + e.reshape(3, 3).T).ravel()
    u = torch.from_numpy(half_spectrum(ms.random_field((3, n[2], n[1], n[0]), 47))).cuda()
    out = {}
    for g in [(1, 1), (2, 2)]:
        ctx = ctx_of(dbf, n, "small", *g)
        ctx.set_phases(ph, ISO2)
        f, r = ctx.apply_K_aug(mask, u, e)
        out[g] = (f.cpu().numpy(), r)
    assert rel(out[(2, 2)][0], out[(1, 1)][0]) <= 1e-14
    assert np.allclose(out[(2, 2)][1], out[(1, 1)][1], rtol=1e-13, atol=1e-16)


@pytest.mark.parametrize("grid", [(2, 2), (4, 2), (2, 1)])
def test_solve_c1_pencil(dbf, grid):
    cfg = configs.c1()
    L = cfg["loads"][0]
    ref = O.solve_small_strain(cfg["phase"], cfg["materials"], L, tol=1e-10)
    ctx = ctx_of(dbf, cfg["n"], "small", *grid)
    ctx.set_phases(cfg["phase"], cfg["materials"])
    rep = ctx.solve_increment(L["target"], L["mask"])
    assert rep["converged"] and abs(rep["cg_iters"] - ref["iters"]) <= 1
    assert rel(rep["macro_stress"], ref["mean_sig"]) <= 1e-9
    assert rel(ctx.get_field(dbf.FIELD_STRESS), ref["sig"]) <= 1e-8
    assert rel(ctx.get_field(dbf.FIELD_STRAIN), ref["eps"]) <= 1e-8
    assert rel(ctx.get_field(dbf.FIELD_U), O.displacement(ref["u_hat"])) <= 1e-8
    uh = ctx.get_field(dbf.FIELD_U_HAT).cpu().numpy()
    assert rel(full_from_half(uh, cfg["n"][0]), ref["u_hat"]) <= 1e-8


def test_solve_c2_mixed_pencil_matches_single(dbf):
    cfg = configs.c2(n=32, radius_vox=3)
    L = cfg["loads"][0]
    out = {}
    for g in [(1, 1), (2, 2), (4, 2)]:
        ctx = ctx_of(dbf, cfg["n"], "small", *g)
        ctx.set_phases(cfg["phase"], cfg["materials"])
        rep = ctx.solve_increment(L["target"], L["mask"])
        out[g] = (rep, ctx.get_field(dbf.FIELD_STRESS), ctx.residuals(L["target"], L["mask"]))
    for g in [(2, 2), (4, 2)]:
        assert abs(out[g][0]["cg_iters"] - out[(1, 1)][0]["cg_iters"]) <= 1
        assert rel(out[g][0]["macro_stress"], out[(1, 1)][0]["macro_stress"]) <= 1e-10
        assert rel(out[g][1], out[(1, 1)][1]) <= 1e-9
        r, r1 = out[g][2], out[(1, 1)][2]
        assert r["equilibrium"] <= 2e-10 and r["loading"] <= 1e-10
        assert r["compatibility"] == pytest.approx(r1["compatibility"], rel=0.5, abs=1e-13)


def test_solve_c4_twin_pencil(dbf):
    cfg = configs.c4(n=32, radius_vox=3)
    st = O.FiniteStrainState(cfg["n"])
    ctx = ctx_of(dbf, cfg["n"], "finite", 2, 2)
    ctx.set_phases(cfg["phase"], cfg["materials"])
    for L in cfg["loads"][:2]:
        ref = O.solve_finite_increment(st, cfg["phase"], cfg["materials"], L, tol=1e-10)
        rep = ctx.solve_increment(L["target"], L["mask"])
        assert rep["converged"] and rep["newton_iters"] == ref["newton_iters"]
        assert rel(rep["macro_stress"], ref["mean_P"]) <= 1e-9
        assert rel(ctx.get_field(dbf.FIELD_STRESS), ref["P"]) <= 1e-8
        assert rel(ctx.get_field(dbf.FIELD_STRAIN), ref["F"]) <= 1e-9
    r = ctx.residuals(L["target"], L["mask"])
    assert r["loading"] <= 1e-10 and r["compatibility"] <= 1e-10 and r["equilibrium"] <= 1e-6


def test_solve_c5_twin_pencil(dbf):
    cfg = configs.c5(n=16, grains=6, increments=3)
    st = O.J2State(cfg["n"])
    ctx = ctx_of(dbf, cfg["n"], "small", 2, 4)
    ctx.set_phases(cfg["phase"], cfg["materials"])
    for L in cfg["loads"]:
        ref = O.solve_j2_increment(st, cfg["phase"], cfg["materials"], L, 1.0, tol=1e-10)
        rep = ctx.solve_increment(L["target"], L["mask"], dt=1.0)
        assert rep["converged"]
        assert rel(rep["macro_stress"], ref["mean_sig"]) <= 1e-9
        assert rel(ctx.get_field(dbf.FIELD_STRESS), ref["sig"]) <= 1e-8


def test_pencil_invalid(dbf):
    with pytest.raises(dbf.DBFFTError):
        dbf.DBFFT((16, 16, 16), world=4, loopback=True, pencil_rows=3)    # not a power of two
    with pytest.raises(dbf.DBFFTError):
        dbf.DBFFT((16, 16, 16), world=4, loopback=True, pencil_rows=16)   # > world
    with pytest.raises(dbf.DBFFTError):
        dbf.DBFFT((8, 16, 16), world=8, loopback=True, pencil_rows=8)     # n1 / 2 < Py
    with pytest.raises(dbf.DBFFTError):
        dbf.DBFFT((15, 16, 16), world=2, loopback=True, pencil_rows=2)    # odd n1
    with pytest.raises(dbf.DBFFTError):
        dbf.DBFFT((16, 16, 16), world=4, loopback=True, pencil_rows=2, transport="peer")
