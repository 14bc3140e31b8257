"""GPU-vs-oracle parity through the C ABI (libdbfft.so).  Marked `gpu`.

Bars (BASELINE.json north_star): single operator applications 1e-12 relative (fp64),
macroscopic stress/strain 1e-9 relative, per-voxel fields 1e-8 relative L2 at tol 1e-10."""
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


def to_gpu_spec(dbf, u_real):
    return torch.from_numpy(half_spectrum(u_real)).cuda()


def gpu_full(dbf, t, n1):
    return full_from_half(t.cpu().numpy(), n1)


def two_phase(n, seed, frac=0.3):
    u = ms.SplitMix64(seed).uniform(n[0] * n[1] * n[2]).reshape(n[2], n[1], n[0])
    return (u < frac).astype(np.uint16)


ISO2 = [dict(kind="iso", E=1.0, nu=0.3), dict(kind="iso", E=10.0, nu=0.25)]
GRIDS = [(8, 8, 8), (16, 8, 32), (32, 64, 16), (64, 64, 64)]


@pytest.mark.parametrize("n", GRIDS)
def test_apply_K_small_linear(dbf, n):
    ph = two_phase(n, 1)
    ctx = dbf.DBFFT(n, kinematics="small")
    ctx.set_phases(ph, ISO2)
    u = ms.random_field((3, n[2], n[1], n[0]), 7)
    f = ctx.apply_K(to_gpu_spec(dbf, u))
    torch.cuda.synchronize()
    XI = O.frequency_grid(n)
    ref, _ = O.apply_K(O.fft(u), O.stiffness_field(ph, ISO2), XI)
    assert rel(gpu_full(dbf, f, n[0]), ref) <= 1e-12


@pytest.mark.parametrize("n", [(8, 8, 8), (32, 16, 64)])
def test_apply_K_cubic_polycrystal(dbf, n):
    cfg = configs.c3(n=n[0], grains=12, seed=3) if n[0] == n[1] == n[2] else None
    if cfg is None:
        ph, _ = ms.voronoi(n, 12, 3)
        R = ms.random_rotations(12, 1003)
        mats = [dict(kind="cubic", C11=168.4, C12=121.4, C44=75.4, R=R[g]) for g in range(12)]
    else:
        ph, mats = cfg["phase"], cfg["materials"]
    ctx = dbf.DBFFT(n, kinematics="small")
    ctx.set_phases(ph, mats)
    u = ms.random_field((3, n[2], n[1], n[0]), 8)
    f = ctx.apply_K(to_gpu_spec(dbf, u))
    ref, _ = O.apply_K(O.fft(u), O.stiffness_field(ph, mats), O.frequency_grid(n))
    assert rel(gpu_full(dbf, f, n[0]), ref) <= 1e-12


@pytest.mark.parametrize("tangent", ["compact", "full"])
@pytest.mark.parametrize("n", [(8, 8, 8), (16, 32, 8), (32, 32, 32)])
def test_apply_K_finite_neohooke(dbf, n, tangent, monkeypatch):
    monkeypatch.setenv("DBFFT_TANGENT", tangent)
    ph = two_phase(n, 2)
    mats = [dict(kind="neohooke", mu=1.0, kappa=2.5), dict(kind="neohooke", mu=10.0, kappa=25.0)]
    F = np.eye(3).reshape(3, 3, 1, 1, 1) + 0.1 * ms.random_field((3, 3, n[2], n[1], n[0]), 9)
    ctx = dbf.DBFFT(n, kinematics="finite")
    ctx.set_phases(ph, mats)
    ctx.eval_state(F.reshape(9, n[2], n[1], n[0]))
    u = ms.random_field((3, n[2], n[1], n[0]), 10)
    f = ctx.apply_K(to_gpu_spec(dbf, u))
    mu = np.array([1.0, 10.0])[ph]
    kap = np.array([2.5, 25.0])[ph]
    _, K = O.neo_hookean(F, mu, kap)
    ref, _ = O.apply_K(O.fft(u), K, O.frequency_grid(n), finite=True)
    assert rel(gpu_full(dbf, f, n[0]), ref) <= 1e-12


# grids whose z / y sweeps take the TMA column kernel (N in {64, 128, 256}, n1/2 a multiple of
# 2048/N): several kx blocks + the Nyquist tail tiles, and an outer count (8) below the tile
# width (16 at N = 128: narrower tail boxes); N = 512 runs 4-column tiles (64-byte rows, 64B
# swizzle) with a column's 64 threads on two warps (named-barrier exchanges)
TMA_GRIDS = [(32, 128, 256), (64, 256, 128), (32, 8, 128), (128, 64, 64), (16, 8, 512), (8, 512, 16)]


@pytest.mark.parametrize("n", TMA_GRIDS)
def test_apply_K_tma_small(dbf, n):
    ph = two_phase(n, 31)
    ctx = dbf.DBFFT(n, kinematics="small")
    ctx.set_phases(ph, ISO2)
    u = ms.random_field((3, n[2], n[1], n[0]), 32)
    f = ctx.apply_K(to_gpu_spec(dbf, u))
    ref, _ = O.apply_K(O.fft(u), O.stiffness_field(ph, ISO2), O.frequency_grid(n))
    assert rel(gpu_full(dbf, f, n[0]), ref) <= 1e-12


@pytest.mark.parametrize("n", TMA_GRIDS[:3] + TMA_GRIDS[4:] + [(256, 16, 8), (256, 8, 32)])
def test_apply_K_tma_finite(dbf, n):
    ph = two_phase(n, 33)
    mats = [dict(kind="neohooke", mu=1.0, kappa=2.5), dict(kind="neohooke", mu=10.0, kappa=25.0)]
    F = np.eye(3).reshape(3, 3, 1, 1, 1) + 0.1 * ms.random_field((3, 3, n[2], n[1], n[0]), 34)
    ctx = dbf.DBFFT(n, kinematics="finite")
    ctx.set_phases(ph, mats)
    ctx.eval_state(F.reshape(9, n[2], n[1], n[0]))
    u = ms.random_field((3, n[2], n[1], n[0]), 35)
    f = ctx.apply_K(to_gpu_spec(dbf, u))
    _, K = O.neo_hookean(F, np.array([1.0, 10.0])[ph], np.array([2.5, 25.0])[ph])
    ref, _ = O.apply_K(O.fft(u), K, O.frequency_grid(n), finite=True)
    assert rel(gpu_full(dbf, f, n[0]), ref) <= 1e-12


@pytest.mark.parametrize("n", [(8, 8, 8), (32, 16, 16)])
def test_apply_K_j2_tangent(dbf, n):
    ph = two_phase(n, 3, 0.5)
    mats = [dict(kind="j2", E=2e5, nu=0.3, sigma_y=300.0, n=20.0, edot0=1e-3),
            dict(kind="j2", E=2e5, nu=0.3, sigma_y=200.0, n=20.0, edot0=1e-3)]
    eps = 2e-3 * np.diag([-0.5, -0.5, 1.0]).reshape(3, 3, 1, 1, 1) + 5e-4 * ms.random_field((3, 3, n[2], n[1], n[0]), 11)
    eps = 0.5 * (eps + np.swapaxes(eps, 0, 1))
    ctx = dbf.DBFFT(n, kinematics="small")
    ctx.set_phases(ph, mats)
    ctx.eval_state(eps.reshape(9, n[2], n[1], n[0]), dt=1.0)
    u = ms.random_field((3, n[2], n[1], n[0]), 12)
    f = ctx.apply_K(to_gpu_spec(dbf, u))
    sy = np.array([300.0, 200.0])[ph]
    _, C, _, dp = O.j2_perzyna(eps, np.zeros_like(eps), 2e5, 0.3, sy, 20.0, 1e-3, 1.0)
    assert np.mean(dp > 0) > 0.2  # a real mix of plastic and elastic voxels
    ref, _ = O.apply_K(O.fft(u), C, O.frequency_grid(n))
    assert rel(gpu_full(dbf, f, n[0]), ref) <= 1e-12


def test_precond_and_aug(dbf):
    n = (16, 32, 8)
    ph = two_phase(n, 4)
    C = O.stiffness_field(ph, ISO2)
    ctx = dbf.DBFFT(n, kinematics="small")
    ctx.set_phases(ph, ISO2)
    r = ms.random_field((3, n[2], n[1], n[0]), 13)
    z = ctx.precond(to_gpu_spec(dbf, r))
    XI = O.frequency_grid(n)
    zref = O.precondition(O.fft(r), O.volume_average(C), XI)
    assert rel(gpu_full(dbf, z, n[0]), zref) <= 1e-12
    mask = np.zeros((3, 3), bool); mask[0, 0] = mask[1, 1] = mask[0, 1] = mask[1, 0] = True
    e = np.array([[1e-3, 2e-4, 0], [2e-4, -5e-4, 0], [0, 0, 0.0]])
    u = ms.random_field((3, n[2], n[1], n[0]), 14)
    f, rout = ctx.apply_K_aug(mask, to_gpu_spec(dbf, u), e)
    fref, msig = O.apply_K(O.fft(u), C, XI, e=e)
    assert rel(gpu_full(dbf, f, n[0]), fref) <= 1e-12
    assert np.allclose(rout, np.where(mask, msig, 0.0), rtol=1e-12, atol=1e-15 * np.abs(msig).max())


def test_hermitian_and_null_modes_full_size(dbf):
    """Full c4-size property test (any size): <Kv,w> = <v,Kw> and K = 0 on Z."""
    n = (256, 256, 256)
    cfg = configs.c4()
    ctx = dbf.DBFFT(n, kinematics="finite")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    g = torch.Generator(device="cuda").manual_seed(0)

    def rnd():
        x = torch.randn((3, n[2], n[1], n[0]), dtype=torch.float64, device="cuda", generator=g)
        h = torch.fft.rfftn(x, dim=(1, 2, 3)) / x[0].numel()
        return h.permute(0, 2, 1, 3).contiguous()

    v, w = rnd(), rnd()
    Kv, Kw = ctx.apply_K(v), ctx.apply_K(w)

    def dot(a, b):
        wgt = torch.full((n[0] // 2 + 1,), 2.0, dtype=torch.float64, device="cuda")
        wgt[0] = 1.0; wgt[-1] = 1.0
        return float(((a.conj() * b).real * wgt).sum())

    a, b = dot(Kv, w), dot(v, Kw)
    assert abs(a - b) <= 1e-12 * abs(a)
    assert dot(Kv, v) > 0
    # null set: DC and the 7 Nyquist combinations are exactly zero
    for ky in (0, n[1] // 2):
        for kz in (0, n[2] // 2):
            for kx in (0, n[0] // 2):
                assert float(Kv[:, ky, kz, kx].abs().max()) == 0.0


# ------------------------------------------------------------------------------- solves


def _field_rel(a, b):
    return rel(a, b)


def test_solve_c1(dbf):
    cfg = configs.c1()
    ref = O.solve_small_strain(cfg["phase"], cfg["materials"], cfg["loads"][0], tol=1e-10)
    ctx = dbf.DBFFT(cfg["n"], kinematics="small")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    L = cfg["loads"][0]
    rep = ctx.solve_increment(L["target"], L["mask"])
    assert rep["converged"]
    assert abs(rep["cg_iters"] - ref["iters"]) <= 1
    assert rel(rep["macro_stress"], ref["mean_sig"]) <= 1e-9
    assert rel(ctx.get_field(dbf.FIELD_STRESS), ref["sig"]) <= 1e-8
    assert rel(ctx.get_field(dbf.FIELD_STRAIN), ref["eps"]) <= 1e-8
    assert rel(ctx.get_field(dbf.FIELD_U), O.displacement(ref["u_hat"])) <= 1e-8
    # caller-owned host buffers (bench.py's e2e reuses a pinned one)
    import torch
    buf = torch.empty((3,) + cfg["phase"].shape, dtype=torch.float64, pin_memory=True).numpy()
    assert ctx.get_field(dbf.FIELD_U, out=buf) is buf
    assert rel(buf, O.displacement(ref["u_hat"])) <= 1e-8
    buf9 = np.empty((9,) + cfg["phase"].shape)
    ctx.get_field(dbf.FIELD_STRESS, out=buf9)
    assert rel(buf9.reshape(3, 3, *cfg["phase"].shape), ref["sig"]) <= 1e-8
    with pytest.raises(ValueError):
        ctx.get_field(dbf.FIELD_U, out=np.empty(5))


@pytest.mark.parametrize("n", [32, 64])
def test_solve_c2_mixed(dbf, n):
    cfg = configs.c2(n=n, radius_vox=6 * n // 64)
    L = cfg["loads"][0]
    ref = O.solve_small_strain(cfg["phase"], cfg["materials"], L, tol=1e-10)
    ctx = dbf.DBFFT(cfg["n"], kinematics="small")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    rep = ctx.solve_increment(L["target"], L["mask"])
    assert rep["converged"]
    assert rel(rep["macro_stress"], ref["mean_sig"]) <= 1e-9
    assert rel(rep["macro_strain"], ref["mean_eps"]) <= 1e-9
    assert rep["macro_strain"][2, 2] == pytest.approx(1e-3, rel=1e-14)
    assert rel(ctx.get_field(dbf.FIELD_STRESS), ref["sig"]) <= 1e-8


def test_solve_c3_twin(dbf):
    cfg = configs.c3(n=32, grains=24)
    L = cfg["loads"][0]
    ref = O.solve_small_strain(cfg["phase"], cfg["materials"], L, tol=1e-10)
    ctx = dbf.DBFFT(cfg["n"], kinematics="small")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    rep = ctx.solve_increment(L["target"], L["mask"])
    assert rel(rep["macro_stress"], ref["mean_sig"]) <= 1e-9
    assert rel(ctx.get_field(dbf.FIELD_STRESS), ref["sig"]) <= 1e-8


def test_solve_c4_twin_newton(dbf):
    cfg = configs.c4(n=32, radius_vox=3, increments=10)
    st = O.FiniteStrainState(cfg["n"])
    ctx = dbf.DBFFT(cfg["n"], kinematics="finite")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    for L in cfg["loads"][:3]:
        ref = O.solve_finite_increment(st, cfg["phase"], cfg["materials"], L, tol=1e-10)
        rep = ctx.solve_increment(L["target"], L["mask"])
        assert rep["converged"] and ref["converged"]
        assert rep["newton_iters"] == ref["newton_iters"]
        assert rel(rep["macro_stress"], ref["mean_P"]) <= 1e-9
        assert rel(rep["macro_strain"], ref["mean_F"]) <= 1e-9
        assert rel(ctx.get_field(dbf.FIELD_STRAIN), ref["F"]) <= 1e-8
        assert rel(ctx.get_field(dbf.FIELD_STRESS), ref["P"]) <= 1e-8


def test_solve_tma_grids(dbf):
    """Full PCG solves (fused <p, Kp> in the F3 TMA kernel, both kinematics) on a grid whose
    column sweeps take the TMA path."""
    n = (32, 64, 128)
    ph = two_phase(n, 36)
    L = dict(target=np.diag([1e-3, 0.0, 0.0]), mask=np.zeros((3, 3), bool))
    ref = O.solve_small_strain(ph, ISO2, L, tol=1e-10)
    ctx = dbf.DBFFT(n, kinematics="small")
    ctx.set_phases(ph, ISO2)
    rep = ctx.solve_increment(L["target"], L["mask"])
    assert rep["converged"]
    assert rel(rep["macro_stress"], ref["mean_sig"]) <= 1e-9
    assert rel(ctx.get_field(dbf.FIELD_STRESS), ref["sig"]) <= 1e-8


def test_solve_c5_twin_j2(dbf):
    cfg = configs.c5(n=16, grains=6, increments=4)
    st = O.J2State(cfg["n"])
    ctx = dbf.DBFFT(cfg["n"], kinematics="small")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    for L in cfg["loads"]:
        ref = O.solve_j2_increment(st, cfg["phase"], cfg["materials"], L, 1.0, tol=1e-10)
        rep = ctx.solve_increment(L["target"], L["mask"], dt=1.0)
        assert rep["converged"]
        assert rel(rep["macro_stress"], ref["mean_sig"]) <= 1e-9
        assert rel(ctx.get_field(dbf.FIELD_STRESS), ref["sig"]) <= 1e-8


# ------------------------------------------------------------- preconditioner variants (8(f4))

NU2 = [dict(kind="iso", E=1.0, nu=0.2), dict(kind="iso", E=100.0, nu=0.45)]


@pytest.mark.parametrize("medium", [0, 1, 2])
def test_solve_reference_media(dbf, medium):
    """Reference medium of M (P:255 arithmetic; P:394 harmonic / Hill): the GPU takes the same
    PCG path as the oracle with the same medium (iteration count) and the same solution."""
    cfg = configs.c2(n=32, radius_vox=3)
    L = cfg["loads"][0]
    name = ("arithmetic", "harmonic", "hill")[medium]
    ref = O.solve_small_strain(cfg["phase"], NU2, L, tol=1e-10, medium=name)
    ctx = dbf.DBFFT(cfg["n"], kinematics="small")
    ctx.set_phases(cfg["phase"], NU2)
    rep = ctx.solve_increment(L["target"], L["mask"], precond_medium=medium)
    assert rep["converged"]
    # same M, same algorithm: counts agree up to round-off near the stop test (~135 iterations)
    assert abs(rep["cg_iters"] - ref["iters"]) <= max(2, 0.03 * ref["iters"]), (rep["cg_iters"], ref["iters"])
    assert rel(rep["macro_stress"], ref["mean_sig"]) <= 1e-9
    assert rel(ctx.get_field(dbf.FIELD_STRESS), ref["sig"]) <= 1e-8


@pytest.mark.parametrize("policy", [(1, 1), (2, 1), (3, 2)])
def test_solve_refresh_policies_finite(dbf, policy):
    """Mean-tangent refresh of M every Newton iteration / never (initial tangent) / every
    2nd increment: same Newton path and converged state as the oracle's per-increment
    refresh (the preconditioner never changes the solution)."""
    cfg = configs.c4(n=32, radius_vox=3, increments=10)
    st = O.FiniteStrainState(cfg["n"])
    ctx = dbf.DBFFT(cfg["n"], kinematics="finite")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    for L in cfg["loads"][:3]:
        ref = O.solve_finite_increment(st, cfg["phase"], cfg["materials"], L, tol=1e-10)
        rep = ctx.solve_increment(L["target"], L["mask"], precond_refresh=policy[0], precond_period=policy[1])
        assert rep["converged"] and rep["newton_iters"] == ref["newton_iters"]
        assert rel(rep["macro_stress"], ref["mean_P"]) <= 1e-9
        assert rel(ctx.get_field(dbf.FIELD_STRAIN), ref["F"]) <= 1e-8


def test_solve_refresh_initial_j2(dbf):
    cfg = configs.c5(n=16, grains=6, increments=4)
    st = O.J2State(cfg["n"])
    ctx = dbf.DBFFT(cfg["n"], kinematics="small")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    for L in cfg["loads"]:
        ref = O.solve_j2_increment(st, cfg["phase"], cfg["materials"], L, 1.0, tol=1e-10)
        rep = ctx.solve_increment(L["target"], L["mask"], dt=1.0, precond_refresh=2)
        assert rep["converged"]
        assert rel(rep["macro_stress"], ref["mean_sig"]) <= 1e-9
        assert rel(ctx.get_field(dbf.FIELD_STRESS), ref["sig"]) <= 1e-8


def test_precond_opts_rejected(dbf):
    cfg = configs.c4(n=8, radius_vox=1)
    ctx = dbf.DBFFT(cfg["n"], kinematics="finite")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    L = cfg["loads"][0]
    for bad in (dict(precond_medium=1), dict(precond_refresh=4), dict(precond_refresh=3, precond_period=0)):
        with pytest.raises(dbf.DBFFTError):
            ctx.solve_increment(L["target"], L["mask"], **bad)


# -------------------------------------------------- Saint Venant-Kirchhoff, SS3.3 porous run (8(f2))

@pytest.mark.parametrize("n", [(16, 8, 32), (32, 32, 32)])
def test_apply_K_svk_mixed(dbf, n):
    """K(x):grad du with SVK and neo-Hookean phases mixed in one cell (45-entry tangent)."""
    ph = two_phase(n, 41)
    mats = [dict(kind="svk", E=70.0, nu=0.3), dict(kind="neohooke", mu=1.0, kappa=2.5)]
    F = np.eye(3).reshape(3, 3, 1, 1, 1) + 0.1 * ms.random_field((3, 3, n[2], n[1], n[0]), 42)
    ctx = dbf.DBFFT(n, kinematics="finite")
    ctx.set_phases(ph, mats)
    ctx.eval_state(F.reshape(9, n[2], n[1], n[0]))
    u = ms.random_field((3, n[2], n[1], n[0]), 43)
    f = ctx.apply_K(to_gpu_spec(dbf, u))
    _, K = O.hyperelastic(F, ph, mats)
    ref, _ = O.apply_K(O.fft(u), K, O.frequency_grid(n), finite=True)
    assert rel(gpu_full(dbf, f, n[0]), ref) <= 1e-12


def test_solve_p33_porous_twin(dbf):
    """SS3.3 synthetic stand-in at 16^3: SVK matrix, 5 voids (vf 0.2) 100x softer,
    stretch 1 -> 2 along z in 5 increments with the other directions held."""
    from synth import configs as C
    cfg = C.p33(n=16)
    st = O.FiniteStrainState(cfg["n"])
    ctx = dbf.DBFFT(cfg["n"], kinematics="finite")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    for L in cfg["loads"]:
        ref = O.solve_finite_increment(st, cfg["phase"], cfg["materials"], L, tol=1e-10)
        rep = ctx.solve_increment(L["target"], L["mask"])
        assert rep["converged"] and ref["converged"]
        assert rep["newton_iters"] == ref["newton_iters"]
        assert rel(rep["macro_stress"], ref["mean_P"]) <= 1e-9
        assert rel(ctx.get_field(dbf.FIELD_STRAIN), ref["F"]) <= 1e-8
        assert rel(ctx.get_field(dbf.FIELD_STRESS), ref["P"]) <= 1e-8


# ------------------------------------------------------ residual monitors

@pytest.mark.parametrize("kin", ["small", "finite"])
@pytest.mark.parametrize("n", [(16, 8, 32), (32, 64, 128)])
def test_incompatibility_vs_oracle(dbf, kin, n):
    """max|curl curl eps| / max|curl F| of an incompatible random field: same value as the oracle."""
    fin = kin == "finite"
    f = ms.random_field((3, 3, n[2], n[1], n[0]), 61)
    if not fin:
        f = 0.5 * (f + np.swapaxes(f, 0, 1))
    ctx = dbf.DBFFT(n, kinematics=kin)
    mats = [dict(kind="neohooke", mu=1.0, kappa=2.5)] if fin else ISO2[:1]
    ctx.set_phases(np.zeros((n[2], n[1], n[0]), np.uint16), mats)
    got = ctx.incompatibility(f)
    ref = O.incompatibility(f, O.frequency_grid(n), finite=fin)
    assert got == pytest.approx(ref, rel=1e-12)


def test_residuals_after_solves(dbf):
    """The three residuals of a converged state (GPU) against the oracle's on its own solution:
    equilibrium at the PCG tolerance level on both, compatibility at round-off, loading 0."""
    # linear mixed control (c2 structure, 32^3)
    cfg = configs.c2(n=32, radius_vox=3)
    L = cfg["loads"][0]
    ctx = dbf.DBFFT(cfg["n"], kinematics="small")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    ctx.solve_increment(L["target"], L["mask"])
    r = ctx.residuals(L["target"], L["mask"])
    ref = O.solve_small_strain(cfg["phase"], cfg["materials"], L, tol=1e-10)
    XI = O.frequency_grid(cfg["n"])
    eq_ref = O.equilibrium_residual(ref["sig"], XI)
    assert r["equilibrium"] <= 2e-10 and eq_ref <= 2e-10
    xi2 = np.max(np.abs(XI)) ** 2  # round-off bound of a compatible field: ~ eps_machine |xi|^2
    assert r["compatibility"] <= 1e-14 * xi2
    assert O.incompatibility(ref["eps"], XI, finite=False) / np.linalg.norm(ref["mean_eps"]) <= 1e-14 * xi2
    assert r["loading"] <= 1e-10
    # finite strain: p33 twin, two increments
    from synth import configs as C
    cfg = C.p33(n=16)
    ctx = dbf.DBFFT(cfg["n"], kinematics="finite")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    st = O.FiniteStrainState(cfg["n"])
    for L in cfg["loads"][:2]:
        ctx.solve_increment(L["target"], L["mask"])
        ref = O.solve_finite_increment(st, cfg["phase"], cfg["materials"], L, tol=1e-10)
    r = ctx.residuals(L["target"], L["mask"])
    XI = O.frequency_grid(cfg["n"])
    assert r["loading"] <= 1e-14
    assert r["compatibility"] <= 1e-10
    assert O.incompatibility(ref["F"], XI, finite=True) / np.linalg.norm(ref["mean_F"] - np.eye(3)) <= 1e-10
    # equilibrium of the converged Newton state: both sides below the Newton-level tolerance
    eq_ref = O.equilibrium_residual(ref["P"], XI)
    assert r["equilibrium"] <= 1e-6 and eq_ref <= 1e-6
    assert r["equilibrium"] == pytest.approx(eq_ref, rel=0.5, abs=1e-11)


# ------------------------------------------------------ odd grids, Eq. 1 verbatim

ODD_GRIDS = [(15, 21, 27), (63, 15, 21), (21, 16, 63), (27, 27, 27)]


@pytest.mark.parametrize("n", ODD_GRIDS)
def test_apply_K_odd_small(dbf, n):
    """Mixed-radix (3, 5, 7) column and X passes, no Nyquist frequency (Eq. 1)."""
    ph = two_phase(n, 71)
    ctx = dbf.DBFFT(n, kinematics="small")
    ctx.set_phases(ph, ISO2)
    u = ms.random_field((3, n[2], n[1], n[0]), 72)
    f = ctx.apply_K(to_gpu_spec(dbf, u))
    ref, _ = O.apply_K(O.fft(u), O.stiffness_field(ph, ISO2), O.frequency_grid(n))
    assert rel(gpu_full(dbf, f, n[0]), ref) <= 1e-12


@pytest.mark.parametrize("n", ODD_GRIDS[:3])
def test_apply_K_odd_finite(dbf, n):
    ph = two_phase(n, 73)
    mats = [dict(kind="svk", E=70.0, nu=0.3), dict(kind="neohooke", mu=1.0, kappa=2.5)]
    F = np.eye(3).reshape(3, 3, 1, 1, 1) + 0.1 * ms.random_field((3, 3, n[2], n[1], n[0]), 74)
    ctx = dbf.DBFFT(n, kinematics="finite")
    ctx.set_phases(ph, mats)
    ctx.eval_state(F.reshape(9, n[2], n[1], n[0]))
    u = ms.random_field((3, n[2], n[1], n[0]), 75)
    f = ctx.apply_K(to_gpu_spec(dbf, u))
    _, K = O.hyperelastic(F, ph, mats)
    ref, _ = O.apply_K(O.fft(u), K, O.frequency_grid(n), finite=True)
    assert rel(gpu_full(dbf, f, n[0]), ref) <= 1e-12


def test_solve_odd_63_sphere_contrast(dbf):
    """The paper's SS3.1 cell: 63^3, centred sphere vf 0.2, E_m = 70, nu = 0.3, uniaxial
    strain 0.1 %, contrast k = 10 (and a soft k = 1e-2 case): GPU = oracle."""
    from synth import configs as C
    for k in (10.0, 1e-2):
        cfg = C.s31(n=63, contrast=k)
        L = cfg["loads"][0]
        ref = O.solve_small_strain(cfg["phase"], cfg["materials"], L, tol=1e-10)
        ctx = dbf.DBFFT(cfg["n"], kinematics="small")
        ctx.set_phases(cfg["phase"], cfg["materials"])
        rep = ctx.solve_increment(L["target"], L["mask"])
        assert rep["converged"]
        assert abs(rep["cg_iters"] - ref["iters"]) <= max(2, 0.03 * ref["iters"])
        assert rel(rep["macro_stress"], ref["mean_sig"]) <= 1e-9
        assert rel(ctx.get_field(dbf.FIELD_STRESS), ref["sig"]) <= 1e-8


def test_solve_odd_p33_twin(dbf):
    """SS3.3 on an odd grid (21^3 twin of the 63^3 cell): two increments, GPU = oracle."""
    from synth import configs as C
    cfg = C.p33(n=21)
    st = O.FiniteStrainState(cfg["n"])
    ctx = dbf.DBFFT(cfg["n"], kinematics="finite")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    for L in cfg["loads"][:2]:
        ref = O.solve_finite_increment(st, cfg["phase"], cfg["materials"], L, tol=1e-10)
        rep = ctx.solve_increment(L["target"], L["mask"])
        assert rep["converged"] and rep["newton_iters"] == ref["newton_iters"]
        assert rel(rep["macro_stress"], ref["mean_P"]) <= 1e-9
        assert rel(ctx.get_field(dbf.FIELD_STRAIN), ref["F"]) <= 1e-8


def test_residual_trace_vs_oracle(dbf):
    """Per-iteration equilibrium residual (the paper's Fig. div): the GPU's PCG history
    follows the oracle's iteration by iteration (same algorithm, round-off apart)."""
    for name in ("c1", "c2"):
        cfg = configs.c1() if name == "c1" else configs.c2(n=32, radius_vox=3)
        L = cfg["loads"][0]
        ref = O.solve_small_strain(cfg["phase"], cfg["materials"], L, tol=1e-10)
        ctx = dbf.DBFFT(cfg["n"], kinematics="small")
        ctx.set_phases(cfg["phase"], cfg["materials"])
        rep = ctx.solve_increment(L["target"], L["mask"])
        tr = ctx.trace()
        hist = np.asarray(ref["hist"])
        assert tr.shape[0] == rep["cg_iters"] + 1
        m = min(len(hist), tr.shape[0], 40)
        # early iterations agree tightly; PCG round-off grows with the iteration count
        assert np.allclose(tr[:m, 0], hist[:m], rtol=1e-6, atol=1e-12 * hist[0])  # atol: round-off floor
        assert tr[-1, 0] <= 1e-10
    # Newton: one PCG history per Newton iteration, concatenated
    cfg = configs.c4(n=16, radius_vox=2)
    ctx = dbf.DBFFT(cfg["n"], kinematics="finite")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    L = cfg["loads"][0]
    rep = ctx.solve_increment(L["target"], L["mask"])
    tr = ctx.trace()
    assert tr.shape[0] == rep["cg_iters"] + rep["newton_iters"]
    assert np.sum(tr[:, 0] <= 1e-10) >= rep["newton_iters"]


def test_solve_fused_update_finite(dbf, monkeypatch):
    """Finite-strain PCG with the residual update fused into the TMA F3 pass (z sweep of 256): same
    Newton path and state as the oracle, and as the unfused GPU path."""
    n = (16, 8, 256)
    ph = two_phase(n, 81)
    mats = [dict(kind="neohooke", mu=1.0, kappa=2.5), dict(kind="neohooke", mu=10.0, kappa=25.0)]
    loads = []
    for k in (1, 2):
        t = np.eye(3); t[2, 2] = 1.0 + 0.01 * k
        m = np.zeros((3, 3), bool); m[0, 0] = m[1, 1] = True
        loads.append(dict(target=np.where(m, 0.0, t), mask=m))
    st = O.FiniteStrainState(n)
    runs = {}
    for fused in ("1", "0"):
        monkeypatch.setenv("DBFFT_FUSED_UPDATE", fused)
        ctx = dbf.DBFFT(n, kinematics="finite")
        ctx.set_phases(ph, mats)
        runs[fused] = [ctx.solve_increment(L["target"], L["mask"]) for L in loads]
        runs[fused + "F"] = ctx.get_field(dbf.FIELD_STRAIN)
    for L, r1, r0 in zip(loads, runs["1"], runs["0"]):
        ref = O.solve_finite_increment(st, ph, mats, L, tol=1e-10)
        assert r1["converged"] and r1["newton_iters"] == ref["newton_iters"] == r0["newton_iters"]
        assert abs(r1["cg_iters"] - r0["cg_iters"]) <= 2
        assert rel(r1["macro_stress"], ref["mean_P"]) <= 1e-9
    assert rel(runs["1F"], ref["F"]) <= 1e-8


# ------------------------------------------------------------- full size and degenerate cases

def _half_xi(n):
    """Eq. 1 frequencies on the product's half-spectrum layout [ky][kz][kx <= n1/2] (oracle tables)."""
    fx = O.axis_frequencies(n[0], 1.0)[: n[0] // 2 + 1]
    fy = O.axis_frequencies(n[1], 1.0)
    fz = O.axis_frequencies(n[2], 1.0)
    X, Z, Y = np.broadcast_arrays(fx[None, None, :], fz[None, :, None], fy[:, None, None])
    return np.stack([X, Y, Z])  # XI[a] = xi_a (a = x, y, z) on [ky][kz][kx]


@pytest.mark.parametrize("kin", ["small", "finite"])
def test_apply_K_full_size_homogeneous(dbf, kin):
    """At c4's full 256^3 size, in the bench's launch configuration: a homogeneous medium makes the
    operator diagonal in Fourier space, f(xi) = A(xi) u(xi) with A = xi . C . xi (closed form at
    every one of the 8.5M points), so the whole FFT chain is checked element by element."""
    n = (256, 256, 256)
    if kin == "small":
        mats = [dict(kind="iso", E=3.0, nu=0.28)]
        C = O.isotropic_stiffness(3.0, 0.28)
    else:  # neo-Hookean at F = I: K = isotropic (lam = kappa - 2 mu / 3, mu)
        mats = [dict(kind="neohooke", mu=1.3, kappa=3.1)]
        C = O.isotropic_from_lame(3.1 - 2.0 * 1.3 / 3.0, 1.3)
    ctx = dbf.DBFFT(n, kinematics=kin)
    ctx.set_phases(np.zeros((n[2], n[1], n[0]), np.uint16), mats)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn((3, n[2], n[1], n[0]), dtype=torch.float64, device="cuda", generator=g)
    u = (torch.fft.rfftn(x, dim=(1, 2, 3)) / x[0].numel()).permute(0, 2, 1, 3).contiguous()  # [3][ky][kz][kx]
    del x
    f = ctx.apply_K(u).cpu().numpy()
    un = u.cpu().numpy()
    XI = _half_xi(n)                                    # [a][ky][kz][kx]
    A = np.einsum("ijkl,j...,l...->ik...", C, XI, XI)   # [3,3][ky][kz][kx]
    ref = np.einsum("ik...,k...->i...", A, un)
    assert rel(f, ref) <= 1e-12


def test_degenerate_homogeneous_and_zero_load(dbf):
    """Homogeneous media converge with no PCG iteration to the uniform Hooke state (P7), for linear
    strain control and finite-strain mixed control; a zero load returns the zero state."""
    n = (32, 16, 64)
    ph = np.zeros((n[2], n[1], n[0]), np.uint16)
    ctx = dbf.DBFFT(n, kinematics="small")
    ctx.set_phases(ph, [dict(kind="iso", E=2.0, nu=0.3)])
    t = np.array([[1e-3, 2e-4, 0], [2e-4, -5e-4, 0], [0, 0, 3e-4]])
    rep = ctx.solve_increment(t, np.zeros((3, 3), bool))
    assert rep["converged"] and rep["cg_iters"] == 0
    sig = np.einsum("ijkl,kl->ij", O.isotropic_stiffness(2.0, 0.3), t)
    assert np.abs(ctx.get_field(dbf.FIELD_STRESS) - sig.reshape(3, 3, 1, 1, 1)).max() <= 1e-15 * np.abs(sig).max() * 10
    rep = ctx.solve_increment(np.zeros((3, 3)), np.zeros((3, 3), bool))
    assert rep["converged"] and rep["cg_iters"] == 0 and np.abs(ctx.get_field(dbf.FIELD_STRESS)).max() == 0.0
    ctx = dbf.DBFFT(n, kinematics="finite")
    ctx.set_phases(ph, [dict(kind="neohooke", mu=1.0, kappa=2.5)])
    m = np.zeros((3, 3), bool); m[0, 0] = m[1, 1] = True
    tf = np.eye(3); tf[2, 2] = 1.05; tf[0, 0] = tf[1, 1] = 0.0
    rep = ctx.solve_increment(tf, m)
    # mixed control: the macro block is solved exactly by (P Cbar P)^-1 - one PCG step per Newton step
    assert rep["converged"] and rep["cg_iters"] <= rep["newton_iters"]
    assert abs(rep["macro_stress"][0, 0]) <= 1e-10 and abs(rep["macro_stress"][1, 1]) <= 1e-10
    F = ctx.get_field(dbf.FIELD_STRAIN)
    assert np.abs(F - F[:, :, :1, :1, :1]).max() <= 1e-14  # uniform deformation


def test_invalid_inputs_rejected(dbf):
    """Bad grids, out-of-range phase ids and material/kinematics mismatches fail loudly."""
    with pytest.raises(dbf.DBFFTError):
        dbf.DBFFT((12, 16, 16), kinematics="small")
    with pytest.raises(dbf.DBFFTError):
        dbf.DBFFT((16, 16, 1024), kinematics="small")
    ctx = dbf.DBFFT((8, 8, 8), kinematics="small")
    with pytest.raises(dbf.DBFFTError):
        ctx.set_phases(np.full((8, 8, 8), 3, np.uint16), ISO2)
    with pytest.raises(dbf.DBFFTError):
        ctx.set_phases(np.zeros((8, 8, 8), np.uint16), [dict(kind="neohooke", mu=1.0, kappa=2.0)])
