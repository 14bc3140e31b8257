"""C-ABI surface on the GPU: the per-voxel tangent field (DBFFT_FIELD_TANGENT) against the oracle's
constitutive tangents, the env allocator hooks (torch's caching allocator vs cudaMalloc), argument
validation of the binding, dbfft_info, and non-convergence reported as a status.  Marked `gpu`."""
import numpy as np
import pytest

from oracle import dbfft_oracle as O
from spectra import half_spectrum
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


def two_phase(n, seed, frac=0.4):
    u = ms.SplitMix64(seed).uniform(n[0] * n[1] * n[2]).reshape(n[2], n[1], n[0])
    return (u < frac).astype(np.uint16)


N = (16, 8, 32)
SHP = (N[2], N[1], N[0])


@pytest.mark.parametrize("tangent", ["compact", "full"])
def test_tangent_field_neohooke(dbf, tangent, monkeypatch):
    """dP/dF per voxel (R14) after eval_state at a random F: both tangent storages."""
    monkeypatch.setenv("DBFFT_TANGENT", tangent)
    ph = two_phase(N, 61)
    mats = [dict(kind="neohooke", mu=1.0, kappa=2.5), dict(kind="neohooke", mu=10.0, kappa=25.0)]
    F = np.eye(3).reshape(3, 3, 1, 1, 1) + 0.1 * ms.random_field((3, 3) + SHP, 62)
    ctx = dbf.DBFFT(N, kinematics="finite")
    ctx.set_phases(ph, mats)
    ctx.eval_state(F.reshape((9,) + SHP))
    K = ctx.get_field(dbf.FIELD_TANGENT)
    _, Kref = O.neo_hookean(F, np.array([1.0, 10.0])[ph], np.array([2.5, 25.0])[ph])
    assert K.shape == Kref.shape and rel(K, Kref) <= 1e-13


def test_tangent_field_svk_neohooke_mix(dbf):
    ph = two_phase(N, 63)
    mats = [dict(kind="svk", E=70.0, nu=0.3), dict(kind="neohooke", mu=3.0, kappa=7.0)]
    F = np.eye(3).reshape(3, 3, 1, 1, 1) + 0.1 * ms.random_field((3, 3) + SHP, 64)
    ctx = dbf.DBFFT(N, kinematics="finite")
    ctx.set_phases(ph, mats)
    ctx.eval_state(F.reshape((9,) + SHP))
    _, Kref = O.hyperelastic(F, ph, mats)
    assert rel(ctx.get_field(dbf.FIELD_TANGENT), Kref) <= 1e-13


def test_tangent_field_j2(dbf):
    """The J2 algorithmic tangent (R16) at a strain field with plastic and elastic voxels."""
    ph = two_phase(N, 65, 0.5)
    sy = np.array([300.0, 200.0])
    mats = [dict(kind="j2", E=2e5, nu=0.3, sigma_y=float(s), n=20.0, edot0=1e-3) for s in sy]
    eps = 2e-3 * np.diag([-0.5, -0.5, 1.0]).reshape(3, 3, 1, 1, 1) + 5e-4 * ms.random_field((3, 3) + SHP, 66)
    eps = 0.5 * (eps + np.swapaxes(eps, 0, 1))
    ctx = dbf.DBFFT(N, kinematics="small")
    ctx.set_phases(ph, mats)
    ctx.eval_state(eps.reshape((9,) + SHP), dt=1.0)
    _, C, _, dp = O.j2_perzyna(eps, np.zeros_like(eps), 2e5, 0.3, sy[ph], 20.0, 1e-3, 1.0)
    assert 0.2 < np.mean(dp > 0) < 1.0
    assert rel(ctx.get_field(dbf.FIELD_TANGENT), C) <= 1e-12


def test_tangent_field_cubic_and_loopback(dbf):
    """Rotated cubic grains (linear): the phase stiffness per voxel; loopback slabs give the same."""
    cfg = configs.c3(n=16, grains=5)
    ref = O.stiffness_field(cfg["phase"], cfg["materials"])
    for kw in ({}, dict(world=2, loopback=True)):
        ctx = dbf.DBFFT(cfg["n"], kinematics="small", **kw)
        ctx.set_phases(cfg["phase"], cfg["materials"])
        assert rel(ctx.get_field(dbf.FIELD_TANGENT), ref) <= 1e-14


def test_allocator_hooks(dbf):
    """dbfft_env dev_alloc / dev_free: with the torch allocator the ctx's buffers are torch memory
    (memory_allocated grows while the ctx lives, shrinks after close); both allocators compute
    the same operator."""
    n = (32, 16, 16)
    ph = two_phase(n, 67)
    mats = [dict(kind="iso", E=1.0, nu=0.3), dict(kind="iso", E=5.0, nu=0.2)]
    u = torch.from_numpy(half_spectrum(ms.random_field((3, n[2], n[1], n[0]), 68))).cuda()
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    out = {}
    for alloc in ("torch", "cuda"):
        ctx = dbf.DBFFT(n, kinematics="small", allocator=alloc)
        ctx.set_phases(ph, mats)
        grown = torch.cuda.memory_allocated() - base
        if alloc == "torch":
            assert grown > 7 * 3 * 16 * (n[0] // 2 + 1) * n[1] * n[2]   # at least the 7 spectral vectors
        else:
            assert grown < 1 << 20
        out[alloc] = ctx.apply_K(u).cpu().numpy()
        ctx.close()
        torch.cuda.synchronize()
        assert torch.cuda.memory_allocated() - base < 1 << 20
    assert np.array_equal(out["torch"], out["cuda"])


def test_binding_validates_arguments(dbf):
    n = (16, 8, 8)
    ctx = dbf.DBFFT(n, kinematics="small")
    mats = [dict(kind="iso", E=1.0, nu=0.3)]
    with pytest.raises(ValueError):
        ctx.set_phases(torch.zeros(n[::-1], dtype=torch.int64, device="cuda") - 1, mats)   # negative ids
    with pytest.raises(ValueError):
        ctx.set_phases(np.zeros((4, 4, 4), np.uint16), mats)                                   # wrong size
    ctx.set_phases(torch.zeros(n[::-1], dtype=torch.int64, device="cuda"), mats)             # int64 on device: fine
    good = ctx.empty_spectral()
    with pytest.raises(ValueError):
        ctx.apply_K(good.to(torch.complex64))
    with pytest.raises(ValueError):
        ctx.apply_K(good[:, :, :, :-1])
    with pytest.raises(ValueError):
        ctx.apply_K(good.cpu())
    with pytest.raises(ValueError):
        ctx.apply_K(good, out=torch.empty((3, 8, 8, 8), dtype=torch.complex128, device="cuda"))
    info = ctx.info()
    assert info["world"] == 1 and info["transport"] == "none" and info["sms"] > 0


def test_not_converged_is_a_status(dbf):
    """max_cg exhausted: DBFFT_E_NOT_CONVERGED with the report filled and the state rolled back."""
    cfg = configs.c2(n=32, radius_vox=3)
    ctx = dbf.DBFFT(cfg["n"], kinematics="small")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    L = cfg["loads"][0]
    rep = ctx.solve_increment(L["target"], L["mask"], raise_on_error=False, max_cg=3)
    assert rep["status"] == "E_NOT_CONVERGED" and not rep["converged"] and rep["cg_iters"] >= 3
    assert np.allclose(ctx.get_field(dbf.FIELD_U_HAT).abs().cpu().numpy(), 0.0)
    rep = ctx.solve_increment(L["target"], L["mask"])
    assert rep["converged"]


@pytest.mark.parametrize("which", ["finite", "j2", "linear_loopback"])
def test_checkpoint_restore_resumes_exactly(dbf, which):
    """dbfft_checkpoint after two increments; a fresh ctx restored from it runs the third increment
    bit-identically to the original ctx (same Newton / PCG counts, fields, macro values)."""
    if which == "finite":
        cfg, kin, kw = configs.c4(n=16, radius_vox=2), "finite", {}
    elif which == "j2":
        cfg, kin, kw = configs.c5(n=16, grains=4, increments=3), "small", {}
    else:
        cfg, kin, kw = configs.c2(n=32, radius_vox=3), "small", dict(world=2, loopback=True)
        cfg["loads"] = [dict(target=t * cfg["loads"][0]["target"], mask=cfg["loads"][0]["mask"]) for t in (1, 2, 3)]
    loads = cfg["loads"][:3]
    a = dbf.DBFFT(cfg["n"], kinematics=kin, **kw)
    a.set_phases(cfg["phase"], cfg["materials"])
    for L in loads[:2]:
        a.solve_increment(L["target"], L["mask"], dt=1.0)
    blob = a.checkpoint()
    ra = a.solve_increment(loads[2]["target"], loads[2]["mask"], dt=1.0)
    b = dbf.DBFFT(cfg["n"], kinematics=kin, **kw)
    b.set_phases(cfg["phase"], cfg["materials"])
    b.restore(blob)
    rb = b.solve_increment(loads[2]["target"], loads[2]["mask"], dt=1.0)
    assert (ra["cg_iters"], ra["newton_iters"]) == (rb["cg_iters"], rb["newton_iters"])
    assert np.array_equal(ra["macro_stress"], rb["macro_stress"])
    for f in (dbf.FIELD_STRAIN, dbf.FIELD_STRESS, dbf.FIELD_U):
        assert np.array_equal(a.get_field(f), b.get_field(f))
    with pytest.raises(dbf.DBFFTError):
        b.restore(blob[:-8])
