"""Slab-decomposed (multi-rank) DBFFT through the C ABI in loopback mode: P virtual ranks in one
process on one GPU run the exact distributed data path (rank-chunked z/y passes, the two
exchanges per operator, per-rank partial sums + all-reduce) with device copies standing in for
NCCL.  Compared against the oracle and against P = 1.  Marked `gpu`."""
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


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("n", [(16, 8, 32), (32, 32, 16), (32, 128, 256), (16, 32, 512)])
def test_apply_K_small_loopback(dbf, n, P):
    if n[1] % P or n[2] % P:
        pytest.skip("P must divide n2 and n3")
    ph = two_phase(n, 21)
    ctx = dbf.DBFFT(n, kinematics="small", world=P, loopback=True)
    ctx.set_phases(ph, ISO2)
    u = ms.random_field((3, n[2], n[1], n[0]), 22)
    f = ctx.apply_K(torch.from_numpy(half_spectrum(u)).cuda())
    ref, _ = O.apply_K(O.fft(u), O.stiffness_field(ph, ISO2), O.frequency_grid(n))
    assert rel(full_from_half(f.cpu().numpy(), n[0]), ref) <= 1e-12
    # preconditioner with the rank-local ky offsets of xi_y
    z = ctx.precond(torch.from_numpy(half_spectrum(u)).cuda())
    zref = O.precondition(O.fft(u), O.volume_average(O.stiffness_field(ph, ISO2)), O.frequency_grid(n))
    assert rel(full_from_half(z.cpu().numpy(), n[0]), zref) <= 1e-12


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
    f = ctx.apply_K(torch.from_numpy(half_spectrum(u)).cuda())
    _, K = O.neo_hookean(F, np.array([1.0, 10.0])[ph], np.array([2.5, 25.0])[ph])
    ref, _ = O.apply_K(O.fft(u), K, O.frequency_grid(n), finite=True)
    assert rel(full_from_half(f.cpu().numpy(), n[0]), ref) <= 1e-12


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


# ---------------------------------------------------------------- peer transport
# The z-inverse and y-forward passes store their chunk for rank d straight into rank d's receive
# buffer through a VMM window (peer.cuh); in loopback the windows map the other virtual slabs'
# buffers on the same GPU, so the kernels run the exact addressing (padded chunk stride, window
# chunks backed by different physical allocations) of the multi-GPU path.  The arithmetic is the
# NCCL transport's, so the results must agree bit for bit.

@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("n", [(16, 8, 32), (32, 128, 256), (16, 32, 512)])
def test_apply_K_small_peer(dbf, n, P):
    if n[1] % P or n[2] % P:
        pytest.skip("P must divide n2 and n3")
    ph = two_phase(n, 31)
    u_real = ms.random_field((3, n[2], n[1], n[0]), 32)
    u = torch.from_numpy(half_spectrum(u_real)).cuda()
    out = {}
    for tr in ("nccl", "peer"):
        ctx = dbf.DBFFT(n, kinematics="small", world=P, loopback=True, transport=tr)
        ctx.set_phases(ph, ISO2)
        out[tr] = ctx.apply_K(u).cpu().numpy()
        ctx.close()
    assert np.array_equal(out["peer"], out["nccl"])
    ref, _ = O.apply_K(O.fft(u_real), O.stiffness_field(ph, ISO2), O.frequency_grid(n))
    assert rel(full_from_half(out["peer"], n[0]), ref) <= 1e-12


@pytest.mark.parametrize("P", [2, 4])
def test_apply_K_finite_peer(dbf, P):
    n = (16, 16, 64)
    ph = two_phase(n, 33)
    mats = [dict(kind="neohooke", mu=1.0, kappa=2.5), dict(kind="neohooke", mu=10.0, kappa=25.0)]
    F = np.eye(3).reshape(3, 3, 1, 1, 1) + 0.1 * ms.random_field((3, 3, n[2], n[1], n[0]), 34)
    u = ms.random_field((3, n[2], n[1], n[0]), 35)
    ctx = dbf.DBFFT(n, kinematics="finite", world=P, loopback=True, transport="peer")
    ctx.set_phases(ph, mats)
    ctx.eval_state(F.reshape(9, n[2], n[1], n[0]))
    f = ctx.apply_K(torch.from_numpy(half_spectrum(u)).cuda())
    _, K = O.neo_hookean(F, np.array([1.0, 10.0])[ph], np.array([2.5, 25.0])[ph])
    ref, _ = O.apply_K(O.fft(u), K, O.frequency_grid(n), finite=True)
    assert rel(full_from_half(f.cpu().numpy(), n[0]), ref) <= 1e-12


def test_solve_c4_twin_peer_matches_nccl(dbf):
    """Two finite-strain increments (fused PCG update, Newton residuals, monitors, get_field all
    route through the windows): identical iteration counts and bit-identical fields."""
    cfg = configs.c4(n=32, radius_vox=3)
    st = O.FiniteStrainState(cfg["n"])
    out = {}
    for tr in ("nccl", "peer"):
        ctx = dbf.DBFFT(cfg["n"], kinematics="finite", world=4, loopback=True, transport=tr)
        ctx.set_phases(cfg["phase"], cfg["materials"])
        reps = [ctx.solve_increment(L["target"], L["mask"]) for L in cfg["loads"][:2]]
        L = cfg["loads"][1]
        out[tr] = (reps, ctx.get_field(dbf.FIELD_STRESS), ctx.get_field(dbf.FIELD_U),
                   ctx.residuals(L["target"], L["mask"]), ctx.incompatibility(ctx.get_field(dbf.FIELD_STRAIN)))
        ctx.close()
    for a, b in zip(out["peer"][0], out["nccl"][0]):
        assert a["cg_iters"] == b["cg_iters"] and a["newton_iters"] == b["newton_iters"]
        assert np.array_equal(a["macro_stress"], b["macro_stress"])
    assert np.array_equal(out["peer"][1], out["nccl"][1])
    assert np.array_equal(out["peer"][2], out["nccl"][2])
    assert out["peer"][3] == out["nccl"][3] and out["peer"][4] == out["nccl"][4]
    for L in cfg["loads"][:2]:
        ref = O.solve_finite_increment(st, cfg["phase"], cfg["materials"], L, tol=1e-10)
    assert rel(out["peer"][1], ref["P"]) <= 1e-8


def test_solve_c5_twin_peer(dbf):
    cfg = configs.c5(n=16, grains=6, increments=2)
    st = O.J2State(cfg["n"])
    ctx = dbf.DBFFT(cfg["n"], kinematics="small", world=8, loopback=True, transport="peer")
    ctx.set_phases(cfg["phase"], cfg["materials"])
    for L in cfg["loads"]:
        ref = O.solve_j2_increment(st, cfg["phase"], cfg["materials"], L, 1.0, tol=1e-10)
        rep = ctx.solve_increment(L["target"], L["mask"], dt=1.0)
        assert rep["converged"]
        assert rel(rep["macro_stress"], ref["mean_sig"]) <= 1e-9
        assert rel(ctx.get_field(dbf.FIELD_STRESS), ref["sig"]) <= 1e-8


def _probe_worker(rank, world, tag, bar, q):
    try:
        import ctypes
        from paper_1905_12725_b200 import dbfft
        lib = dbfft.load_library()
        h = ctypes.c_void_p()
        st = lib.dbfft_peer_probe_open(tag.encode(), rank, world, 0, ctypes.byref(h))
        if st != 0:
            q.put((rank, "open %d: %s" % (st, lib.dbfft_last_error(None).decode())))
            bar.wait()
            bar.wait()
            return
        bar.wait()  # every process stored through its window
        bad = ctypes.c_int32(-1)
        st = lib.dbfft_peer_probe_check(h, ctypes.byref(bad))
        bar.wait()  # nobody unmaps while others still read
        lib.dbfft_peer_probe_close(h)
        q.put((rank, bad.value if st == 0 else "check %d" % st))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, repr(exc)))


@pytest.mark.parametrize("world", [2, 4])
def test_peer_windows_across_processes(dbf, world):
    """The multi-process half of the peer transport on one GPU: VMM export as POSIX fds, the
    SCM_RIGHTS all-gather, import and window mapping in separate processes; stores through the
    windows land in the right chunk of the right process's buffer."""
    import multiprocessing as mp
    import os
    ctx = mp.get_context("spawn")
    q, bar = ctx.Queue(), ctx.Barrier(world)
    tag = f"probe-{os.getpid()}-{world}"
    procs = [ctx.Process(target=_probe_worker, args=(r, world, tag, bar, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] == 0 for r in range(world)), res


@pytest.mark.parametrize("world,transport", [(1, "nccl"), (2, "nccl"), (4, "peer")])
def test_kx_pitch_padding_bit_identical(dbf, world, transport, monkeypatch):
    """DBFFT_KX_PAD=1 pads the kx pitch of the intermediate layouts (X1, B, X2) to 128-byte rows;
    the arithmetic is unchanged, so a finite-strain increment must agree bit for bit."""
    cfg = configs.c4(n=32, radius_vox=3)
    L = cfg["loads"][0]
    out = {}
    for pad in ("0", "1"):
        monkeypatch.setenv("DBFFT_KX_PAD", pad)
        ctx = dbf.DBFFT(cfg["n"], kinematics="finite", world=world, loopback=world > 1,
                        transport=transport)
        ctx.set_phases(cfg["phase"], cfg["materials"])
        rep = ctx.solve_increment(L["target"], L["mask"])
        out[pad] = (rep["cg_iters"], rep["macro_stress"], ctx.get_field(dbf.FIELD_STRESS))
        ctx.close()
    assert out["0"][0] == out["1"][0]
    assert np.array_equal(out["0"][1], out["1"][1]) and np.array_equal(out["0"][2], out["1"][2])
