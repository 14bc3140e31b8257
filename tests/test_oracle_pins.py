"""Pins of the CPU oracle against what the paper and mathematics fix.

Each test pins the oracle to something other than itself: closed forms,
invariants, brute force, dense direct solves and textbook special cases.
No GPU needed (-m "not gpu")."""
import json
import os

import numpy as np
import pytest
from scipy.optimize import brentq

from oracle import dbfft_oracle as O
from synth import configs, microstructure as ms

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _two_phase_random(n, seed, frac=0.3):
    u = ms.SplitMix64(seed).uniform(n[0] * n[1] * n[2]).reshape(n[2], n[1], n[0])
    return (u < frac).astype(np.uint16)


ISO2 = [dict(kind="iso", E=1.0, nu=0.3), dict(kind="iso", E=10.0, nu=0.3)]

# ---------------------------------------------------------------- P1 grid/FFT


def test_P1_frequencies_eq1():
    # Eq. (1) evaluated directly, odd grids
    assert sorted(O.axis_frequencies(3, 1.0)) == pytest.approx([-2 * np.pi, 0.0, 2 * np.pi])
    assert sorted(O.axis_frequencies(5, 2.0)) == pytest.approx([-2 * np.pi, -np.pi, 0, np.pi, 2 * np.pi])
    # native order: slot k holds kappa = k (k < N/2), k - N otherwise; Nyquist zeroed (R1)
    f8 = O.axis_frequencies(8, 1.0) / (2 * np.pi)
    assert list(f8) == [0, 1, 2, 3, 0, -3, -2, -1]
    f5 = O.axis_frequencies(5, 1.0) / (2 * np.pi)
    assert f5 == pytest.approx([0, 1, 2, -2, -1])
    # exactly one zero per odd axis
    assert np.sum(O.axis_frequencies(7) == 0) == 1
    # null set: 8 modes on an all-even grid, 1 on an odd one (R1)
    assert O.null_set(O.frequency_grid((8, 4, 6))).sum() == 8
    assert O.null_set(O.frequency_grid((5, 3, 7))).sum() == 1


def test_P1_fft_normalisation_parseval():
    n = (6, 5, 4)
    a = ms.random_field((3, 4, 5, 6), 11)
    b = ms.random_field((3, 4, 5, 6), 12)
    c = np.full((4, 5, 6), 2.5)
    ch = O.fft(c)
    assert ch[0, 0, 0] == pytest.approx(2.5)
    assert np.max(np.abs(ch.ravel()[1:])) < 1e-14
    assert np.max(np.abs(O.ifft(O.fft(a)) - a)) < 1e-13
    assert O.inner(O.fft(a), O.fft(b)) == pytest.approx(np.mean(np.sum(a * b, axis=0)), rel=1e-12)
    # single cosine mode: exactly two conjugate entries
    x = (np.arange(6) + 0.5) / 6
    cosf = np.broadcast_to(np.cos(2 * np.pi * 2 * x), (4, 5, 6))
    h = O.fft(cosf)
    nz = np.argwhere(np.abs(h) > 1e-12)
    assert len(nz) == 2 and np.allclose(h[tuple(nz[0])], np.conj(h[tuple(nz[1])]))


# ---------------------------------------------------------------- P2 operators


def _mode(n, k, axis):
    xs = ms.voxel_centres(n)
    g = [xs[0][None, None, :], xs[1][None, :, None], xs[2][:, None, None]]
    return np.broadcast_to(np.sin(2 * np.pi * k * g[axis]), (n[2], n[1], n[0])), \
        np.broadcast_to(2 * np.pi * k * np.cos(2 * np.pi * k * g[axis]), (n[2], n[1], n[0]))


@pytest.mark.parametrize("k,axis", [(1, 0), (3, 1), (2, 2)])
def test_P2_analytic_sine_derivatives(k, axis):
    n = (16, 8, 12)
    XI = O.frequency_grid(n)
    s, ds = _mode(n, k, axis)
    zero = np.zeros_like(s)
    # u = sin(2 pi k x_a) e_a  ->  eps_aa = 2 pi k cos, all other components 0
    u = np.stack([s if c == axis else zero for c in range(3)])
    eps = O.ifft(O.sym_grad_hat(O.fft(u), XI))
    for i in range(3):
        for j in range(3):
            ref = ds if (i == j == axis) else zero
            assert np.max(np.abs(eps[i, j] - ref)) < 1e-10
    # u = sin(2 pi k x_a) e_b (b != a): eps_ab = eps_ba = 1/2 d; G_ba = d, G_ab = 0
    b = (axis + 1) % 3
    u = np.stack([s if c == b else zero for c in range(3)])
    eps = O.ifft(O.sym_grad_hat(O.fft(u), XI))
    G = O.ifft(O.grad_hat(O.fft(u), XI))
    assert np.max(np.abs(eps[axis, b] - 0.5 * ds)) < 1e-10
    assert np.max(np.abs(eps[b, axis] - 0.5 * ds)) < 1e-10
    assert np.max(np.abs(G[b, axis] - ds)) < 1e-10
    assert np.max(np.abs(G[axis, b])) < 1e-10
    # divergence of sigma_{b a} = sin(2 pi k x_a) (non-symmetric) -> (div sigma)_b = d, others 0
    sig = np.zeros((3, 3) + s.shape)
    sig[b, axis] = s
    f = O.ifft(O.div_hat(O.fft(sig), XI))
    assert np.max(np.abs(f[b] - ds)) < 1e-10
    assert np.max(np.abs(f[axis])) < 1e-10


def test_P2_adjointness_and_mean_annihilation():
    n = (8, 6, 10)
    XI = O.frequency_grid(n)
    u = ms.random_field((3, 10, 6, 8), 21)
    t = ms.random_field((3, 3, 10, 6, 8), 22)
    t = 0.5 * (t + np.swapaxes(t, 0, 1))
    lhs = np.mean(np.sum(O.ifft(O.div_hat(O.fft(t), XI)) * u, axis=0))
    rhs = -np.mean(np.sum(t * O.ifft(O.sym_grad_hat(O.fft(u), XI)), axis=(0, 1)))
    assert lhs == pytest.approx(rhs, rel=1e-12)
    Z = O.null_set(XI)
    assert np.all(O.sym_grad_hat(O.fft(u), XI)[:, :, Z] == 0)
    assert np.all(O.div_hat(O.fft(t), XI)[:, Z] == 0)


# ---------------------------------------------------------------- materials


def test_P7_hooke_golden():
    g = _gold("hooke_iso.json")
    C = O.isotropic_stiffness(g["E"], g["nu"])
    eps = np.zeros((3, 3)); eps[0, 0] = g["eps11"]
    sig = np.einsum("ijkl,kl->ij", C, eps)
    assert sig[0, 0] == pytest.approx(g["sigma11"], rel=1e-14)
    assert sig[1, 1] == pytest.approx(g["sigma22"], rel=1e-14)
    assert sig[2, 2] == pytest.approx(g["sigma22"], rel=1e-14)
    assert np.count_nonzero(np.abs(sig) > 1e-18) == 3
    # minor and major symmetry
    assert np.allclose(C, np.swapaxes(C, 0, 1)) and np.allclose(C, np.transpose(C, (2, 3, 0, 1)))


def test_cubic_rotation_golden():
    g = _gold("cubic_cu.json")
    C11, C12, C44 = g["C11"], g["C12"], g["C44"]
    C = O.cubic_stiffness(C11, C12, C44, np.eye(3))
    assert C[0, 0, 0, 0] == C11 and C[0, 0, 1, 1] == C12 and C[1, 2, 1, 2] == C44 and C[1, 2, 2, 1] == C44
    c, s = np.cos(np.pi / 4), np.sin(np.pi / 4)
    Rz = np.array([[c, -s, 0], [s, c, 0], [0, 0, 1]])
    C45 = O.cubic_stiffness(C11, C12, C44, Rz)
    assert C45[0, 0, 0, 0] == pytest.approx(g["C1111_45z"], rel=1e-13)
    assert C45[0, 0, 1, 1] == pytest.approx(g["C1122_45z"], rel=1e-13)
    R90 = np.array([[0, -1, 0], [1, 0, 0], [0, 0, 1.0]])
    assert np.allclose(O.cubic_stiffness(C11, C12, C44, R90), C)
    R = ms.random_rotations(5, 7)
    for Ri in R:
        Cr = O.cubic_stiffness(C11, C12, C44, Ri)
        iijj = np.einsum("iijj->", Cr)
        ijij = np.einsum("ijij->", Cr)
        assert iijj / 9 == pytest.approx(g["K"], rel=1e-13)
        assert (ijij - iijj / 3) / 10 == pytest.approx(g["G_V"], rel=1e-13)


def _fd_check(fun, F0, K, h=1e-6):
    err = 0.0
    for k in range(3):
        for l in range(3):
            dF = np.zeros((3, 3)); dF[k, l] = h
            num = (fun(F0 + dF) - fun(F0 - dF)) / (2 * h)
            err = max(err, np.max(np.abs(num - K[:, :, k, l])))
    return err


def test_P15_neo_hookean():
    mu, kappa = 1.0, 2.5
    P, K = O.neo_hookean(np.eye(3).reshape(3, 3, 1), mu, kappa)
    assert np.max(np.abs(P)) < 1e-15
    assert np.allclose(K[..., 0], O.isotropic_from_lame(kappa - 2 * mu / 3, mu), atol=1e-14)
    rng = ms.SplitMix64(5)
    for _ in range(3):
        F0 = np.eye(3) + 0.2 * rng.normal(9).reshape(3, 3)
        P0, K0 = O.neo_hookean(F0.reshape(3, 3, 1), mu, kappa)
        err = _fd_check(lambda F: O.neo_hookean(F.reshape(3, 3, 1), mu, kappa)[0][..., 0], F0, K0[..., 0])
        assert err < 1e-7
        assert np.allclose(K0, np.transpose(K0, (2, 3, 0, 1, 4)), atol=1e-14)
        # frame indifference: P(QF) = Q P(F)
        Q = ms.random_rotations(1, 9)[0]
        PQ, _ = O.neo_hookean((Q @ F0).reshape(3, 3, 1), mu, kappa)
        assert np.allclose(PQ[..., 0], Q @ P0[..., 0], atol=1e-13)


J2P = dict(E=2.0e5, nu=0.3, sy=300.0, nexp=20.0, edot0=1e-3, dt=1.0)


def _j2(eps, epsp):
    s, C, ep, dp = O.j2_perzyna(eps.reshape(3, 3, 1), epsp.reshape(3, 3, 1), J2P["E"], J2P["nu"],
                                J2P["sy"], J2P["nexp"], J2P["edot0"], J2P["dt"])
    return s[..., 0], C[..., 0], ep[..., 0], dp[0]


def test_P15_j2_elastic_below_yield_and_fd_tangent():
    eps = 1e-4 * np.diag([-0.5, -0.5, 1.0])
    s, C, ep, dp = _j2(eps, np.zeros((3, 3)))
    Cel = O.isotropic_stiffness(J2P["E"], J2P["nu"])
    assert dp == 0 and np.allclose(C, Cel) and np.allclose(s, np.einsum("ijkl,kl->ij", Cel, eps))
    # yielding: the SURVEY appendix point eps_eq ~ 2.4e-3 -> dp ~ 1.77e-5, s_vm ~ 545 (checked)
    eps = 2.4e-3 * np.diag([-0.5, -0.5, 1.0]) + 1e-4 * np.array([[0, 1, 0], [1, 0, 0.3], [0, 0.3, 0]])
    epsp = 1e-4 * np.diag([0.2, -0.5, 0.3])
    s, C, ep, dp = _j2(eps, epsp)
    assert dp > 0
    # backward-Euler consistency: dp = edot0 dt <s_vm/sy - 1>^n
    dev = s - np.trace(s) / 3 * np.eye(3)
    svm = np.sqrt(1.5 * np.sum(dev * dev))
    assert dp == pytest.approx(J2P["edot0"] * J2P["dt"] * (svm / J2P["sy"] - 1) ** J2P["nexp"], rel=1e-9)

    def sig(e):
        e = 0.5 * (e + e.T)
        return _j2(e, epsp)[0]
    err = _fd_check(sig, eps, 0.5 * (C + np.swapaxes(C, 2, 3)), h=1e-8)
    assert err / np.max(np.abs(C)) < 1e-6


def test_P15_j2_steady_flow_stress():
    # homogeneous path eps = 1e-3 t diag(-1/2,-1/2,1): eps_eq rate = edot0, so s_vm -> 2 sy
    epsp = np.zeros((3, 3))
    for k in range(1, 401):
        eps = 1e-3 * k * np.diag([-0.5, -0.5, 1.0])
        s, C, epsp, dp = _j2(eps, epsp)
    dev = s - np.trace(s) / 3 * np.eye(3)
    assert np.sqrt(1.5 * np.sum(dev * dev)) == pytest.approx(2 * J2P["sy"], rel=1e-6)


# ---------------------------------------------------------------- P3 / P4 operator


def test_P3_homogeneous_operator_closed_form():
    n = (8, 6, 4)
    XI = O.frequency_grid(n)
    lam, mu = 1.7, 0.9
    C = O.isotropic_from_lame(lam, mu)[..., None, None, None] * np.ones((1,) * 4 + (4, 6, 8))
    uh = O.fft(ms.random_field((3, 4, 6, 8), 31))
    for finite in (False, True):
        f, _ = O.apply_K(uh, C, XI, finite=finite)
        xi2 = XI[0] ** 2 + XI[1] ** 2 + XI[2] ** 2
        xdu = XI[0] * uh[0] + XI[1] * uh[1] + XI[2] * uh[2]
        # Navier acoustic tensor: A u = mu |xi|^2 u + (lam + mu) xi (xi . u)
        ref = mu * xi2 * uh + (lam + mu) * XI * xdu
        assert np.max(np.abs(f - ref)) < 1e-12 * np.max(np.abs(ref))
        # preconditioner = exact inverse of the homogeneous operator off Z
        z = O.precondition(f, O.isotropic_from_lame(lam, mu), XI)
        Z = O.null_set(XI)
        assert np.max(np.abs(z[:, ~Z] - uh[:, ~Z])) < 1e-12 * np.max(np.abs(uh))
        assert np.all(z[:, Z] == 0)


def test_P4_hermitian():
    n = (8, 8, 6)
    XI = O.frequency_grid(n)
    ph = _two_phase_random(n, 3)
    C = O.stiffness_field(ph, ISO2)
    v = O.fft(ms.random_field((3, 6, 8, 8), 41))
    w = O.fft(ms.random_field((3, 6, 8, 8), 42))
    Kv, _ = O.apply_K(v, C, XI)
    Kw, _ = O.apply_K(w, C, XI)
    assert O.inner(Kv, w) == pytest.approx(O.inner(v, Kw), rel=1e-12)
    assert O.inner(Kv, v) > 0
    # finite strain with a heterogeneous neo-Hookean tangent at a random F field
    F = np.eye(3).reshape(3, 3, 1, 1, 1) + 0.1 * ms.random_field((3, 3, 6, 8, 8), 43)
    _, K = O.neo_hookean(F, 1.0 + 9.0 * ph, 2.5 + 22.5 * ph)
    Kv, _ = O.apply_K(v, K, XI, finite=True)
    Kw, _ = O.apply_K(w, K, XI, finite=True)
    assert O.inner(Kv, w) == pytest.approx(O.inner(v, Kw), rel=1e-12)


# ---------------------------------------------------------------- P5 / P6 dense


def test_P5_rank_even_and_odd():
    for n, zeros in (((4, 4, 4), 24), ((5, 3, 3), 3)):
        ph = _two_phase_random(n, 5)
        A = O.dense_operator(O.stiffness_field(ph, ISO2), n)
        assert np.max(np.abs(A - A.T)) < 1e-12 * np.max(np.abs(A))
        ev = np.linalg.eigvalsh(0.5 * (A + A.T))
        tol = 1e-10 * ev[-1]
        assert np.sum(np.abs(ev) < tol) == zeros
        assert np.all(ev[np.abs(ev) >= tol] > 0)


@pytest.mark.parametrize("which", ["4cube", "c1"])
def test_P6_dense_direct_solve(which):
    if which == "4cube":
        n = (4, 4, 4)
        ph = _two_phase_random(n, 6)
        mats = ISO2
        t = np.zeros((3, 3)); t[0, 1] = t[1, 0] = 1e-3; t[2, 2] = -2e-3
        load = dict(target=t, mask=np.zeros((3, 3), bool))
    else:
        cfg = configs.c1()
        n, ph, mats, load = cfg["n"], cfg["phase"], cfg["materials"], cfg["loads"][0]
    res = O.solve_small_strain(ph, mats, load, tol=1e-12)
    C = O.stiffness_field(ph, mats)
    A = O.dense_operator(C, n)
    sig_U = O.contract(C, load["target"].reshape(3, 3, 1, 1, 1) * np.ones((1, 1) + ph.shape))
    b = O.ifft(O.rhs_from_stress(sig_U, O.frequency_grid(n))).ravel()
    u_dense = np.linalg.lstsq(A, b, rcond=1e-10)[0]
    u_pcg = O.displacement(res["u_hat"]).ravel()
    assert np.linalg.norm(u_pcg - u_dense) <= 1e-9 * np.linalg.norm(u_dense)


# ---------------------------------------------------------------- P7 homogeneous


def test_P7_homogeneous_strain_control_zero_iterations():
    g = _gold("hooke_iso.json")
    ph = np.zeros((4, 4, 4), np.uint16)
    mats = [dict(kind="iso", E=g["E"], nu=g["nu"])]
    t = np.zeros((3, 3)); t[0, 0] = g["eps11"]
    res = O.solve_small_strain(ph, mats, dict(target=t, mask=np.zeros((3, 3), bool)))
    assert res["iters"] == 0
    assert res["mean_sig"][0, 0] == pytest.approx(g["sigma11"], rel=1e-14)
    assert res["mean_sig"][1, 1] == pytest.approx(g["sigma22"], rel=1e-14)
    assert np.max(np.abs(res["sig"][0, 0] - g["sigma11"])) < 1e-15


def test_P7_homogeneous_one_iteration():
    n = (6, 4, 8)
    XI = O.frequency_grid(n)
    C0 = O.isotropic_stiffness(3.0, 0.25)
    C = C0[..., None, None, None] * np.ones((1,) * 4 + (8, 4, 6))
    b = O.fft(ms.random_field((3, 8, 4, 6), 51))
    b[:, O.null_set(XI)] = 0

    def apply_A(v):
        f, m = O.apply_K(v.u, C, XI)
        return O.Aug(f, np.zeros((3, 3))), m

    x, it, _ = O.pcg(apply_A, lambda r: O.Aug(O.precondition(r.u, C0, XI), np.zeros((3, 3))),
                     O.Aug(b, np.zeros((3, 3))), np.eye(3), 1e-12)
    assert it == 1
    # mixed control on a homogeneous medium (R4): also one iteration
    ph = np.zeros((8, 4, 6), np.uint16)
    t = np.zeros((3, 3)); t[2, 2] = 1e-3
    mask = np.ones((3, 3), bool); mask[2, 2] = False
    res = O.solve_small_strain(ph, [dict(kind="iso", E=3.0, nu=0.25)], dict(target=t, mask=mask))
    assert res["iters"] == 1
    # uniaxial stress: sigma_zz = E eps_zz, lateral strains -nu eps_zz
    assert res["mean_sig"][2, 2] == pytest.approx(3.0e-3, rel=1e-12)
    assert res["mean_eps"][0, 0] == pytest.approx(-0.25e-3, rel=1e-12)


# ---------------------------------------------------------------- P8 laminate


def _lame(E, nu):
    return E * nu / ((1 + nu) * (1 - 2 * nu)), E / (2 * (1 + nu))


def _laminate_closed_forms(E, nu, frac):
    lam, mu = np.array([_lame(e, v) for e, v in zip(E, nu)]).T
    M = lam + 2 * mu
    avg = lambda q: frac * q[0] + (1 - frac) * q[1]  # noqa: E731
    C1111 = 1 / avg(1 / M)
    C1212 = 1 / avg(1 / mu)
    C2323 = avg(mu)
    C2222 = avg(M - lam ** 2 / M) + avg(lam / M) ** 2 / avg(1 / M)
    C1122 = avg(lam / M) / avg(1 / M)
    # uniaxial stress across the layers (sigma_11 only): E* (see SURVEY R-P8; not Reuss-E)
    t_over_s = -avg(lam / M) / avg(2 * (lam + mu) - 2 * lam ** 2 / M)
    Eacross = 1.0 / (avg(1 / M) - 2 * t_over_s * avg(lam / M))
    return dict(C1111=C1111, C1212=C1212, C2323=C2323, C2222=C2222, C1122=C1122,
                Ealong=avg(np.asarray(E, float)), Eacross=Eacross)


def test_P8_laminate_closed_forms():
    n = (8, 4, 4)
    ph = ms.laminate(n, axis=0, thickness=4)  # 50/50, even thickness on an even grid (R1)
    E, nu = (10.0, 1.0), (0.3, 0.3)
    mats = [dict(kind="iso", E=E[1], nu=nu[1]), dict(kind="iso", E=E[0], nu=nu[0])]
    ref = _laminate_closed_forms(E, nu, 0.5)
    none = np.zeros((3, 3), bool)

    def strain(t):
        return O.solve_small_strain(ph, mats, dict(target=t, mask=none), tol=1e-13)["mean_sig"]

    t = np.zeros((3, 3)); t[0, 0] = 1.0
    assert strain(t)[0, 0] == pytest.approx(ref["C1111"], rel=1e-8)
    t = np.zeros((3, 3)); t[1, 1] = 1.0
    s = strain(t)
    assert s[1, 1] == pytest.approx(ref["C2222"], rel=1e-8)
    assert s[0, 0] == pytest.approx(ref["C1122"], rel=1e-8)
    t = np.zeros((3, 3)); t[0, 1] = t[1, 0] = 0.5
    assert strain(t)[0, 1] == pytest.approx(ref["C1212"], rel=1e-8)
    t = np.zeros((3, 3)); t[1, 2] = t[2, 1] = 0.5
    assert strain(t)[1, 2] == pytest.approx(ref["C2323"], rel=1e-8)
    # uniaxial stress along the layers (equal nu): E* = <E> (Voigt); mixed control
    t = np.zeros((3, 3)); t[1, 1] = 1e-3
    mask = np.ones((3, 3), bool); mask[1, 1] = False
    r = O.solve_small_strain(ph, mats, dict(target=t, mask=mask), tol=1e-13)
    assert r["mean_sig"][1, 1] / 1e-3 == pytest.approx(ref["Ealong"], rel=1e-8)
    # uniaxial stress across the layers: pure stress control on all components
    t = np.zeros((3, 3)); t[0, 0] = 1e-3
    r = O.solve_small_strain(ph, mats, dict(target=t, mask=np.ones((3, 3), bool)), tol=1e-13)
    assert 1e-3 / r["mean_eps"][0, 0] == pytest.approx(ref["Eacross"], rel=1e-8)
    assert abs(ref["Eacross"] - 2 / (1 / E[0] + 1 / E[1])) > 0.1  # S:325 (Reuss) is not this


# ---------------------------------------------------------------- P9-P14 on c1


@pytest.fixture(scope="module")
def c1_solution():
    cfg = configs.c1()
    return cfg, O.solve_small_strain(cfg["phase"], cfg["materials"], cfg["loads"][0], tol=1e-10)


def _mandel(C):
    idx = [(0, 0), (1, 1), (2, 2), (1, 2), (0, 2), (0, 1)]
    w = [1, 1, 1, np.sqrt(2), np.sqrt(2), np.sqrt(2)]
    return np.array([[C[i + j] * w[a] * w[b] for b, j in enumerate(idx)] for a, i in enumerate(idx)])


def test_P9_P10_bounds_hill_mandel(c1_solution):
    cfg, res = c1_solution
    C = O.stiffness_field(cfg["phase"], cfg["materials"])
    eps_bar = cfg["loads"][0]["target"]
    W = np.sum(res["mean_sig"] * eps_bar)
    Cv = _mandel(O.volume_average(C))
    Sr = np.mean([np.linalg.inv(_mandel(C[..., k, j, i])) for k in range(8) for j in range(8) for i in range(8)], axis=0)
    e = np.array([eps_bar[0, 0], eps_bar[1, 1], eps_bar[2, 2], 0, 0, 0])
    assert e @ np.linalg.inv(Sr) @ e < W < e @ Cv @ e
    # Hill-Mandel <sigma:eps> = <sigma>:<eps> (discrete integration by parts)
    hm = np.mean(np.sum(res["sig"] * res["eps"], axis=(0, 1)))
    assert hm == pytest.approx(np.sum(res["mean_sig"] * res["mean_eps"]), rel=1e-9)
    assert res["iters"] > 1


def test_P11_P12_compatibility_and_loading(c1_solution):
    cfg, res = c1_solution
    assert np.allclose(res["mean_eps"], cfg["loads"][0]["target"], atol=1e-17)
    # equilibrium residual of the returned fields meets the stop test
    XI = res["XI"]
    r = O.rhs_from_stress(res["sig"], XI)
    assert np.sqrt(O.inner(r, r)) / np.linalg.norm(res["mean_sig"]) <= 1e-10
    # compatibility: curl(curl eps) = 0 spectrally (eps = sym grad u)
    eh = O.fft(res["eps"])
    lc = np.zeros((3, 3, 3))
    lc[0, 1, 2] = lc[1, 2, 0] = lc[2, 0, 1] = 1
    lc[0, 2, 1] = lc[2, 1, 0] = lc[1, 0, 2] = -1
    cc = np.einsum("ikm,jln,k...,l...,mn...->ij...", lc, lc, XI, XI, eh)
    assert np.max(np.abs(cc)) <= 1e-12 * np.max(np.abs(eh))


def test_P13_c1_symmetry(c1_solution):
    cfg, res = c1_solution
    s = res["sig"]
    # mirror x -> -x (index i -> n-1-i): sigma_xy, sigma_xz flip sign, others even
    sx = s[:, :, :, :, ::-1]
    sign = np.array([[1, -1, -1], [-1, 1, 1], [-1, 1, 1]])
    assert np.max(np.abs(sx - sign[:, :, None, None, None] * s)) < 1e-9 * np.max(np.abs(s))
    # swap y <-> z with eps_xx loading
    sw = np.swapaxes(s, 2, 3)[[0, 2, 1]][:, [0, 2, 1]]
    assert np.max(np.abs(sw - s)) < 1e-9 * np.max(np.abs(s))


def test_P14_strain_stress_consistency(c1_solution):
    cfg, res = c1_solution
    r2 = O.solve_small_strain(cfg["phase"], cfg["materials"],
                              dict(target=res["mean_sig"], mask=np.ones((3, 3), bool)), tol=1e-12)
    assert np.max(np.abs(r2["mean_eps"] - res["mean_eps"])) < 1e-8 * 1e-3
    assert np.max(np.abs(r2["eps"] - res["eps"])) < 1e-7 * np.max(np.abs(res["eps"]))


def test_mixed_control_c2_like_small():
    # c2 structure at 16^3: strain-controlled eps_zz reached exactly, other <sigma> = 0 (P12)
    cfg = configs.c2(n=16, radius_vox=2, count=None)
    res = O.solve_small_strain(cfg["phase"], cfg["materials"], cfg["loads"][0], tol=1e-10)
    assert res["mean_eps"][2, 2] == pytest.approx(1e-3, rel=1e-14)
    ms_ = res["mean_sig"]
    off = np.abs(ms_.copy()); off[2, 2] = 0
    assert np.max(off) <= 1e-9 * abs(ms_[2, 2])


# ---------------------------------------------------------------- P16 / P17 finite strain


def test_P16_homogeneous_neo_hookean_uniaxial():
    mu, kappa = 1.0, 2.5
    lam = kappa - 2 * mu / 3
    Fzz = 1.05

    def Pxx(a):
        J = a * a * Fzz
        return mu * (a - 1 / a) + lam * np.log(J) / a

    a_ref = brentq(Pxx, 0.5, 1.5, xtol=1e-15)
    n = (4, 4, 4)
    ph = np.zeros((4, 4, 4), np.uint16)
    mats = [dict(kind="neohooke", mu=mu, kappa=kappa)]
    st = O.FiniteStrainState(n)
    mask = np.zeros((3, 3), bool); mask[0, 0] = mask[1, 1] = True
    t = np.eye(3); t[2, 2] = Fzz; t[0, 0] = t[1, 1] = 0.0
    res = O.solve_finite_increment(st, ph, mats, dict(target=t, mask=mask), tol=1e-12)
    assert res["mean_F"][0, 0] == pytest.approx(a_ref, rel=1e-10)
    assert res["mean_F"][1, 1] == pytest.approx(a_ref, rel=1e-10)
    assert abs(res["mean_P"][0, 0]) < 1e-10
    assert res["converged"]


def test_P17_small_load_finite_matches_linear():
    cfg = configs.c1()
    mu_m, mu_i = 1.0 / 2.6, 10.0 / 2.6  # E = 1, 10 with nu = 0.3 -> mu = E/2.6, kappa = E/1.2
    mats_nh = [dict(kind="neohooke", mu=mu_m, kappa=1.0 / 1.2), dict(kind="neohooke", mu=mu_i, kappa=10.0 / 1.2)]
    h = 1e-6
    lin = O.solve_small_strain(cfg["phase"], cfg["materials"],
                               dict(target=h * np.diag([1.0, 0, 0]), mask=np.zeros((3, 3), bool)), tol=1e-12)
    st = O.FiniteStrainState(cfg["n"])
    fin = O.solve_finite_increment(st, cfg["phase"], mats_nh,
                                   dict(target=np.eye(3) + h * np.diag([1.0, 0, 0]), mask=np.zeros((3, 3), bool)),
                                   tol=1e-12, tol_newton=1e-13)
    assert np.max(np.abs(fin["P"] - lin["sig"])) <= 1e-5 * np.max(np.abs(lin["sig"]))


def test_j2_dbfft_homogeneous_matches_material_point():
    # homogeneous J2 RVE: DBFFT (0 CG iterations) reproduces the material point update
    n = (4, 4, 4)
    ph = np.zeros((4, 4, 4), np.uint16)
    mats = [dict(kind="j2", E=J2P["E"], nu=J2P["nu"], sigma_y=J2P["sy"], n=J2P["nexp"], edot0=J2P["edot0"])]
    st = O.J2State(n)
    epsp = np.zeros((3, 3))
    for k in range(1, 4):
        t = 1e-3 * k * np.diag([-0.5, -0.5, 1.0])
        res = O.solve_j2_increment(st, ph, mats, dict(target=t, mask=np.zeros((3, 3), bool)), 1.0)
        s, _, epsp, _ = _j2(t, epsp)
        assert np.allclose(res["mean_sig"], s, rtol=1e-12, atol=1e-9)


def test_volume_average_exact_sum():
    """<a> over the voxel axes on a strided tensor field of 2^18 voxels: equals the
    exactly rounded mean (math.fsum) to 1e-15, and a two-phase field's mean stiffness equals the
    closed form (N - n1) C0 / N + n1 C1 / N (the phase-count formula)."""
    import math
    n = (32, 64, 128)
    u = ms.SplitMix64(5).uniform(n[0] * n[1] * n[2]).reshape(n[2], n[1], n[0])
    ph = (u < 0.3).astype(np.uint16)
    mats = [dict(kind="iso", E=1.0, nu=0.3), dict(kind="iso", E=10.0, nu=0.25)]
    C = O.stiffness_field(ph, mats)
    assert not C.flags["C_CONTIGUOUS"] or C.strides[-1] != 8 * 81  # a strided field is the case to pin
    m = O.volume_average(C)
    N = ph.size
    exact = np.array([math.fsum(C[i, j, k, l].ravel()) / N for i in range(3) for j in range(3)
                      for k in range(3) for l in range(3)]).reshape(3, 3, 3, 3)
    assert np.abs(m - exact).max() <= 1e-15 * np.abs(exact).max()
    C0 = O.stiffness_field(np.zeros((1, 1, 1), np.uint16), mats)[..., 0, 0, 0]
    C1 = O.stiffness_field(np.ones((1, 1, 1), np.uint16), mats)[..., 0, 0, 0]
    n1 = int(ph.sum())
    closed = ((N - n1) * C0 + n1 * C1) / N
    assert np.abs(m - closed).max() <= 1e-15 * np.abs(closed).max()


def test_reference_media_closed_forms_and_order():
    """P:255 / P:394 reference media.  Homogeneous field: all media equal C.
    Two isotropic phases: the harmonic mean is isotropic with K = 1/<1/K>, mu = 1/<1/mu>
    (closed form), and Reuss <= Hill <= Voigt in the Loewner order (Mandel eigenvalues)."""
    n = (8, 8, 8)
    mats = [dict(kind="iso", E=1.0, nu=0.3), dict(kind="iso", E=10.0, nu=0.25)]
    C0 = O.stiffness_field(np.zeros(n, np.uint16), mats)
    for m in ("arithmetic", "harmonic", "hill"):
        assert np.allclose(O.reference_medium(C0, m), C0[..., 0, 0, 0], rtol=1e-14, atol=1e-15)
    u = ms.SplitMix64(9).uniform(512).reshape(n)
    ph = (u < 0.35).astype(np.uint16)
    C = O.stiffness_field(ph, mats)
    f1 = ph.mean()

    def KG(E, nu):
        return E / (3 * (1 - 2 * nu)), E / (2 * (1 + nu))
    (K0, G0), (K1, G1) = KG(1.0, 0.3), KG(10.0, 0.25)
    KR = 1.0 / ((1 - f1) / K0 + f1 / K1)
    GR = 1.0 / ((1 - f1) / G0 + f1 / G1)
    CR = O.isotropic_from_lame(KR - 2.0 * GR / 3.0, GR)
    assert np.allclose(O.reference_medium(C, "harmonic"), CR, rtol=1e-13, atol=1e-14)
    MV = _mandel(O.reference_medium(C, "arithmetic"))
    MH = _mandel(O.reference_medium(C, "hill"))
    MR = _mandel(O.reference_medium(C, "harmonic"))
    assert np.linalg.eigvalsh(MV - MH).min() >= -1e-12
    assert np.linalg.eigvalsh(MH - MR).min() >= -1e-12


def test_reference_medium_changes_iterations_not_solution():
    """The preconditioner's reference medium (P:394 variants) never changes the solution of the
    system.  c2 structure at 24^3 (mixed control, E contrast 100, equal nu): isotropic phases of
    equal nu make every medium a multiple of <C>, and PCG is invariant under M -> cM, so the
    iteration counts are identical too; with unequal nu (0.2 / 0.45) they differ."""
    cfg = configs.c2(n=24, radius_vox=2)
    L = cfg["loads"][0]
    for mats, same_iters in ((cfg["materials"], True),
                             ([dict(kind="iso", E=1.0, nu=0.2), dict(kind="iso", E=100.0, nu=0.45)], False)):
        res = {m: O.solve_small_strain(cfg["phase"], mats, L, tol=1e-11, medium=m)
               for m in ("arithmetic", "harmonic", "hill")}
        ref = res["arithmetic"]
        for m in ("harmonic", "hill"):
            r = res[m]
            assert np.linalg.norm(r["mean_sig"] - ref["mean_sig"]) <= 1e-9 * np.linalg.norm(ref["mean_sig"])
            assert np.linalg.norm(r["sig"] - ref["sig"]) <= 1e-8 * np.linalg.norm(ref["sig"])
        n_iters = {res[m]["iters"] for m in res}
        assert (len(n_iters) == 1) == same_iters, n_iters


# ----------------------------------------------------------------- Saint Venant-Kirchhoff

def _svk_energy(F, E, nu):
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    Eg = 0.5 * (F.T @ F - np.eye(3))
    return 0.5 * lam * np.trace(Eg) ** 2 + mu * np.sum(Eg * Eg)


def test_svk_energy_tangent_limits():
    """SVK: P = dW/dF of W = lam/2 (tr E)^2 + mu E:E by central differences of W, K = dP/dF
    by differences of P, K(I) = the isotropic C(E, nu), and frame indifference P(QF) = Q P(F)."""
    E, nu = 70.0, 0.3
    rng = np.random.default_rng(3)
    F = np.eye(3) + 0.4 * rng.standard_normal((3, 3))
    P, K = O.svk(F.reshape(3, 3, 1), E, nu)
    P, K = P[..., 0], K[..., 0]
    h = 1e-6
    Pfd = np.zeros((3, 3))
    Kfd = np.zeros((3, 3, 3, 3))
    for k in range(3):
        for l in range(3):
            d = np.zeros((3, 3)); d[k, l] = h
            Pfd[k, l] = (_svk_energy(F + d, E, nu) - _svk_energy(F - d, E, nu)) / (2 * h)
            Kfd[:, :, k, l] = (O.svk((F + d).reshape(3, 3, 1), E, nu)[0][..., 0]
                               - O.svk((F - d).reshape(3, 3, 1), E, nu)[0][..., 0]) / (2 * h)
    assert np.abs(P - Pfd).max() <= 1e-7 * np.abs(P).max()
    assert np.abs(K - Kfd).max() <= 1e-7 * np.abs(K).max()
    _, K0 = O.svk(np.eye(3).reshape(3, 3, 1), E, nu)
    assert np.allclose(K0[..., 0], O.isotropic_stiffness(E, nu), rtol=1e-14, atol=1e-12)
    th = 0.7
    Q = np.array([[np.cos(th), -np.sin(th), 0], [np.sin(th), np.cos(th), 0], [0, 0, 1.0]])
    PQ, _ = O.svk((Q @ F).reshape(3, 3, 1), E, nu)
    assert np.allclose(PQ[..., 0], Q @ P, rtol=1e-13, atol=1e-12)


def test_svk_homogeneous_uniaxial_closed_form():
    """Homogeneous SVK cell under the SS3.3 load (stretch lambda, other directions held):
    F = diag(1, 1, lambda) exactly, P_zz = lambda (lam + 2 mu)(lambda^2 - 1)/2 and
    P_xx = P_yy = lam (lambda^2 - 1)/2, with no PCG work (homogeneous medium)."""
    n = (8, 8, 8)
    E, nu = 70.0, 0.3
    lam = E * nu / ((1 + nu) * (1 - 2 * nu)); mu = E / (2 * (1 + nu))
    ph = np.zeros((n[2], n[1], n[0]), np.uint16)
    mats = [dict(kind="svk", E=E, nu=nu)]
    st = O.FiniteStrainState(n)
    for stretch in (1.2, 1.6, 2.0):
        L = dict(target=np.diag([1.0, 1.0, stretch]), mask=np.zeros((3, 3), bool))
        r = O.solve_finite_increment(st, ph, mats, L, tol=1e-10)
        assert r["converged"] and r["cg_iters"] == 0
        e = 0.5 * (stretch ** 2 - 1)
        assert r["mean_P"][2, 2] == pytest.approx(stretch * (lam + 2 * mu) * e, rel=1e-13)
        assert r["mean_P"][0, 0] == pytest.approx(lam * e, rel=1e-13)
        assert np.abs(r["F"] - np.diag([1.0, 1.0, stretch]).reshape(3, 3, 1, 1, 1)).max() <= 1e-14


# ----------------------------------------------------------- residual monitors

def test_incompatibility_closed_forms():
    """eps_xx = a sin(2 pi y): curl curl eps has eta_zz = -d_yy eps_xx, max = (2 pi)^2 a; F_xy =
    a sin(2 pi z): curl of row x has (curl F)_xx = -d_z F_xy, max = 2 pi a; symmetric gradients and
    F = I + grad u are compatible (round-off only)."""
    n = (8, 12, 16)
    XI = O.frequency_grid(n)
    z, y, x = np.meshgrid(np.arange(n[2]) / n[2], np.arange(n[1]) / n[1], np.arange(n[0]) / n[0], indexing="ij")
    a = 1e-3
    eps = np.zeros((3, 3) + z.shape)
    eps[0, 0] = a * np.sin(2 * np.pi * y)
    assert O.incompatibility(eps, XI, finite=False) == pytest.approx((2 * np.pi) ** 2 * a, rel=1e-12)
    F = np.zeros((3, 3) + z.shape) + np.eye(3).reshape(3, 3, 1, 1, 1)
    F[0, 1] += a * np.sin(2 * np.pi * z)
    assert O.incompatibility(F, XI, finite=True) == pytest.approx(2 * np.pi * a, rel=1e-12)
    u = O.fft(ms.random_field((3,) + z.shape, 51))
    xi2 = np.max(np.abs(XI)) ** 2
    E = O.ifft(O.sym_grad_hat(u, XI))
    assert O.incompatibility(E, XI, finite=False) <= 1e-14 * xi2 * np.abs(E).max()  # vs ~(2 pi a) xi^2
    G = O.ifft(O.grad_hat(u, XI))
    assert O.incompatibility(np.eye(3).reshape(3, 3, 1, 1, 1) + G, XI, finite=True) <= 1e-14 * np.sqrt(xi2) * np.abs(G).max()


def test_equilibrium_and_loading_residual_closed_forms():
    """sigma_xy = sigma_yx = s0 + sin(2 pi x): (div sigma)_y = 2 pi cos(2 pi x), rms = 2 pi/sqrt 2,
    <sigma> = s0 (e_xy + e_yx); a converged c1 solve has equilibrium <= its PCG tolerance (R7)
    and loading 0 under strain control."""
    n = (16, 8, 8)
    XI = O.frequency_grid(n)
    z, y, x = np.meshgrid(np.arange(n[2]) / n[2], np.arange(n[1]) / n[1], np.arange(n[0]) / n[0], indexing="ij")
    s0 = 3.0
    sig = np.zeros((3, 3) + z.shape)
    sig[0, 1] = sig[1, 0] = s0 + np.sin(2 * np.pi * x)
    assert O.equilibrium_residual(sig, XI) == pytest.approx((2 * np.pi / np.sqrt(2)) / (s0 * np.sqrt(2)), rel=1e-12)
    cfg = configs.c1()
    L = cfg["loads"][0]
    r = O.solve_small_strain(cfg["phase"], cfg["materials"], L, tol=1e-10)
    X1 = O.frequency_grid(cfg["n"])
    assert O.equilibrium_residual(r["sig"], X1) <= 1e-10
    assert O.loading_residual(r["mean_eps"], r["mean_sig"], L["target"], L["mask"]) <= 1e-15
    assert O.incompatibility(r["eps"], X1, finite=False) <= 1e-12


# ----------------------------------------------------------------- mixed hyperelastic families

def _nh_energy(F, mu, kappa):
    """R14: W = mu/2 (tr F^T F - 3) - mu ln J + lam/2 (ln J)^2, lam = kappa - 2 mu/3."""
    lam = kappa - 2.0 * mu / 3.0
    J = np.linalg.det(F)
    return 0.5 * mu * (np.trace(F.T @ F) - 3.0) - mu * np.log(J) + 0.5 * lam * np.log(J) ** 2


def test_hyperelastic_mixed_phase_dispatch():
    """A phase map mixing neo-Hookean (R14) and SVK phases: at every voxel P = dW/dF of
    THAT voxel's phase energy (central differences of W, written out here), and K = dP/dF by
    differences of the mixed P — a phase routed to the wrong law or parameters fails."""
    mats = [dict(kind="neohooke", mu=1.0, kappa=2.5), dict(kind="svk", E=70.0, nu=0.3),
            dict(kind="neohooke", mu=7.0, kappa=20.0), dict(kind="svk", E=5.0, nu=0.2)]
    rng = np.random.default_rng(11)
    nv = 12
    phase = np.array([0, 1, 2, 3, 3, 2, 1, 0, 1, 3, 0, 2], np.uint16).reshape(1, 1, nv)
    F = np.eye(3).reshape(3, 3, 1, 1, 1) + 0.3 * rng.standard_normal((3, 3, 1, 1, nv))
    P, K = O.hyperelastic(F, phase, mats)
    h = 1e-6

    def W(Fv, m):
        return _nh_energy(Fv, m["mu"], m["kappa"]) if m["kind"] == "neohooke" else _svk_energy(Fv, m["E"], m["nu"])

    for v in range(nv):
        m = mats[phase[0, 0, v]]
        Fv = F[:, :, 0, 0, v]
        Pfd = np.zeros((3, 3))
        Kfd = np.zeros((3, 3, 3, 3))
        for k in range(3):
            for l in range(3):
                d = np.zeros((3, 3)); d[k, l] = h
                Pfd[k, l] = (W(Fv + d, m) - W(Fv - d, m)) / (2 * h)
                Fp, Fm = F.copy(), F.copy()
                Fp[k, l, 0, 0, v] += h
                Fm[k, l, 0, 0, v] -= h
                Kfd[:, :, k, l] = (O.hyperelastic(Fp, phase, mats)[0][:, :, 0, 0, v]
                                   - O.hyperelastic(Fm, phase, mats)[0][:, :, 0, 0, v]) / (2 * h)
        Pv, Kv = P[:, :, 0, 0, v], K[:, :, :, :, 0, 0, v]
        assert np.abs(Pv - Pfd).max() <= 1e-7 * max(np.abs(Pv).max(), 1.0), (v, m)
        assert np.abs(Kv - Kfd).max() <= 1e-6 * np.abs(Kv).max(), (v, m)


# ----------------------------------------------------------------- loading residual

def test_loading_residual_stress_branch_closed_forms():
    """Eq. chedckimp under mixed control, worked by hand: the stress-controlled part is
    ||<sigma> - sigma_bar|| / ||<sigma>|| over the masked components, the strain part
    ||<eps> - eps_bar|| / ||eps_bar|| over the others, the residual the larger of the two."""
    mask = np.zeros((3, 3), bool)
    mask[0, 0] = True                          # sigma_xx prescribed
    target = np.diag([2.0, 1e-3, 0.0])         # sigma_xx = 2; eps_yy = 1e-3, other strains 0
    mean_sig = np.diag([2.5, 0.0, 0.0])        # |2.5 - 2| / 2.5 = 0.2
    mean_eps = np.diag([7.0, 1e-3 + 1e-6, 0.0])  # eps_xx is free; |1e-6| / 1e-3 = 1e-3
    assert O.loading_residual(mean_eps, mean_sig, target, mask) == pytest.approx(0.2, rel=1e-14)
    # strain part dominating: <eps_yy> off by 5e-4 -> 0.5; stress exact
    mean_sig = np.diag([2.0, 0.0, 0.0])
    mean_eps = np.diag([7.0, 1.5e-3, 0.0])
    assert O.loading_residual(mean_eps, mean_sig, target, mask) == pytest.approx(0.5, rel=1e-12)
    # a zero prescribed stress: relative to ||<sigma>|| (3, 4 -> 5), not to the target
    mask = np.zeros((3, 3), bool)
    mask[1, 1] = mask[2, 2] = True
    target = np.diag([1e-3, 0.0, 0.0])
    mean_sig = np.diag([0.0, 3.0, 4.0])
    mean_eps = np.diag([1e-3, 9.0, 9.0])
    assert O.loading_residual(mean_eps, mean_sig, target, mask) == pytest.approx(1.0, rel=1e-14)


# ----------------------------------------------------------------- heterogeneous J2 Newton (R16)

def _j2_mats(sy):
    return [dict(kind="j2", E=J2P["E"], nu=J2P["nu"], sigma_y=s, n=J2P["nexp"], edot0=J2P["edot0"]) for s in sy]


def _j2_point(eps, epsp, m, dt):
    s, C, ep, dp = O.j2_perzyna(eps.reshape(3, 3, 1), epsp.reshape(3, 3, 1), m["E"], m["nu"], m["sigma_y"],
                                m["n"], m["edot0"], dt)
    return s[..., 0], ep[..., 0], dp[0]


def test_j2_laminate_elasto_viscoplastic():
    """Elasto-viscoplastic laminate (layers normal to x, 50/50, yield stresses 300 / 450), three
    plastic increments under strain control.  The exact discrete solution has uniform strain in
    each layer: the in-plane components (yy, zz, yz) equal the macro strain, the out-of-plane
    ones (xx, xy, xz) average to it, and the tractions sigma_xx, sigma_xy, sigma_xz are continuous
    across the interfaces (equilibrium).  That is a 3-unknown root per increment on the
    material-point update (P15) — solved here with scipy, independent of the DBFFT machinery —
    against solve_j2_increment's Newton-PCG on the full grid (even layer widths: no Nyquist
    content, R1)."""
    from scipy.optimize import root
    n = (8, 4, 4)
    ph = ms.laminate(n, axis=0, thickness=4)            # phase 1 in the first 4 x-planes
    mats = _j2_mats([300.0, 450.0])
    st = O.J2State(n)
    dt = 1.0
    oop = [(0, 0), (0, 1), (0, 2)]
    base = 2e-3 * np.diag([-0.5, -0.5, 1.0])
    base[0, 1] = base[1, 0] = 0.6e-3
    base[1, 2] = base[2, 1] = 0.3e-3
    ep = [np.zeros((3, 3)), np.zeros((3, 3))]
    for k in range(1, 4):
        target = k * base

        def layers(a):
            e = [target.copy(), target.copy()]
            for (i, j), v in zip(oop, a):
                e[0][i, j] = e[0][j, i] = v
                e[1][i, j] = e[1][j, i] = 2.0 * target[i, j] - v   # 50/50 average
            return e

        def resid(a):
            e = layers(a)
            s0 = _j2_point(e[0], ep[0], mats[0], dt)[0]
            s1 = _j2_point(e[1], ep[1], mats[1], dt)[0]
            return [(s0[i, j] - s1[i, j]) / J2P["E"] for (i, j) in oop]

        sol = root(resid, [target[i, j] for (i, j) in oop], method="hybr", tol=1e-14)
        assert np.max(np.abs(resid(sol.x))) < 1e-15   # tractions equal to ~1e-12 relative
        e = layers(sol.x)
        pts = [_j2_point(e[p], ep[p], mats[p], dt) for p in range(2)]
        res = O.solve_j2_increment(st, ph, mats, dict(target=target, mask=np.zeros((3, 3), bool)), dt,
                                   tol=1e-12, tol_newton=1e-12)
        assert res["converged"]
        for p in range(2):
            sel = ph == p
            scale = np.abs(e[p]).max()
            assert np.abs(res["eps"][:, :, sel] - e[p][:, :, None]).max() <= 1e-10 * scale, (k, p)
            assert np.abs(res["sig"][:, :, sel] - pts[p][0][:, :, None]).max() <= 1e-9 * np.abs(pts[p][0]).max()
            assert np.abs(res["eps_p"][:, :, sel] - pts[p][1][:, :, None]).max() <= 1e-10 * scale
        ep = [pts[0][1], pts[1][1]]
        mean_ref = 0.5 * (pts[0][0] + pts[1][0])
        assert np.abs(res["mean_sig"] - mean_ref).max() <= 1e-10 * np.abs(mean_ref).max()
    assert pts[0][2] > 0 and pts[1][2] > 0   # both layers flow in the last increment


def test_j2_polycrystal_twin_equilibrium_hill_mandel():
    """Heterogeneous J2 polycrystal (c5 recipe, 8^3 / 6 grains, lognormal yield stresses), three
    increments into plastic flow: every increment converges (flag), the final stress field is in
    equilibrium (Eq. chedckeq, <= 1e-9: PCG tol 1e-10 then one more constitutive update)
    and satisfies Hill-Mandel <sigma:eps> = <sigma>:<eps> (an equilibrated stress against a
    compatible fluctuation strain: their product averages to zero), and the plastic strain is
    traceless (J2 flow) and non-zero."""
    cfg = configs.c5(n=8, grains=6, increments=3)
    st = O.J2State(cfg["n"])
    newton = []
    for L in cfg["loads"]:
        res = O.solve_j2_increment(st, cfg["phase"], cfg["materials"], L, cfg["dt"], tol=1e-10)
        assert res["converged"]
        newton.append(res["newton_iters"])
    assert newton[0] == 1 and newton[-1] >= 3   # elastic first increment; plastic Newton later
    XI = O.frequency_grid(cfg["n"])
    assert O.equilibrium_residual(res["sig"], XI) <= 1e-9
    hm = O.volume_average(np.einsum("ij...,ij...->...", res["sig"], res["eps"]))
    macro = np.sum(res["mean_sig"] * res["mean_eps"])
    assert abs(hm - macro) <= 1e-9 * abs(macro)
    tr = res["eps_p"][0, 0] + res["eps_p"][1, 1] + res["eps_p"][2, 2]
    assert np.abs(tr).max() <= 1e-18 + 1e-12 * np.abs(res["eps_p"]).max()
    assert (res["dp"] > 0).sum() > 0
