"""DBFFT oracle: a plain, slow, obviously-correct CPU implementation (fp64).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this module.
It shares no code with the CUDA path (`paper_1905_12725_b200/`) and imports
nothing from it; the only common dependency is `synth/` (seeded inputs).

Everything follows Lucarini & Segurado, "DBFFT" (PAPER.md = /root/reference/
PAPER.md; citations are "P:<line> <equation/section>").  Where the paper is
silent or garbled, the reading of SURVEY.md section 8(c) (R1..R22) is used and
named.  Deliberate choices:
  * full complex spectra (scipy.fft.fftn on all host cores as the library FFT
    step), no half spectrum, no fusion;
  * tensors are full 3x3 / 3x3x3x3 arrays contracted with explicit einsum
    index strings (no Voigt/Mandel packing);
  * spectra are mean-normalised, u_hat = F(u)/N (R5), so the Euclidean
    spectral inner product equals the voxel-mean real inner product;
  * arrays are [component...][z][y][x] with x fastest; XI[a] is the frequency
    of axis a (0=x, 1=y, 2=z) broadcast on the [z][y][x] grid.

Pinned by tests/test_oracle_pins.py (-m "not gpu").  Functions that no pin
covers say "parity unpinned" in their docstring.
"""
import os

import numpy as np
import scipy.fft

# the library FFT step runs on every host core (scipy's pocketfft, the same transform numpy's
# fft computes; bit-identical results here); the rest of the oracle is plain numpy
FFT_WORKERS = os.cpu_count() or 1

# ----------------------------------------------------------------------------
# Volume average <a> = (1/N) sum_x a(x) ("average of the stiffness", the
# macroscopic stress/strain of P:126).  Summed pairwise over a contiguous copy of
# each component: numpy reduces a strided multi-axis mean by plain accumulation,
# whose error grows like N eps (1e-11 relative at 2^20 voxels).
# ----------------------------------------------------------------------------
def volume_average(a):
    a = np.asarray(a)
    flat = np.ascontiguousarray(a).reshape(a.shape[:-3] + (-1,))
    return flat.mean(axis=-1)


# ----------------------------------------------------------------------------
# Grid and frequencies (Eq. (1); reading R1 for even grids)
# ----------------------------------------------------------------------------


def axis_frequencies(N, L=1.0):
    """Frequencies xi of one axis in numpy-FFT native order (Eq. (1)).

    Odd N: Eq. (1) verbatim, xi = 2 pi (n - (N+1)/2)/L for n = 1..N, permuted
    into FFT order (the centred list is a permutation of FFT frequencies).
    Even N (R1): "neglect" the Nyquist frequency, i.e. xi = 0 at k = N/2.
    """
    if N % 2 == 1:
        centred = 2.0 * np.pi * (np.arange(1, N + 1) - (N + 1) / 2.0) / L
        # centred index n-1 holds frequency index kappa = n - (N+1)/2; FFT slot = kappa mod N
        out = np.empty(N)
        for idx, xi in enumerate(centred):
            kappa = idx + 1 - (N + 1) // 2
            out[kappa % N] = xi
        return out
    k = np.arange(N)
    kappa = np.where(k < N // 2, k, k - N).astype(np.float64)
    kappa[N // 2] = 0.0  # R1: Nyquist neglected
    return 2.0 * np.pi * kappa / L


def frequency_grid(n, L=(1.0, 1.0, 1.0)):
    """XI[a][z][y][x] = xi_a at each frequency point; n = (n1, n2, n3) = (nx, ny, nz)."""
    nx, ny, nz = n
    fx = axis_frequencies(nx, L[0])
    fy = axis_frequencies(ny, L[1])
    fz = axis_frequencies(nz, L[2])
    XI = np.zeros((3, nz, ny, nx))
    XI[0] = fx[None, None, :]
    XI[1] = fy[None, :, None]
    XI[2] = fz[:, None, None]
    return XI


def null_set(XI):
    """Z = {xi : xi_1 = xi_2 = xi_3 = 0} (R1): boolean [z][y][x]."""
    return (XI[0] == 0) & (XI[1] == 0) & (XI[2] == 0)


# ----------------------------------------------------------------------------
# Discrete Fourier transform, mean-normalised ("computed using the FFT"; R5)
# ----------------------------------------------------------------------------


def fft(f):
    """F(f)/N over the last three axes (library FFT as one step)."""
    N = f.shape[-1] * f.shape[-2] * f.shape[-3]
    return scipy.fft.fftn(f, axes=(-3, -2, -1), workers=FFT_WORKERS) / N


def ifft(fh, check=True):
    """Inverse of `fft`; returns the real part, asserting |Im| is round-off only."""
    N = fh.shape[-1] * fh.shape[-2] * fh.shape[-3]
    f = scipy.fft.ifftn(fh, axes=(-3, -2, -1), workers=FFT_WORKERS) * N
    if check:
        scale = max(np.max(np.abs(f.real)), 1e-300)
        assert np.max(np.abs(f.imag)) <= 1e-10 * scale, "spectrum is not Hermitian"
    return f.real


# ----------------------------------------------------------------------------
# Spectral differential operators
# ----------------------------------------------------------------------------


def sym_grad_hat(u_hat, XI):
    """eps_hat_ij = s_ijk u_k with s_ijk = 1/2 (i xi_j delta_ik + i xi_i delta_jk)."""
    out = np.empty((3, 3) + u_hat.shape[1:], dtype=np.complex128)
    for i in range(3):
        for j in range(3):
            out[i, j] = 0.5 * (1j * XI[j] * u_hat[i] + 1j * XI[i] * u_hat[j])
    return out


def grad_hat(u_hat, XI):
    """G_hat_ij = g_ijk u_k with g_ijk = i xi_j delta_ik (P:219 with the `i` restored, R2)."""
    out = np.empty((3, 3) + u_hat.shape[1:], dtype=np.complex128)
    for i in range(3):
        for j in range(3):
            out[i, j] = 1j * XI[j] * u_hat[i]
    return out


def div_hat(sig_hat, XI):
    """f_hat_i = d_ijk sig_jk with d_ijk = i xi_k delta_ij: f_i = i xi_k sig_ik."""
    out = np.zeros((3,) + sig_hat.shape[2:], dtype=np.complex128)
    for i in range(3):
        for k in range(3):
            out[i] += 1j * XI[k] * sig_hat[i, k]
    return out


# ----------------------------------------------------------------------------
# Materials (P:71-75 linear elasticity; R14 neo-Hookean; R16 J2-Perzyna)
# ----------------------------------------------------------------------------

I3 = np.eye(3)


def isotropic_stiffness(E, nu):
    """C_ijkl = lambda d_ij d_kl + mu (d_ik d_jl + d_il d_jk) (standard Hooke)."""
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    return isotropic_from_lame(lam, mu)


def isotropic_from_lame(lam, mu):
    C = np.zeros((3, 3, 3, 3))
    for i in range(3):
        for j in range(3):
            for k in range(3):
                for l in range(3):
                    C[i, j, k, l] = lam * I3[i, j] * I3[k, l] + mu * (I3[i, k] * I3[j, l] + I3[i, l] * I3[j, k])
    return C


def cubic_stiffness(C11, C12, C44, R):
    """Crystal-frame cubic tensor rotated C'_ijkl = R_ia R_jb R_kc R_ld C_abcd (BJ c3)."""
    C0 = np.zeros((3, 3, 3, 3))
    for a in range(3):
        for b in range(3):
            for c in range(3):
                for d in range(3):
                    if a == b and c == d:
                        C0[a, b, c, d] = C11 if a == c else C12
                    elif (a == c and b == d) or (a == d and b == c):
                        C0[a, b, c, d] = C44
    C = np.zeros((3, 3, 3, 3))
    for i in range(3):
        for j in range(3):
            for k in range(3):
                for l in range(3):
                    s = 0.0
                    for a in range(3):
                        for b in range(3):
                            for c in range(3):
                                for d in range(3):
                                    s += R[i, a] * R[j, b] * R[k, c] * R[l, d] * C0[a, b, c, d]
                    C[i, j, k, l] = s
    return C


def material_stiffness(m):
    """Fourth-order stiffness of a linear material record (synth.configs)."""
    if m["kind"] == "iso":
        return isotropic_stiffness(m["E"], m["nu"])
    if m["kind"] == "cubic":
        return cubic_stiffness(m["C11"], m["C12"], m["C44"], m["R"])
    if m["kind"] == "j2":
        return isotropic_stiffness(m["E"], m["nu"])
    if m["kind"] == "neohooke":
        mu, kappa = m["mu"], m["kappa"]
        return isotropic_from_lame(kappa - 2.0 * mu / 3.0, mu)
    if m["kind"] == "svk":
        return isotropic_stiffness(m["E"], m["nu"])
    raise ValueError(m["kind"])


def stiffness_field(phase, materials):
    """C(x)_ijkl as [3,3,3,3,z,y,x] ("stiffness tensor of the phase located at x")."""
    table = np.stack([material_stiffness(m) for m in materials])  # [P,3,3,3,3]
    return np.moveaxis(table[phase], (3, 4, 5, 6), (0, 1, 2, 3))


def contract(C, eps):
    """sigma_ij = C_ijkl eps_kl voxelwise."""
    return np.einsum("ijkl...,kl...->ij...", C, eps)


def neo_hookean(F, mu, kappa):
    """Compressible neo-Hookean (R14): W = mu/2 (tr F^T F - 3) - mu ln J + lam/2 (ln J)^2.

    Returns (P, K) with P_ij = mu (F_ij - Finv_ji) + lam ln J Finv_ji and
    K_ijkl = dP_ij/dF_kl = mu d_ik d_jl + (mu - lam ln J) Finv_li Finv_jk
             + lam Finv_ji Finv_lk.   F: [3,3,...]; mu, kappa broadcastable."""
    lam = kappa - 2.0 * mu / 3.0
    Fm = np.moveaxis(F, (0, 1), (-2, -1))
    J = np.linalg.det(Fm)
    if np.any(J <= 0):
        raise FloatingPointError("det F <= 0")
    Finv = np.moveaxis(np.linalg.inv(Fm), (-2, -1), (0, 1))  # Finv[a,b] = (F^-1)_ab
    lnJ = np.log(J)
    FinvT = np.swapaxes(Finv, 0, 1)
    P = mu * (F - FinvT) + lam * lnJ * FinvT
    c1 = mu - lam * lnJ
    K = np.zeros((3, 3, 3, 3) + F.shape[2:])
    for i in range(3):
        for j in range(3):
            for k in range(3):
                for l in range(3):
                    K[i, j, k, l] = (mu * I3[i, k] * I3[j, l] + c1 * Finv[l, i] * Finv[j, k]
                                     + lam * Finv[j, i] * Finv[l, k])
    return P, K


def svk(F, E, nu):
    """Saint Venant-Kirchhoff (SS3.3 matrix and voids): W = lam/2 (tr E)^2 + mu E:E,
    E = (F^T F - I)/2.  Returns (P, K): S = lam tr(E) I + 2 mu E, P = F S, and
    K_ijkl = dP_ij/dF_kl = d_ik S_lj + lam F_ij F_kl + mu (F_il F_kj + (F F^T)_ik d_jl).
    F: [3,3,...]; E, nu broadcastable."""
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = E / (2.0 * (1.0 + nu))
    C = np.einsum("ki...,kj...->ij...", F, F)
    Eg = 0.5 * (C - I3.reshape((3, 3) + (1,) * (F.ndim - 2)))
    trE = Eg[0, 0] + Eg[1, 1] + Eg[2, 2]
    S = 2.0 * mu * Eg + lam * trE * I3.reshape((3, 3) + (1,) * (F.ndim - 2))
    P = np.einsum("ip...,pj...->ij...", F, S)
    B = np.einsum("ip...,kp...->ik...", F, F)
    K = np.zeros((3, 3, 3, 3) + F.shape[2:])
    for i in range(3):
        for j in range(3):
            for k in range(3):
                for l in range(3):
                    K[i, j, k, l] = (I3[i, k] * S[l, j] + lam * F[i, j] * F[k, l]
                                     + mu * (F[i, l] * F[k, j] + B[i, k] * I3[j, l]))
    return P, K


def hyperelastic(F, phase, materials):
    """(P, K) voxelwise for a finite-strain phase map (neo-Hookean R14 / SVK P:326 phases)."""
    kinds = np.array([m["kind"] for m in materials])
    P = np.zeros_like(F)
    K = np.zeros((3, 3) + F.shape)
    for kind in set(kinds.tolist()):
        sel = np.isin(phase, np.nonzero(kinds == kind)[0])
        Fs = F[:, :, sel]
        if kind == "neohooke":
            mu = np.array([m.get("mu", 0.0) for m in materials])[phase][sel]
            kap = np.array([m.get("kappa", 0.0) for m in materials])[phase][sel]
            Ps, Ks = neo_hookean(Fs, mu, kap)
        elif kind == "svk":
            E = np.array([m.get("E", 0.0) for m in materials])[phase][sel]
            nu = np.array([m.get("nu", 0.0) for m in materials])[phase][sel]
            Ps, Ks = svk(Fs, E, nu)
        else:
            raise ValueError(kind)
        P[:, :, sel] = Ps
        K[:, :, :, :, sel] = Ks
    return P, K


def _j2_root_bisect(s_tr, mu3, sy, rate_dt, nexp):
    """Root x>=0 of g(x) = s_tr - mu3 rate_dt x^n - sy (1 + x) by plain bisection (R16)."""
    lo = np.zeros_like(s_tr)
    hi = np.maximum(s_tr / sy - 1.0, 0.0)
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        g = s_tr - mu3 * rate_dt * mid ** nexp - sy * (1.0 + mid)
        lo = np.where(g > 0, mid, lo)
        hi = np.where(g > 0, hi, mid)
    return 0.5 * (lo + hi)


def j2_perzyna(eps, eps_p_n, E, nu, sy, nexp, edot0, dt):
    """Small-strain J2 elasto-viscoplastic, Perzyna overstress law (R16), backward Euler.

    eps_p_rate = edot0 <s_vm/sy - 1>^n (3/2) s/s_vm.  Returns
    (sigma, C_alg, eps_p, dp).  Arrays [3,3,...]; parameters broadcastable.
    Consistent tangent C_alg = kappa 1x1 + 2 mu theta I_dev - 2 mu thetabar n x n."""
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    kappa = lam + 2.0 * mu / 3.0
    ee = eps - eps_p_n
    tr = ee[0, 0] + ee[1, 1] + ee[2, 2]
    dev = ee - tr / 3.0 * I3.reshape((3, 3) + (1,) * (eps.ndim - 2))
    s_tr = 2 * mu * dev
    svm_tr = np.sqrt(1.5 * np.einsum("ij...,ij...->...", s_tr, s_tr))
    rate_dt = edot0 * dt
    yielding = svm_tr > sy
    x = np.where(yielding, _j2_root_bisect(np.where(yielding, svm_tr, 2 * sy), 3 * mu, sy, rate_dt, nexp), 0.0)
    dp = rate_dt * x ** nexp
    safe = np.where(svm_tr > 0, svm_tr, 1.0)
    nhat = np.where(yielding, 1.0, 0.0) * 1.5 * s_tr / safe  # (3/2) s/s_vm (flow direction)
    eps_p = eps_p_n + dp * nhat
    theta = np.where(yielding, 1.0 - 3 * mu * dp / safe, 1.0)
    s = theta * s_tr
    sigma = s + kappa * tr * I3.reshape((3, 3) + (1,) * (eps.ndim - 2))
    # H' = d(sy (1 + (dp/rate_dt)^(1/n)))/d dp = sy/(n rate_dt) (dp/rate_dt)^(1/n - 1)
    with np.errstate(divide="ignore", invalid="ignore"):
        Hp = np.where(yielding & (dp > 0), sy / (nexp * rate_dt) * (dp / rate_dt) ** (1.0 / nexp - 1.0), 0.0)
        thetabar = np.where(yielding, 1.0 / (1.0 + Hp / (3 * mu)) - (1.0 - theta), 0.0)
    nn = np.where(yielding, 1.0, 0.0) * s_tr / np.where(svm_tr > 0, np.sqrt(np.einsum("ij...,ij...->...", s_tr, s_tr)), 1.0)
    C = np.zeros((3, 3, 3, 3) + eps.shape[2:])
    for i in range(3):
        for j in range(3):
            for k in range(3):
                for l in range(3):
                    Idev = 0.5 * (I3[i, k] * I3[j, l] + I3[i, l] * I3[j, k]) - I3[i, j] * I3[k, l] / 3.0
                    C[i, j, k, l] = (kappa * I3[i, j] * I3[k, l] + 2 * mu * theta * Idev
                                     - 2 * mu * thetabar * nn[i, j] * nn[k, l])
    return sigma, C, eps_p, dp


# ----------------------------------------------------------------------------
# The DBFFT operator (P:116-121 Eq. (lineqf); P:164-176 mixed; P:214-215 finite)
# ----------------------------------------------------------------------------


def apply_K(u_hat, C, XI, e=None, finite=False):
    """Positive operator K u = -d : F( C : ( F^-1(s . u) + e ) )  (R3).

    `s` is the symmetric gradient (small strain) or the full gradient
    (finite strain, P:219/R2); C is [3,3,3,3,z,y,x] (stiffness or tangent K^i).
    Returns (f_hat, mean_sigma) where mean_sigma = <C:(eps + e)> (the xi = 0
    row of P:174 before masking).  f_hat = 0 on the null set Z."""
    g = grad_hat(u_hat, XI) if finite else sym_grad_hat(u_hat, XI)
    # real part = restriction to real fields (R6): rounding-level anti-Hermitian
    # parts of CG vectors lie in the kernel and are dropped here
    eps = ifft(g, check=False)
    if e is not None:
        eps = eps + e.reshape(3, 3, 1, 1, 1)
    sig = contract(C, eps)
    f = -div_hat(fft(sig), XI)
    f[:, null_set(XI)] = 0.0
    return f, volume_average(sig)


def rhs_from_stress(sig, XI):
    """b = d : F(sig) = F(div sig) (R3; right-hand side of P:118 / P:215 up to sign)."""
    b = div_hat(fft(sig), XI)
    b[:, null_set(XI)] = 0.0
    return b


def inner(a, b):
    """Real part of the Hermitian spectral inner product (mean-normalised spectra)."""
    return float(np.real(np.sum(np.conj(a) * b)))


# ----------------------------------------------------------------------------
# Preconditioner (Eqs. (pred1)-(pred3); R4, R12)
# ----------------------------------------------------------------------------


def acoustic(Cbar, XI):
    """A(xi)_ik = xi_j Cbar_ijkl xi_l at every frequency: [3,3,z,y,x]."""
    return np.einsum("ijkl,j...,l...->ik...", Cbar, XI, XI)


def precondition(r_hat, Cbar, XI):
    """z(xi) = M(xi) r(xi), M = [xi . Cbar . xi]^-1 for xi != 0; 0 on Z (R4)."""
    A = acoustic(Cbar, XI)
    Z = null_set(XI)
    Am = np.moveaxis(A, (0, 1), (-2, -1)).copy()
    Am[Z] = np.eye(3)
    rv = np.moveaxis(r_hat, 0, -1)[..., None]
    z = np.linalg.solve(Am, rv)[..., 0]
    z = np.moveaxis(z, -1, 0)
    z[:, Z] = 0.0
    return z


def macro_basis(mask, symmetric):
    """Orthonormal basis (Frobenius) of the stress-controlled macro subspace.

    Small strain (symmetric): e_i(x)e_i for masked diagonals and
    (e_i(x)e_j + e_j(x)e_i)/sqrt 2 for masked off-diagonal pairs.
    Finite strain: unit tensors of the masked entries."""
    basis = []
    for i in range(3):
        for j in range(3):
            if not mask[i, j]:
                continue
            E = np.zeros((3, 3))
            if symmetric:
                if j < i:
                    continue
                if i == j:
                    E[i, i] = 1.0
                else:
                    E[i, j] = E[j, i] = 1.0 / np.sqrt(2.0)
            else:
                E[i, j] = 1.0
            basis.append(E)
    return basis


def macro_precondition(r_e, Cbar, basis):
    """z_e = (P Cbar P)^-1 r_e on the stress-controlled subspace (R4)."""
    if not basis:
        return np.zeros((3, 3))
    M = np.array([[np.einsum("ij,ijkl,kl->", Ea, Cbar, Eb) for Eb in basis] for Ea in basis])
    rv = np.array([np.sum(Ea * r_e) for Ea in basis])
    c = np.linalg.solve(M, rv)
    return sum(ci * Ea for ci, Ea in zip(c, basis))


# ----------------------------------------------------------------------------
# Preconditioned CG on the augmented system {u_hat | e}
# ----------------------------------------------------------------------------


class Aug:
    """Vector {u_hat | e}: fluctuation spectrum + macro block."""

    def __init__(self, u, e):
        self.u, self.e = u, e

    def dot(self, o):
        return inner(self.u, o.u) + float(np.sum(self.e * o.e))


def pcg(apply_A, precond, b, mean_sig0, tol, max_iter=10000, macro=False):
    """Preconditioned conjugate gradients ("conjugate gradient method for
    complex numbers"; at most 1e4 iterations), x0 = 0.

    Stop test (R7): eps_eq = ||r_u|| / ||<sigma>|| <= tol, where by Parseval
    ||r_u|| = ||div sigma||_L2 (Eq. (chedckeq)); under mixed control
    also eps_load = ||r_e|| / ||<sigma>|| <= tol (R9).  <sigma> of
    the current iterate is mean_sig0 + sum alpha_k <sigma(p_k)> (R7).  At exit
    the true residual b - A x is recomputed and iteration continues if it fails.
    apply_A(v) -> (Aug, mean_sigma_of_v).  Returns (x, iters, history)."""
    x = Aug(np.zeros_like(b.u), np.zeros((3, 3)))
    r = Aug(b.u.copy(), b.e.copy())
    msig = mean_sig0.copy()
    hist = []

    def errors(r, msig):
        den = max(np.linalg.norm(msig), 1e-300)
        eq = np.sqrt(inner(r.u, r.u)) / den
        ld = np.linalg.norm(r.e) / den if macro else 0.0
        return eq, ld

    it = 0
    eq, ld = errors(r, msig)
    hist.append(eq)
    if eq <= tol and ld <= tol:
        return x, 0, hist
    while True:
        z = precond(r)
        p = Aug(z.u.copy(), z.e.copy())
        rz = r.dot(z)
        while it < max_iter:
            q, msig_p = apply_A(p)
            pq = p.dot(q)
            if not (pq > 0):
                raise FloatingPointError("CG breakdown: <p,Kp> <= 0")
            alpha = rz / pq
            x = Aug(x.u + alpha * p.u, x.e + alpha * p.e)
            r = Aug(r.u - alpha * q.u, r.e - alpha * q.e)
            msig = msig + alpha * msig_p
            it += 1
            eq, ld = errors(r, msig)
            hist.append(eq)
            if eq <= tol and ld <= tol:
                break
            z = precond(r)
            rz_new = r.dot(z)
            beta = rz_new / rz
            rz = rz_new
            p = Aug(z.u + beta * p.u, z.e + beta * p.e)
        # true-residual confirmation (R7)
        Ax, msig_x = apply_A(x)
        r = Aug(b.u - Ax.u, b.e - Ax.e)
        msig = mean_sig0 + msig_x
        eq, ld = errors(r, msig)
        if (eq <= tol and ld <= tol) or it >= max_iter:
            return x, it, hist


# ----------------------------------------------------------------------------
# Drivers: small strain linear and finite strain Newton
# ----------------------------------------------------------------------------


def _masks(load):
    mask = np.asarray(load["mask"], bool)
    target = np.asarray(load["target"], float)
    return mask, target


_MANDEL_IDX = [(0, 0), (1, 1), (2, 2), (1, 2), (0, 2), (0, 1)]
_MANDEL_W = np.array([1.0, 1.0, 1.0, np.sqrt(2.0), np.sqrt(2.0), np.sqrt(2.0)])


def to_mandel(C):
    """6x6 Mandel matrix(es) of minor-symmetric C[i,j,k,l,...] (leading four indices)."""
    M = np.empty((6, 6) + C.shape[4:])
    for a, (i, j) in enumerate(_MANDEL_IDX):
        for b, (k, l) in enumerate(_MANDEL_IDX):
            M[a, b] = C[i, j, k, l] * _MANDEL_W[a] * _MANDEL_W[b]
    return M


def from_mandel(M):
    """Full C[i,j,k,l] (minor and major symmetric) of a 6x6 Mandel matrix."""
    C = np.empty((3, 3, 3, 3))
    for a, (i, j) in enumerate(_MANDEL_IDX):
        for b, (k, l) in enumerate(_MANDEL_IDX):
            v = M[a, b] / (_MANDEL_W[a] * _MANDEL_W[b])
            for (p, q) in {(i, j), (j, i)}:
                for (r, s) in {(k, l), (l, k)}:
                    C[p, q, r, s] = v
    return C


def reference_medium(C, medium="arithmetic"):
    """Reference stiffness of the preconditioner M(xi) = [xi.C0.xi]^-1 (Eq. pred3).

    "arithmetic": C0 = <C(x)> (the paper's choice).  "harmonic": <C(x)^-1>^-1 (Reuss),
    "hill": their mean - the "new ad-hoc preconditioners" left as future work at P:394
    (SURVEY 8(f4) reading: any symmetric positive-definite C0 keeps PCG valid and changes only
    the iteration count).  Small-strain (minor-symmetric) fields only for the harmonic mean."""
    CA = volume_average(C)
    if medium == "arithmetic":
        return CA
    M = to_mandel(C)                                    # 6 x 6 x nz x ny x nx
    Mv = np.moveaxis(M.reshape(6, 6, -1), -1, 0)        # voxels x 6 x 6
    S = np.linalg.inv(Mv).mean(axis=0)                  # <C^-1> (Mandel)
    CR = from_mandel(np.linalg.inv(S))
    if medium == "harmonic":
        return CR
    if medium == "hill":
        return 0.5 * (CA + CR)
    raise ValueError(medium)


def solve_small_strain(phase, materials, load, tol=1e-10, max_iter=10000, L=(1.0, 1.0, 1.0), C=None,
                       medium="arithmetic"):
    """Linear small-strain DBFFT under strain/stress/mixed control.

    Unknown {u_hat | eps_f}.  eps_U = target on strain-controlled
    components, sigma_f = target on stress-controlled ones (IJ != ij).
    b_u = d:F(C:eps_U) (P:173 rhs, R3), b_e = P(sigma_f - <C:eps_U>).
    Returns dict(u_hat, e, eps, sig, mean_eps, mean_sig, iters, hist)."""
    nz, ny, nx = phase.shape
    XI = frequency_grid((nx, ny, nz), L)
    if C is None:
        C = stiffness_field(phase, materials)
    mask, target = _masks(load)
    eps_U = np.where(mask, 0.0, target)
    sig_f = np.where(mask, target, 0.0)
    Cbar = reference_medium(C, medium)  # P:255 (arithmetic, default) / P:394 variants
    basis = macro_basis(mask, symmetric=True)
    sig_U = contract(C, eps_U.reshape(3, 3, 1, 1, 1) * np.ones((1, 1, nz, ny, nx)))
    mean_sig_U = volume_average(sig_U)
    b = Aug(rhs_from_stress(sig_U, XI), np.where(mask, sig_f - mean_sig_U, 0.0))
    macro = bool(mask.any())

    def apply_A(v):
        f, ms = apply_K(v.u, C, XI, e=v.e if macro else None)
        return Aug(f, np.where(mask, ms, 0.0)), ms

    def precond(r):
        return Aug(precondition(r.u, Cbar, XI), macro_precondition(r.e, Cbar, basis))

    x, iters, hist = pcg(apply_A, precond, b, mean_sig_U, tol, max_iter, macro)
    eps = ifft(sym_grad_hat(x.u, XI)) + (eps_U + x.e).reshape(3, 3, 1, 1, 1)
    sig = contract(C, eps)
    return dict(u_hat=x.u, e=x.e, eps=eps, sig=sig, mean_eps=volume_average(eps),
                mean_sig=volume_average(sig), iters=iters, hist=hist, XI=XI)


# ----------------------------------------------------------------------------
# Residual monitors (P:270-290 Eqs. chedckeq / chedckcomp / chedckimp; finite strain
# P:327-330).  Derivatives are the method's discrete ones (i xi, Eq. 1 with R1).
# ----------------------------------------------------------------------------
def _levi_civita():
    e = np.zeros((3, 3, 3))
    e[0, 1, 2] = e[1, 2, 0] = e[2, 0, 1] = 1.0
    e[0, 2, 1] = e[2, 1, 0] = e[1, 0, 2] = -1.0
    return e


def incompatibility(field, XI, finite):
    """max over components and voxels of |curl curl eps| (small strain, the symmetric part of
    `field`, Eq. chedckcomp) or of |curl_0 F| (finite strain, row-wise curl
    (curl F)_ij = e_jkl d_k F_il).  field: [3,3,z,y,x] real.  Unnormalised."""
    e = _levi_civita()
    dhat = 1j * XI                                          # spectral d_k
    if finite:
        Fh = fft(field)
        C = np.einsum("jkl,k...,il...->ij...", e, dhat, Fh)
        return float(np.max(np.abs(ifft(C, check=False))))
    eps = 0.5 * (field + np.swapaxes(field, 0, 1))
    Eh = fft(eps)
    eta = np.einsum("ikl,jmn,k...,m...,ln...->ij...", e, e, dhat, dhat, Eh)
    return float(np.max(np.abs(ifft(eta, check=False))))


def equilibrium_residual(sig, XI):
    """||div sigma||_L2 / ||<sigma>|| (Eq. chedckeq; P / reference divergence at finite
    strain).  ||.||_L2 = voxel-mean L2 norm = sqrt(sum |f_hat|^2) (Parseval, R5)."""
    f = div_hat(fft(sig), XI)
    return float(np.sqrt(np.sum(np.abs(f) ** 2)) / np.linalg.norm(volume_average(sig)))


def loading_residual(mean_eps, mean_sig, target, mask):
    """Eq. chedckimp: ||<eps> - eps_bar|| / ||eps_bar|| over the strain-controlled
    components, ||<sigma> - sigma_bar|| / ||<sigma>|| over the stress-controlled ones (mixed
    control: the larger)."""
    de = np.where(mask, 0.0, mean_eps - target)
    te = np.where(mask, 0.0, target)
    ds = np.where(mask, mean_sig - target, 0.0)
    r1 = np.linalg.norm(de) / np.linalg.norm(te) if np.linalg.norm(te) > 0 else np.linalg.norm(de)
    return float(max(r1, np.linalg.norm(ds) / np.linalg.norm(mean_sig)))


def displacement(u_hat):
    """Real-space fluctuation displacement u~(x) (obtained directly)."""
    return ifft(u_hat)


class FiniteStrainState:
    """Converged state between increments: u_hat (fluctuation) and Fbar."""

    def __init__(self, n):
        nx, ny, nz = n
        self.u_hat = np.zeros((3, nz, ny, nx), dtype=np.complex128)
        self.Fbar = np.eye(3)


def solve_finite_increment(state, phase, materials, load, tol=1e-10, tol_newton=1e-6,
                           max_newton=25, max_iter=10000, L=(1.0, 1.0, 1.0)):
    """One load increment of finite-strain DBFFT with Newton.

    F^0 = Fbar^{k+1} + grad u~^k.  Newton iteration i: P(F^i), K^i
    (P:204), b = F(div P) and P(Pbar - <P>) (P:215, P:233-234 read as R11);
    K_bar and M at i = 0 (R12); solve the linear system by
    PCG; u~ += du~, Fbar_f += dF_f; stop when max|grad du~ + dF_f| < tol_newton
    (R10).  Materials: neo-Hookean (R14) / SVK per phase.  Modifies `state`."""
    nz, ny, nx = phase.shape
    XI = frequency_grid((nx, ny, nz), L)
    mask, target = _masks(load)
    Fbar = np.where(mask, state.Fbar, target)
    P_f = np.where(mask, target, 0.0)
    basis = macro_basis(mask, symmetric=False)
    macro = bool(mask.any())
    F = Fbar.reshape(3, 3, 1, 1, 1) + ifft(grad_hat(state.u_hat, XI))
    total_cg = 0
    newton = 0
    Kbar = None
    while True:
        P, K = hyperelastic(F, phase, materials)
        meanP = volume_average(P)
        b = Aug(rhs_from_stress(P, XI), np.where(mask, P_f - meanP, 0.0))
        if Kbar is None:
            Kbar = volume_average(K)

        def apply_A(v, K=K):
            f, ms = apply_K(v.u, K, XI, e=v.e if macro else None, finite=True)
            return Aug(f, np.where(mask, ms, 0.0)), ms

        def precond(r, Kbar=Kbar):
            return Aug(precondition(r.u, Kbar, XI), macro_precondition(r.e, Kbar, basis))

        dx, iters, _ = pcg(apply_A, precond, b, meanP, tol, max_iter, macro)
        total_cg += iters
        newton += 1
        # real part (R6): the correction's rounding-level anti-Hermitian CG noise is dropped
        dG = ifft(grad_hat(dx.u, XI), check=False) + dx.e.reshape(3, 3, 1, 1, 1)
        state.u_hat = state.u_hat + dx.u
        Fbar = Fbar + dx.e
        F = F + dG
        if np.max(np.abs(dG)) < tol_newton or newton >= max_newton:
            break
    last = np.max(np.abs(dG))
    state.Fbar = Fbar
    P, _ = hyperelastic(F, phase, materials)
    return dict(F=F, P=P, mean_F=volume_average(F), mean_P=volume_average(P),
                cg_iters=total_cg, newton_iters=newton, converged=bool(last < tol_newton))


class J2State:
    """Committed J2 state (P:190 internal variables; committed at acceptance)."""

    def __init__(self, n):
        nx, ny, nz = n
        self.u_hat = np.zeros((3, nz, ny, nx), dtype=np.complex128)
        self.ebar = np.zeros((3, 3))
        self.eps_p = np.zeros((3, 3, nz, ny, nx))


def solve_j2_increment(state, phase, materials, load, dt, tol=1e-10, tol_newton=1e-6,
                       max_newton=25, max_iter=10000, L=(1.0, 1.0, 1.0)):
    """One increment of small-strain DBFFT with Newton for the J2-Perzyna law.

    Same Newton structure as P:201-221 with sym grad and the
    algorithmic tangent; state committed at the end.  Strain control only
    (R17).  Returns `converged` (max|d eps| < tol_newton before max_newton).
    Pinned by the elasto-viscoplastic laminate (per-layer uniform strains, out-of-plane
    tractions continuous: a 3-unknown root per increment) and by equilibrium + Hill-Mandel
    on a heterogeneous polycrystal twin (tests/test_oracle_pins.py)."""
    nz, ny, nx = phase.shape
    XI = frequency_grid((nx, ny, nz), L)
    mask, target = _masks(load)
    assert not mask.any()
    par = {k: np.array([m[k] for m in materials])[phase] for k in ("E", "nu", "sigma_y", "n", "edot0")}
    eps = target.reshape(3, 3, 1, 1, 1) + ifft(sym_grad_hat(state.u_hat, XI))
    total_cg = 0
    newton = 0
    Cbar = None
    while True:
        sig, Calg, eps_p, _ = j2_perzyna(eps, state.eps_p, par["E"], par["nu"], par["sigma_y"],
                                         par["n"], par["edot0"], dt)
        mean_sig = volume_average(sig)
        b = Aug(rhs_from_stress(sig, XI), np.zeros((3, 3)))
        if Cbar is None:
            Cbar = volume_average(Calg)

        def apply_A(v, C=Calg):
            f, ms = apply_K(v.u, C, XI)
            return Aug(f, np.zeros((3, 3))), ms

        def precond(r, Cbar=Cbar):
            return Aug(precondition(r.u, Cbar, XI), np.zeros((3, 3)))

        dx, iters, _ = pcg(apply_A, precond, b, mean_sig, tol, max_iter, False)
        total_cg += iters
        newton += 1
        de = ifft(sym_grad_hat(dx.u, XI), check=False)  # real part (R6)
        state.u_hat = state.u_hat + dx.u
        eps = eps + de
        last = np.max(np.abs(de))
        if last < tol_newton or newton >= max_newton:
            break
    sig, _, eps_p, dp = j2_perzyna(eps, state.eps_p, par["E"], par["nu"], par["sigma_y"],
                                   par["n"], par["edot0"], dt)
    state.eps_p = eps_p
    state.ebar = target.copy()
    return dict(eps=eps, sig=sig, mean_eps=volume_average(eps), eps_p=eps_p, dp=dp,
                mean_sig=volume_average(sig), cg_iters=total_cg, newton_iters=newton,
                converged=bool(last < tol_newton))


# ----------------------------------------------------------------------------
# Dense assembly (pins P5, P6): the operator as a real matrix on real fields
# ----------------------------------------------------------------------------


def dense_operator(C, n, finite=False, L=(1.0, 1.0, 1.0)):
    """Real matrix A with (A v)(x) = F^-1(K F(v))(x) for real fields v, v in R^{3N}.

    Column m is K applied to the m-th real unit field.  A is symmetric (the
    spectral inner product is the voxel mean), its kernel is spanned by the
    modes of Z."""
    nx, ny, nz = n
    XI = frequency_grid(n, L)
    Nv = nx * ny * nz
    A = np.zeros((3 * Nv, 3 * Nv))
    for m in range(3 * Nv):
        v = np.zeros(3 * Nv)
        v[m] = 1.0
        f, _ = apply_K(fft(v.reshape(3, nz, ny, nx)), C, XI, finite=finite)
        A[:, m] = ifft(f).ravel()
    return A
