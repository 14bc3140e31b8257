"""Writes the oracle references of the full-size config parity tests (tests/test_gpu_configs.py).

Calls ONLY oracle/ (the plain fp64 CPU DBFFT) and synth/ (the seeded inputs shared by both
sides); no value here comes from the CUDA path.  The oracle at 128^3 / 256^3 takes minutes to
tens of minutes on CPU, longer than a GPU test should wait, so its results are stored — sampled:
macroscopic quantities in full, fields at a seeded set of voxels / frequencies (SAMPLES of them,
plus the full-field norms for relative errors).  Usage:

    python tests/golden/make_config_refs.py c3 c5s c4op c4inc    # -> tests/golden/<name>_ref.npz
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import dbfft_oracle as O  # noqa: E402
from synth import configs, microstructure as ms  # noqa: E402
from synth.rng import SplitMix64  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SAMPLES = 20000
SAMPLE_SEED = 424242


def voxel_sample(n, seed=SAMPLE_SEED, count=SAMPLES):
    """Seeded voxel indices (flat [z][y][x]), first and last voxel included."""
    N = n[0] * n[1] * n[2]
    idx = np.unique(np.concatenate([[0, N - 1], (SplitMix64(seed).uniform(count) * N).astype(np.int64)]))
    return idx


def freq_sample(n, seed=SAMPLE_SEED + 1, count=SAMPLES):
    """Seeded half-spectrum points (kz, ky, kx <= n1/2), with the zero, Nyquist and axis points."""
    n1, n2, n3 = n
    u = SplitMix64(seed).uniform(3 * count).reshape(3, count)
    kx = (u[0] * (n1 // 2 + 1)).astype(np.int64)
    ky = (u[1] * n2).astype(np.int64)
    kz = (u[2] * n3).astype(np.int64)
    special = [(0, 0, 0), (0, 0, n1 // 2), (n3 // 2, n2 // 2, n1 // 2), (0, 1, 0), (1, 0, 0), (0, 0, 1),
               (n3 // 2, 0, 3), (5, n2 // 2, 0), (n3 - 1, n2 - 1, n1 // 2 - 1)]
    pts = set(zip(kz.tolist(), ky.tolist(), kx.tolist())) | set(special)
    return np.array(sorted(pts), dtype=np.int64)   # [m, 3] = (kz, ky, kx)


def c3():
    cfg = configs.c3()
    L = cfg["loads"][0]
    t0 = time.time()
    r = O.solve_small_strain(cfg["phase"], cfg["materials"], L, tol=1e-10)
    vs = voxel_sample(cfg["n"])
    sig = r["sig"].reshape(9, -1)
    eps = r["eps"].reshape(9, -1)
    return dict(mean_sig=r["mean_sig"], mean_eps=r["mean_eps"], cg_iters=r["iters"], voxels=vs,
                sig=sig[:, vs], eps=eps[:, vs], sig_norm=np.linalg.norm(sig), eps_norm=np.linalg.norm(eps),
                seconds=time.time() - t0)


C5S_INCREMENTS = 3


def c5s():
    cfg = configs.c5s(increments=C5S_INCREMENTS)
    st = O.J2State(cfg["n"])
    out = dict(mean_sig=[], mean_eps=[], newton=[], cg=[])
    t0 = time.time()
    for k, L in enumerate(cfg["loads"]):
        r = O.solve_j2_increment(st, cfg["phase"], cfg["materials"], L, cfg["dt"], tol=1e-10)
        assert r["converged"]
        out["mean_sig"].append(r["mean_sig"])
        out["mean_eps"].append(r["mean_eps"])
        out["newton"].append(r["newton_iters"])
        out["cg"].append(r["cg_iters"])
        print(f"c5s increment {k + 1}: newton {r['newton_iters']} cg {r['cg_iters']} ({time.time() - t0:.0f} s)",
              flush=True)
    vs = voxel_sample(cfg["n"])
    f = {k: r[k].reshape(9, -1) for k in ("sig", "eps", "eps_p")}
    out = {k: np.array(v) for k, v in out.items()}
    out.update(voxels=vs, sig=f["sig"][:, vs], eps=f["eps"][:, vs], eps_p=f["eps_p"][:, vs],
               sig_norm=np.linalg.norm(f["sig"]), eps_norm=np.linalg.norm(f["eps"]),
               eps_p_norm=np.linalg.norm(f["eps_p"]), plastic_fraction=float(np.mean(r["dp"] > 0)),
               seconds=time.time() - t0)
    return out


C4OP_F_SEED, C4OP_U_SEED, C4OP_F_AMP = 4401, 4402, 0.05


def c4op():
    """One heterogeneous c4 operator application at 256^3: the tangent of the c4 phase map at
    F = I + 0.05 N(0,1) (seeded), applied to a seeded white-noise displacement spectrum."""
    cfg = configs.c4()
    n = cfg["n"]
    ph = cfg["phase"]
    t0 = time.time()
    F = np.eye(3).reshape(3, 3, 1, 1, 1) + C4OP_F_AMP * ms.random_field((3, 3, n[2], n[1], n[0]), C4OP_F_SEED)
    mu = np.array([m["mu"] for m in cfg["materials"]])[ph]
    kap = np.array([m["kappa"] for m in cfg["materials"]])[ph]
    _, K = O.neo_hookean(F, mu, kap)
    del F
    u = ms.random_field((3, n[2], n[1], n[0]), C4OP_U_SEED)
    uh = O.fft(u)
    del u
    f, msig = O.apply_K(uh, K, O.frequency_grid(n), finite=True)
    del K, uh
    pts = freq_sample(n)
    vals = f[:, pts[:, 0], pts[:, 1], pts[:, 2]]
    return dict(points=pts, f=vals, f_norm=np.linalg.norm(f), mean_sig=msig, seconds=time.time() - t0)


def c4inc():
    """c4's first load increment at 256^3 (Newton-PCG, mixed control P_xx = P_yy = 0, F_zz = 1.01):
    macro F / P, Newton and PCG counts, sampled F and P fields."""
    cfg = configs.c4()
    st = O.FiniteStrainState(cfg["n"])
    t0 = time.time()
    r = O.solve_finite_increment(st, cfg["phase"], cfg["materials"], cfg["loads"][0], tol=1e-10)
    assert r["converged"]
    vs = voxel_sample(cfg["n"])
    F = r["F"].reshape(9, -1)
    P = r["P"].reshape(9, -1)
    return dict(mean_F=r["mean_F"], mean_P=r["mean_P"], newton=r["newton_iters"], cg=r["cg_iters"], voxels=vs,
                F=F[:, vs], P=P[:, vs], F_norm=np.linalg.norm(F), P_norm=np.linalg.norm(P), seconds=time.time() - t0)


if __name__ == "__main__":
    for name in sys.argv[1:] or ["c3", "c5s", "c4op"]:
        res = globals()[name]()
        np.savez_compressed(os.path.join(HERE, f"{name}_ref.npz"), **res)
        print(name, "done", f"{res['seconds']:.0f} s", flush=True)
