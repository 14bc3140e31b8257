"""Seeded voxel microstructures (phase maps) on a periodic unit cell L = (1,1,1).

Arrays are indexed [z][y][x] (x fastest), dtype uint16, as SURVEY "Notation"
fixes.  A voxel (i,j,k) has centre ((i+1/2)/n1, (j+1/2)/n2, (k+1/2)/n3): the
paper's fields live "at the center of each voxel" (section 2.1).
Geometry readings R20/R21 are implemented here once and
fed identically to both sides, so geometry is not a parity risk.
"""
import numpy as np
from .rng import SplitMix64


def voxel_centres(n):
    """Per-axis voxel-centre coordinates in cell units (x, y, z)."""
    return [(np.arange(m, dtype=np.float64) + 0.5) / m for m in n]


def centred_sphere(n, radius=0.25):
    """c1 (R20): phase 1 inside the sphere of `radius` centred at (1/2,1/2,1/2)."""
    x, y, z = voxel_centres(n)
    d2 = (x[None, None, :] - 0.5) ** 2 + (y[None, :, None] - 0.5) ** 2 + (z[:, None, None] - 0.5) ** 2
    return (d2 < radius * radius).astype(np.uint16)


def laminate(n, axis=0, thickness=None):
    """Two-phase laminate with interfaces normal to `axis` (0=x,1=y,2=z).

    Phase 1 occupies voxel indices [0, thickness) along `axis` (default: half)."""
    m = n[axis]
    t = m // 2 if thickness is None else thickness
    idx = (np.arange(m) < t).astype(np.uint16)
    shape = [1, 1, 1]
    shape[2 - axis] = m
    return np.broadcast_to(idx.reshape(shape), (n[2], n[1], n[0])).astype(np.uint16).copy()


def _min_image(d):
    return d - np.round(d)


def rsa_spheres(n, count, radius_vox, seed, max_tries=2_000_000):
    """Random sequential addition of `count` non-overlapping spheres (R21).

    Centres uniform in the cell; a candidate is accepted when its minimum-image
    distance to every accepted centre is >= 2r.  Voxel membership is
    centre-in (minimum image).  Returns (phase map, centres[count,3])."""
    rng = SplitMix64(seed)
    r = radius_vox / n[0]
    centres = np.empty((0, 3))
    tries = 0
    while len(centres) < count:
        if tries > max_tries:
            raise RuntimeError("RSA jammed")
        c = rng.uniform(3)
        tries += 1
        if len(centres):
            d = _min_image(centres - c)
            if np.min(np.einsum("ij,ij->i", d, d)) < (2 * r) ** 2:
                continue
        centres = np.vstack([centres, c])
    phase = np.zeros((n[2], n[1], n[0]), dtype=np.uint16)
    xs = voxel_centres(n)
    for c in centres:
        sl, dd = [], []
        for a in range(3):
            m = n[a]
            lo = int(np.floor((c[a] - r) * m)) - 1
            hi = int(np.ceil((c[a] + r) * m)) + 1
            ids = np.arange(lo, hi + 1)
            coords = xs[a][ids % m]
            dd.append(_min_image(coords - c[a]))
            sl.append(ids % m)
        d2 = dd[2][:, None, None] ** 2 + dd[1][None, :, None] ** 2 + dd[0][None, None, :] ** 2
        inside = d2 < r * r
        zz, yy, xx = np.nonzero(inside)
        phase[sl[2][zz], sl[1][yy], sl[0][xx]] = 1
    return phase, centres


def voronoi(n, grains, seed, chunk=1 << 22):
    """Periodic Voronoi tessellation with `grains` uniform seeds (R21).

    Grain id = nearest seed under the minimum-image metric (scipy cKDTree with
    periodic boxsize).  Exact distance ties have probability zero for
    continuous seeds.  Returns (phase map, seeds[grains,3])."""
    from scipy.spatial import cKDTree
    rng = SplitMix64(seed)
    seeds = rng.uniform(3 * grains).reshape(grains, 3)
    tree = cKDTree(seeds, boxsize=1.0)
    xs = voxel_centres(n)
    phase = np.empty(n[0] * n[1] * n[2], dtype=np.uint16)
    total = phase.size
    plane = n[0] * n[1]
    for start in range(0, total, chunk):
        stop = min(total, start + chunk)
        idx = np.arange(start, stop)
        pts = np.stack([xs[0][idx % n[0]], xs[1][(idx // n[0]) % n[1]], xs[2][idx // plane]], axis=1)
        _, g = tree.query(pts, workers=-1)
        phase[start:stop] = g
    return phase.reshape(n[2], n[1], n[0]), seeds


def random_rotations(count, seed):
    """Uniform SO(3) samples: unit quaternion from 4 standard normals (R21)."""
    rng = SplitMix64(seed)
    q = rng.normal(4 * count).reshape(count, 4)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    R = np.empty((count, 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z); R[:, 0, 1] = 2 * (x * y - w * z); R[:, 0, 2] = 2 * (x * z + w * y)
    R[:, 1, 0] = 2 * (x * y + w * z); R[:, 1, 1] = 1 - 2 * (x * x + z * z); R[:, 1, 2] = 2 * (y * z - w * x)
    R[:, 2, 0] = 2 * (x * z - w * y); R[:, 2, 1] = 2 * (y * z + w * x); R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def lognormal(count, seed, median, sigma_log):
    """Per-grain lognormal values median*exp(sigma_log*Z) (c5 yield stress, R21)."""
    return median * np.exp(sigma_log * SplitMix64(seed).normal(count))


def random_field(shape, seed):
    """i.i.d. N(0,1) real field (operator-parity inputs)."""
    return SplitMix64(seed).normal(int(np.prod(shape))).reshape(shape)
