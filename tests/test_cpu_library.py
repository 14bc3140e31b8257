"""CPU-side checks (no GPU): the C-ABI library builds/loads and exports every symbol that
include/dbfft.h declares; host-side marshalling helpers; seeded inputs are deterministic."""
import ctypes
import os
import re

import numpy as np
import pytest

from synth import configs, microstructure as ms
from synth.rng import SplitMix64

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1905_12725_b200 import build, dbfft
    build.build()  # no-op when up to date
    return dbfft.load_library()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "dbfft.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dbfft_[A-Za-z_]+)\s*\(", src)))


def test_header_symbols_exported(lib):
    syms = header_symbols()
    assert len(syms) >= 16
    for s in syms:
        assert hasattr(lib, s), s
    from paper_1905_12725_b200 import dbfft
    assert sorted(dbfft.EXPORTS) == syms


def test_default_opts_and_names(lib):
    o = lib.dbfft_default_opts()
    assert o.tol_eq == 1e-10 and o.tol_load == 1e-10 and o.tol_newton == 1e-6
    assert o.max_cg == 10000 and o.max_newton == 25
    names = [lib.dbfft_profile_name(k).decode() for k in range(lib.dbfft_profile_count())]
    assert "pass_X" in names and "cg_update" in names


def test_invalid_grid_rejected_without_device(lib):
    h = ctypes.c_void_p()
    n = (ctypes.c_int32 * 3)(12, 8, 8)  # not a power of two
    L = (ctypes.c_double * 3)(1, 1, 1)
    st = lib.dbfft_create(n, L, 6, None, ctypes.byref(h))
    assert st == 1  # DBFFT_E_INVALID_GRID (validated before any CUDA call)
    assert b"power" in lib.dbfft_last_error(None)
    n = (ctypes.c_int32 * 3)(8, 8, 8)
    st = lib.dbfft_create(n, L, 7, None, ctypes.byref(h))
    assert st == 2  # bad kinematics


def test_half_spectrum_layout_roundtrip():
    from spectra import full_from_half, half_spectrum
    u = ms.random_field((3, 6, 4, 8), 3)  # [3][z][y][x]: n = (8, 4, 6)
    h = half_spectrum(u)
    assert h.shape == (3, 4, 6, 5)  # [3][ky][kz][kx<=n1/2]
    full = full_from_half(h, 8)
    ref = np.fft.fftn(u, axes=(1, 2, 3)) / u[0].size
    assert np.max(np.abs(full - ref)) < 1e-15


def test_material_marshalling():
    from paper_1905_12725_b200.dbfft import MAT_CUBIC, MAT_J2, material_record
    R = ms.random_rotations(1, 1)[0]
    rec = material_record(dict(kind="cubic", C11=1.0, C12=2.0, C44=3.0, R=R))
    assert rec.kind == MAT_CUBIC and list(rec.p[:3]) == [1.0, 2.0, 3.0]
    assert np.allclose(np.array(rec.p[3:12]).reshape(3, 3), R)
    rec = material_record(dict(kind="j2", E=2e5, nu=0.3, sigma_y=300.0, n=20.0, edot0=1e-3))
    assert rec.kind == MAT_J2 and list(rec.p[:5]) == [2e5, 0.3, 300.0, 20.0, 1e-3]


def test_synth_determinism_and_geometry():
    assert [hex(int(v)) for v in SplitMix64(0).next_u64(2)] == ["0xe220a8397b1dcdaf", "0x6e789e6aa1b965f4"]
    assert configs.c1()["phase"].sum() == 32  # R20
    a = configs.c2(n=32, radius_vox=3)["phase"]
    b = configs.c2(n=32, radius_vox=3)["phase"]
    assert np.array_equal(a, b) and abs(a.mean() - 0.2) < 0.03
    R = ms.random_rotations(50, 5)
    assert np.allclose(np.einsum("nij,nkj->nik", R, R), np.eye(3), atol=1e-14)
    assert np.allclose(np.linalg.det(R), 1.0)
    ph, seeds = ms.voronoi((16, 16, 16), 10, 3)
    assert set(np.unique(ph)) <= set(range(10))


def test_env_struct_matches_header():
    """The binding's ctypes dbfft_env mirrors include/dbfft.h field by field, in order (a mismatch
    would hand the library garbage for e.g. the allocator hooks or pencil_rows)."""
    from paper_1905_12725_b200 import dbfft
    src = open(os.path.join(ROOT, "include", "dbfft.h")).read()
    body = re.search(r"typedef struct \{(.*?)\} dbfft_env;", src, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        m = re.search(r"\(\*\s*(\w+)\)", decl)
        names += [m.group(1)] if m else re.findall(r"(\w+)\s*(?:,|$)", decl)
    assert names == [f[0] for f in dbfft.Env._fields_]
    assert "pencil_rows" in names
