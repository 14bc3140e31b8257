"""Out-of-bounds and race checks of our own (compute-sanitizer is not available on the GPU pool):

  * guard bands: every device buffer of a ctx comes from an allocator (dbfft_env dev_alloc /
    dev_free hooks) that surrounds it with 64 KB guard bands of a known byte pattern; after the
    hot-path kernels ran — register and TMA column passes incl. the N = 512 two-warp columns,
    pass_X incl. n1 = 512, the fused F3 update, the device-side PCG loop, constitutive kinds,
    loopback slabs, monitors and the tangent field — every band is intact (a stray store of any
    kernel into a neighbouring buffer lands in a band: buffers are laid out band | data | band);
  * determinism: repeated operator applications and repeated solves are bit-identical (the
    reductions are fixed-order by design; a shared-memory race or a missing barrier shows up as
    run-to-run differences).  Marked `gpu`."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

GUARD = 1 << 16


class GuardAllocator:
    def __init__(self):
        self.live = {}
        self.bad = []

    def alloc(self, nbytes):
        pad = (-nbytes) % 256
        t = torch.empty(GUARD + nbytes + pad + GUARD, dtype=torch.uint8, device="cuda")
        t[:GUARD].fill_(0xA5)
        t[GUARD + nbytes:].fill_(0x5A)
        ptr = t.data_ptr() + GUARD
        self.live[ptr] = (t, nbytes)
        return ptr

    def check(self, ptr):
        t, nbytes = self.live[ptr]
        torch.cuda.synchronize()
        if not (bool((t[:GUARD] == 0xA5).all()) and bool((t[GUARD + nbytes:] == 0x5A).all())):
            self.bad.append((nbytes, int((t[:GUARD] != 0xA5).sum()), int((t[GUARD + nbytes:] != 0x5A).sum())))

    def free(self, ptr):
        self.check(ptr)
        del self.live[ptr]

    def check_all(self):
        for p in list(self.live):
            self.check(p)


@pytest.fixture(scope="module")
def cases():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import sanitize_cases
    return sanitize_cases


@pytest.mark.parametrize("case", ["c1", "finite16", "j2_16", "tma", "n512", "loopback"])
def test_guard_bands_intact(cases, case, monkeypatch):
    from paper_1905_12725_b200 import dbfft
    ga = GuardAllocator()
    orig = dbfft.DBFFT.__init__

    def guarded(self, *a, **kw):
        kw["allocator"] = (ga.alloc, ga.free)
        orig(self, *a, **kw)

    monkeypatch.setattr(dbfft.DBFFT, "__init__", guarded)
    cases.CASES[case]()
    import gc
    gc.collect()      # the case's contexts are closed: their buffers checked on free
    torch.cuda.synchronize()
    ga.check_all()
    assert not ga.bad, ga.bad


def test_bit_identical_repeats(cases):
    from paper_1905_12725_b200 import dbfft
    from synth import configs
    for n, kin, mats in (((16, 128, 256), "finite", cases.NH2), ((512, 8, 16), "small", cases.ISO2)):
        ctx = dbfft.DBFFT(n, kinematics=kin)
        ctx.set_phases(cases.two_phase(n, 81), mats)
        u = cases.spec(ctx, 82)
        ref = ctx.apply_K(u).clone()
        for _ in range(10):
            assert torch.equal(ctx.apply_K(u), ref)
    cfg = configs.c4(n=32, radius_vox=3)
    out = []
    for _ in range(2):
        ctx = dbfft.DBFFT(cfg["n"], kinematics="finite")
        ctx.set_phases(cfg["phase"], cfg["materials"])
        L = cfg["loads"][0]
        rep = ctx.solve_increment(L["target"], L["mask"])
        out.append((rep["cg_iters"], rep["macro_stress"].copy(), ctx.get_field(dbfft.FIELD_STRESS)))
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1]) and np.array_equal(out[0][2], out[1][2])
