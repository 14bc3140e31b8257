"""Host bootstrap of the peer transport (peer.cu, include/dbfft.h dbfft_fd_allgather): file
descriptors all-gathered among processes over abstract Unix sockets with SCM_RIGHTS.  CPU only:
memfd descriptors stand in for the exported CUDA VMM handles."""
import ctypes
import multiprocessing as mp
import os

import pytest


def _worker(rank, world, tag, q):
    try:
        from paper_1905_12725_b200 import dbfft
        lib = dbfft.load_library()
        fds = []
        for i in range(2):
            fd = os.memfd_create(f"r{rank}f{i}")
            os.write(fd, f"rank {rank} fd {i}".encode())
            fds.append(fd)
        out = (ctypes.c_int32 * (2 * world))()
        st = lib.dbfft_fd_allgather(tag.encode(), rank, world, (ctypes.c_int32 * 2)(*fds), 2, out, 20000)
        if st != 0:
            q.put((rank, "status %d: %s" % (st, lib.dbfft_last_error(None).decode())))
            return
        got = {}
        for src in range(world):
            for i in range(2):
                got[(src, i)] = os.pread(out[src * 2 + i], 64, 0).decode()
        q.put((rank, got))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, repr(exc)))


@pytest.mark.parametrize("world", [2, 4])
def test_fd_allgather(world):
    if not hasattr(os, "memfd_create"):
        pytest.skip("no memfd_create")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    tag = f"test-{os.getpid()}-{world}"
    procs = [ctx.Process(target=_worker, args=(r, world, tag, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert isinstance(res[r], dict), res[r]
        for src in range(world):
            for i in range(2):
                assert res[r][(src, i)] == f"rank {src} fd {i}"


def test_fd_allgather_bad_args():
    from paper_1905_12725_b200 import dbfft
    lib = dbfft.load_library()
    out = (ctypes.c_int32 * 4)()
    fds = (ctypes.c_int32 * 1)(0)
    assert lib.dbfft_fd_allgather(b"x", 2, 2, fds, 1, out, 100) == 2   # rank >= world
    assert lib.dbfft_fd_allgather(b"x", 0, 2, fds, 0, out, 100) == 2   # nfd < 1
    # world 1: identity, no sockets
    assert lib.dbfft_fd_allgather(b"x", 0, 1, fds, 1, out, 100) == 0 and out[0] == 0
    # a peer that never shows up: timeout, not a hang
    assert lib.dbfft_fd_allgather(f"lonely-{os.getpid()}".encode(), 0, 2, fds, 1, out, 300) == 3
