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


def _send(tag, dst, src, fds):
    import socket
    import struct
    import time
    deadline = time.time() + 30
    while True:
        s = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        try:
            s.connect(f"\0dbfft-{tag}-{dst}")
            break
        except OSError:
            s.close()
            if time.time() > deadline:
                raise
            time.sleep(0.01)
    socket.send_fds(s, [struct.pack("<i", src)], fds)
    s.close()


def test_fd_allgather_ignores_bad_peers():
    """Malformed messages (unknown rank, wrong descriptor count, no descriptors) are dropped and
    their descriptors closed; the real peer's descriptors still arrive (peer.cu fd_allgather)."""
    import socket
    if not hasattr(os, "memfd_create") or not hasattr(socket, "send_fds"):
        pytest.skip("no memfd_create / send_fds")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    tag = f"bad-{os.getpid()}"
    ls = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)   # this process plays rank 1
    ls.bind(f"\0dbfft-{tag}-1")
    ls.listen(4)
    p = ctx.Process(target=_worker, args=(0, 2, tag, q))
    p.start()
    mine = []
    for i in range(2):
        fd = os.memfd_create(f"r1f{i}")
        os.write(fd, f"rank 1 fd {i}".encode())
        mine.append(fd)
    junk = os.memfd_create("junk")
    _send(tag, 0, 7, [junk, junk])       # rank out of range
    _send(tag, 0, 1, [junk])             # wrong descriptor count
    _send(tag, 0, 0, [junk, junk])       # claims to be the receiver itself
    _send(tag, 0, 1, mine)               # the real message
    a, _ = ls.accept()
    msg, fds, _, _ = socket.recv_fds(a, 4, 4)
    a.close()
    ls.close()
    res = q.get(timeout=60)
    p.join(timeout=30)
    assert res[0] == 0 and isinstance(res[1], dict), res
    assert res[1][(1, 0)] == "rank 1 fd 0" and res[1][(1, 1)] == "rank 1 fd 1"
    assert len(fds) == 2 and os.pread(fds[0], 64, 0).decode() == "rank 0 fd 0"
    for fd in fds + mine + [junk]:
        os.close(fd)
