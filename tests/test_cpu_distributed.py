"""Multi-process host logic on CPU (gloo, world_size 2): the NCCL unique-id bootstrap of the
binding, the bench's max-over-ranks / sum-over-ranks aggregation, and each rank's real-space block
of the global microstructure for z-slabs and 2-D pencils (include/dbfft.h: rank = b Py + a)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1905_12725_b200 import build, dbfft
        build.build()
        buf = dbfft.nccl_unique_id_broadcast(rank)
        import bench
        t, it = bench.aggregate_over_ranks(1.0 + rank, 10 * (rank + 1), device="cpu")
        import numpy as np
        g = np.arange(8 * 4 * 6).reshape(8, 4, 6)  # [z][y][x]
        blocks = {py: bench.rank_block(g, rank, world, py) for py in (1, 2)}
        allb = [None] * world
        dist.all_gather_object(allb, blocks)  # every rank sees every block
        q.put((rank, bytes(buf.raw), t, it, allb))
    finally:
        dist.destroy_process_group()


def test_gloo_bootstrap_and_aggregation():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == res[1][1] and len(res[0][1]) == 128 and any(res[0][1])
    for r in res:
        assert r[2] == 2.0 and r[3] == 30  # max time, summed iterations
    import numpy as np
    g = np.arange(8 * 4 * 6).reshape(8, 4, 6)
    allb = res[0][4]
    # z-slabs: rank r owns z in [4 r, 4 r + 4); pencils 2 x 1 (Pz = 1): rank a owns y in [2 a, 2 a + 2)
    assert np.array_equal(np.concatenate([allb[0][1], allb[1][1]], axis=0), g)
    assert np.array_equal(np.concatenate([allb[0][2], allb[1][2]], axis=1), g)
