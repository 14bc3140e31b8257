"""Multi-process host logic on CPU (gloo, world_size 2): the NCCL unique-id bootstrap of the
binding and the bench's max-over-ranks / sum-over-ranks aggregation."""
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
        q.put((rank, bytes(buf.raw), t, it))
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
