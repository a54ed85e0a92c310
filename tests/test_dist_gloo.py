"""Data-parallel host logic at world_size 2 over gloo (CPU)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1901_07988_b200 import dist as D
    try:
        g = torch.arange(10, dtype=torch.float32) * (rank + 1)
        D.allreduce_mean_(g, bucket_elems=3)      # several buckets, reverse order
        want = torch.arange(10, dtype=torch.float32) * 1.5
        ok_mean = bool(torch.equal(g, want))
        w = torch.full((4,), float(rank))
        D.broadcast_(w, src=0)
        ok_bcast = bool(torch.all(w == 0))
        mx = D.max_over_ranks(float(rank) * 2.0)
        lo, hi = D.shard_range(8, rank, world)
        q.put((rank, ok_mean, ok_bcast, mx, lo, hi))
    finally:
        dist.destroy_process_group()


def test_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[0] == (0, True, True, 2.0, 0, 4)
    assert res[1] == (1, True, True, 2.0, 4, 8)


def test_shard_range_rejects_uneven():
    from paper_1901_07988_b200 import dist as D
    with pytest.raises(ValueError):
        D.shard_range(7, 0, 2)
