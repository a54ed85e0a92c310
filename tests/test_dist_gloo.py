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


class _FakeLayer:
    def __init__(self, gw):
        self.grad_weight = gw


class _FakeParams(list):
    """Flat-slab layout of training.ParamList on CPU tensors:
    [layer weights in layer order | gamma, beta region]."""

    def __init__(self, sizes, tail, fill):
        total = sum(sizes) + tail
        self.grads = fill(total)
        self.n_weight = sum(sizes)
        off = 0
        items = []
        for n in sizes:
            items.append(_FakeLayer(self.grads[off:off + n]))
            off += n
        super().__init__(items)


def _bucket_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1901_07988_b200 import dist as D
    try:
        sizes = [27, 5, 300, 64, 7, 1000, 3, 128]
        tail = 40
        fill = lambda n: torch.arange(n, dtype=torch.float32) * (rank + 1) + 0.25 * rank  # noqa: E731
        params = _FakeParams(sizes, tail, fill)
        gb = D.GradBuckets(params, bucket_bytes=4 * 200)
        # network_backward order: the head first, the stem last
        for i in range(len(sizes) - 1, -1, -1):
            gb.layer_done(i)
        gb.finish()
        total = sum(sizes) + tail
        want = torch.arange(total, dtype=torch.float32) * 1.5 + 0.125
        ok_mean = bool(torch.allclose(params.grads, want, rtol=0, atol=1e-6))
        q.put((rank, ok_mean, gb.issued, [b[0] for b in gb.buckets]))
    finally:
        dist.destroy_process_group()


def test_grad_buckets_gloo_world2():
    """The Trainer's bucketed all-reduce (dist.GradBuckets) at world 2:
    issued in reverse layer order as network_backward finishes each
    layer's weight gradient, every element reduced exactly once, and the
    result is the mean of the two ranks' gradients."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bucket_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, ok, issued, triggers in res:
        assert ok, rank
        # weight buckets cover [0, n_weight) from the top down, then the tail
        assert issued[-1] == (1534, 1574)
        w = issued[:-1]
        assert w[0][1] == 1534 and w[-1][0] == 0
        assert all(a[0] == b[1] for a, b in zip(w, w[1:]))
        assert len(w) >= 3 and triggers == sorted(triggers, reverse=True)
    assert res[0][2] == res[1][2]          # same collective sequence on both ranks


def test_plan_buckets_cover_reverse_order():
    from paper_1901_07988_b200 import dist as D
    spans, off = [], 0
    for i, n in enumerate([10, 1, 50, 50, 3, 200, 7]):
        spans.append((i, off, off + n))
        off += n
    for bb in (4, 40, 200, 4000):
        b = D.plan_buckets(spans, bb)
        assert b[0][2] == off and b[-1][1] == 0 and b[-1][0] == 0
        assert all(x[1] == y[2] for x, y in zip(b, b[1:]))
        # each bucket starts at its trigger layer's first element
        assert all(x[1] == spans[x[0]][1] for x in b)
    assert len(D.plan_buckets(spans, 4)) == len(spans)
    assert len(D.plan_buckets(spans, 4000)) == 1
    with pytest.raises(ValueError):
        D.plan_buckets([(0, 0, 5), (1, 6, 9)], 4)


def test_default_bucket_bytes(monkeypatch):
    from paper_1901_07988_b200 import dist as D
    monkeypatch.delenv("QTAPE_BUCKET_MB", raising=False)
    assert D.default_bucket_bytes(6 << 20) == 2 << 20
    assert D.default_bucket_bytes(212 << 20) == (212 << 20) // 8
    assert D.default_bucket_bytes(4 << 30) == 32 << 20
    monkeypatch.setenv("QTAPE_BUCKET_MB", "5")
    assert D.default_bucket_bytes(1) == 5 << 20


def test_shard_range_rejects_uneven():
    from paper_1901_07988_b200 import dist as D
    with pytest.raises(ValueError):
        D.shard_range(7, 0, 2)
