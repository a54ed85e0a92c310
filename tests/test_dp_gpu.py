"""The data-parallel Trainer path on one GPU: a one-rank NCCL process group
exercises the bucketed all-reduce inside the captured step (communication
stream, events from the weight-gradient side stream, join before SGD).  With
one rank the mean is the identity, so the captured DP step must reproduce the
single-GPU Trainer bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu

import paper_1901_07988_b200 as P  # noqa: E402
from paper_1901_07988_b200 import engine as E  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture
def nccl_world1():
    if dist.is_initialized():
        pytest.skip("a process group is already initialised")
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


def test_captured_dp_step_matches_single_gpu(nccl_world1, monkeypatch):
    monkeypatch.setenv("QTAPE_BUCKET_MB", "1")       # several buckets at C1 scale
    spec = E.resnet164_spec()
    rng = np.random.default_rng(0)
    x = rng.standard_normal((16, 3, 32, 32)).astype(np.float32)
    y = rng.integers(0, 10, 16)
    runs = []
    for group in (None, nccl_world1):
        tr = P.Trainer(spec, 16, mode="approx", bits=4, lr=0.1, seed=0, process_group=group)
        if group is not None:
            assert tr.buckets is not None and len(tr.buckets.buckets) >= 3
        tr.load_batch(x, y)
        tr.capture()
        losses = [tr.step(x, y) for _ in range(3)]
        runs.append((losses, tr.params.values.cpu().numpy().copy()))
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1])
