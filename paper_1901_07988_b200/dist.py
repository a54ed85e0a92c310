"""Batch-sharded data parallelism.

One process per GPU; each rank runs the whole engine on its N/G shard with
its own BufferPool and tape arena (tapes never leave the device, stored
bytes per sample are unchanged).  The only exchange is the mean all-reduce
of the flat gradient slab between network_backward and sgd_step
(training.py:196-199): NCCL over NVLink/NVSwitch on the box, gloo on CPU for
the multi-process tests.  BN statistics stay per rank (standard DP).
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def init_from_env(backend: str = "nccl"):
    """Initialise the default group from torchrun's env (RANK, WORLD_SIZE,
    LOCAL_RANK, MASTER_ADDR=127.0.0.1); returns (rank, world, local_rank)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29500")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def allreduce_mean_(t: torch.Tensor, group=None, bucket_elems: int = 1 << 26) -> torch.Tensor:
    """In-place mean over ranks, in contiguous buckets (reverse order, so the
    last layers' gradients -- final first in backward -- go first)."""
    world = dist.get_world_size(group)
    if world == 1:
        return t
    flat = t.view(-1)
    n = flat.numel()
    nccl = dist.get_backend(group) == "nccl"
    starts = list(range(0, n, bucket_elems))
    for s in reversed(starts):
        chunk = flat[s:s + bucket_elems]
        if nccl:
            dist.all_reduce(chunk, op=dist.ReduceOp.AVG, group=group)
        else:
            dist.all_reduce(chunk, op=dist.ReduceOp.SUM, group=group)
            chunk.div_(world)
    return t


def broadcast_(t: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """Make every rank start from rank ``src``'s parameters."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(t, src=src, group=group)
    return t


def shard_range(global_batch: int, rank: int, world: int):
    """[start, stop) of this rank's shard; the global batch must divide evenly
    (every rank runs the same captured graph shape)."""
    if global_batch % world:
        raise ValueError(f"global batch {global_batch} not divisible by world size {world}")
    per = global_batch // world
    return rank * per, (rank + 1) * per


def max_over_ranks(value: float, group=None, device=None) -> float:
    """Max of a per-rank scalar (timing is reported as the slowest rank)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
