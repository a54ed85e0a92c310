"""Batch-sharded data parallelism.

One process per GPU; each rank runs the whole engine on its N/G shard with
its own BufferPool and tape arena (tapes never leave the device, stored
bytes per sample are unchanged).  The only exchange is the mean all-reduce
of the flat gradient slab between network_backward and sgd_step
(training.py:196-199): NCCL over NVLink/NVSwitch on the box, gloo on CPU for
the multi-process tests.  BN statistics stay per rank (standard DP).

``GradBuckets`` overlaps that all-reduce with the backward pass: the weight
region of the slab is cut into per-layer-range buckets in reverse layer
order; a bucket is issued on a communication stream as soon as the weight
gradient of its lowest layer has been queued (an event on the stream the
weight gradients run on), the gamma/beta region follows the last BN
backward, and the main stream joins the communication stream before SGD.
The whole sequence is captured into the step's CUDA graph.
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


def plan_buckets(layer_spans, bucket_bytes: int, itemsize: int = 4):
    """Cut the weight region into buckets of whole layers, in reverse layer
    order (the order backward finalises weight gradients).

    ``layer_spans``: [(layer, start, stop)] element ranges of each layer's
    weight gradient in the flat slab, ascending and contiguous.  Returns
    [(trigger_layer, start, stop)] in issue order: a bucket covers layers
    trigger_layer..(previous trigger - 1) and is ready once the weight
    gradient of ``trigger_layer`` (its lowest layer) has been produced.
    Every element of the region is covered exactly once."""
    spans = sorted(layer_spans)
    for (_, _, b), (_, a, _) in zip(spans, spans[1:]):
        if a != b:
            raise ValueError("layer weight spans must be contiguous")
    out = []
    stop = None
    acc = 0
    for layer, a, b in reversed(spans):
        if stop is None:
            stop = b
        acc += (b - a) * itemsize
        if acc >= bucket_bytes:
            out.append((layer, a, stop))
            stop, acc = None, 0
    if stop is not None:
        out.append((spans[0][0], spans[0][1], stop))
    return out


def default_bucket_bytes(total_bytes: int) -> int:
    """About 8 buckets per step, each 2..32 MiB (QTAPE_BUCKET_MB overrides):
    small enough that the first ones overlap the backward pass, large enough
    that NCCL's per-call latency stays small next to the transfer."""
    env = os.environ.get("QTAPE_BUCKET_MB")
    if env:
        return max(1, int(float(env) * (1 << 20)))
    return int(min(32 << 20, max(2 << 20, total_bytes // 8)))


class GradBuckets:
    """Bucketed, backward-overlapped mean all-reduce of a ParamList's flat
    gradient slab (see the module docstring).

    ``layer_done(i, stream)`` is called by network_backward after layer i's
    backward has been queued, with the stream its weight gradient runs on;
    ``finish()`` issues the gamma/beta bucket and joins.  On CPU tensors
    (gloo tests) the buckets are reduced synchronously in the same order."""

    def __init__(self, params, group=None, bucket_bytes=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.flat = params.grads.view(-1)
        base = params.grads.data_ptr()
        spans = []
        for i, p in enumerate(params):
            a = (p.grad_weight.data_ptr() - base) // 4
            spans.append((i, a, a + p.grad_weight.numel()))
        self.n_weight = params.n_weight
        bb = bucket_bytes if bucket_bytes is not None else default_bucket_bytes(4 * self.n_weight)
        self.buckets = plan_buckets(spans, bb)
        self.tail = (self.n_weight, self.flat.numel())       # gamma / beta region
        self.trigger = {b[0]: b for b in self.buckets}
        self.cuda = self.flat.is_cuda
        self.comm = torch.cuda.Stream(device=self.flat.device) if self.cuda else None
        self.nccl = dist.get_backend(group) == "nccl"
        self.issued = []                                        # (start, stop) in issue order

    def reset(self):
        self.issued = []

    def _reduce(self, start, stop):
        chunk = self.flat[start:stop]
        if self.nccl:
            dist.all_reduce(chunk, op=dist.ReduceOp.AVG, group=self.group)
        else:
            dist.all_reduce(chunk, op=dist.ReduceOp.SUM, group=self.group)
            chunk.div_(self.world)
        self.issued.append((start, stop))

    def _issue(self, start, stop, producer=None):
        if stop <= start:
            return
        if not self.cuda:
            self._reduce(start, stop)
            return
        ev = torch.cuda.Event()
        ev.record(producer if producer is not None else torch.cuda.current_stream())
        self.comm.wait_event(ev)
        with torch.cuda.stream(self.comm):
            self._reduce(start, stop)

    def layer_done(self, i, producer=None):
        b = self.trigger.get(i)
        if b is not None:
            self._issue(b[1], b[2], producer)

    def finish(self):
        """gamma/beta bucket after the last BN backward (current stream),
        then the current stream waits for every bucket."""
        self._issue(self.tail[0], self.tail[1], None)
        if self.cuda:
            torch.cuda.current_stream().wait_stream(self.comm)


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
