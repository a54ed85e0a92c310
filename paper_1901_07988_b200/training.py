"""Initialisation, momentum SGD, loss, training loop and the captured step.

Drop-in for /root/reference/pkg/src/qtape/training.py (TrainConfig,
init_params, lr_at, sgd_step, softmax_xent, train, evaluate), on device.

``Trainer`` is the B200 execution path of one training iteration
(training.py:192-199): network_forward -> softmax_xent -> network_backward
-> [NCCL gradient all-reduce] -> sgd_step, with every buffer preallocated
(BufferPool slots, one packed-code TapeArena, flat parameter/grad/velocity
slabs) and the whole step captured in ONE CUDA graph, so a 164-1001 layer
network replays thousands of kernels with a single launch.
"""

from __future__ import annotations

import os
import time
from bisect import bisect_right
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

import torch

from . import _native as N
from .engine import (BufferPool, NetworkSpec, TapeArena, Workspace, network_backward,
                     network_forward)
from .errors import ConfigError, DataError
from .layer import LayerParams

CIFAR_LR_SCHEDULE = [(0, 1e-2), (400, 1e-1), (32000, 1e-2), (48000, 1e-3)]


@dataclass
class TrainConfig:
    """Run configuration (training.py:21-61); JSON-compatible."""

    mode: str = "exact"
    bits: Optional[int] = 8
    batch_size: int = 128
    total_iters: int = 64000
    momentum: float = 0.9
    weight_decay: float = 2e-4
    lr_schedule: list = field(default_factory=lambda: list(CIFAR_LR_SCHEDULE))
    seed: int = 0
    hflip: bool = True
    translate: bool = True
    log_path: Optional[str] = None

    def __post_init__(self):
        if self.batch_size < 1:
            raise ConfigError("batch_size must be >= 1")
        self.lr_schedule = [(int(s), float(lr)) for s, lr in self.lr_schedule]
        starts = [s for s, _ in self.lr_schedule]
        if not starts or starts[0] != 0 or starts != sorted(set(starts)):
            raise ConfigError("lr_schedule needs strictly increasing starts from 0")

    _KEYS = ("mode", "bits", "batch_size", "total_iters", "momentum", "weight_decay",
             "lr_schedule", "seed", "hflip", "translate", "log_path")

    def to_json(self) -> dict:
        d = {k: getattr(self, k) for k in self._KEYS}
        d["lr_schedule"] = [list(p) for p in self.lr_schedule]
        return d

    @classmethod
    def from_json(cls, d: dict) -> "TrainConfig":
        return cls(**{k: d[k] for k in cls._KEYS if k in d})


class ParamList(list):
    """List of LayerParams whose tensors are views into three flat device
    slabs (values / grads / velocities): [all weights | all gamma,beta].
    sgd_step then runs two launches for the whole network and the gradient
    all-reduce is one contiguous buffer."""

    def __init__(self, items, values, grads, vels, n_weight):
        super().__init__(items)
        self.values, self.grads, self.vels = values, grads, vels
        self.n_weight = n_weight


def init_params(spec: NetworkSpec, seed: int, dtype=torch.float32, device=None) -> ParamList:
    """He init, gamma=1, beta=0 (training.py:64-89).  The draws come from
    the same numpy Generator sequence as the reference, so parameters are
    bit-identical; they are then uploaded once into flat device slabs."""
    if dtype not in (torch.float32, np.float32, "float32"):
        raise ConfigError("device parameters are float32")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    rng = np.random.default_rng(seed)
    host_w, host_c = [], []
    for l, (ins, _) in zip(spec.layers, spec.layer_shapes(1)):
        cin = ins[1]
        if l.kind == "conv":
            fan = cin * l.kernel * l.kernel
            w = rng.standard_normal((l.out_channels, cin, l.kernel, l.kernel))
        else:
            fan = cin
            w = rng.standard_normal((cin, l.out_channels))
        host_w.append((w * np.sqrt(2.0 / fan)).astype(np.float32))
        host_c.append(cin if l.preact else 0)
    n_w = sum(w.size for w in host_w)
    n_c = sum(2 * c for c in host_c)
    values = torch.empty(n_w + n_c, dtype=torch.float32, device=dev)
    flat = np.concatenate([w.ravel() for w in host_w] +
                          [np.concatenate([np.ones(c, np.float32), np.zeros(c, np.float32)])
                           for c in host_c if c] + [np.zeros(0, np.float32)])
    values.copy_(torch.from_numpy(flat))
    grads = torch.zeros_like(values)
    vels = torch.zeros_like(values)
    items = []
    ow, oc = 0, n_w
    for l, w, c in zip(spec.layers, host_w, host_c):
        def view(buf, off, shape):
            return buf[off:off + int(np.prod(shape))].view(shape)
        kw = dict(kind=l.kind, weight=view(values, ow, w.shape), stride=l.stride, pad=l.pad,
                  grad_weight=view(grads, ow, w.shape), vel_weight=view(vels, ow, w.shape))
        ow += w.size
        if l.preact:
            kw.update(gamma=view(values, oc, (c,)), beta=view(values, oc + c, (c,)),
                      grad_gamma=view(grads, oc, (c,)), grad_beta=view(grads, oc + c, (c,)),
                      vel_gamma=view(vels, oc, (c,)), vel_beta=view(vels, oc + c, (c,)))
            oc += 2 * c
        items.append(LayerParams(**kw))
    return ParamList(items, values, grads, vels, n_w)


def params_to_host(params) -> list:
    """Numpy copies of every parameter (tests / checkpoints)."""
    out = []
    for p in params:
        d = {"weight": p.weight.detach().cpu().numpy()}
        if p.preact:
            d["gamma"] = p.gamma.detach().cpu().numpy()
            d["beta"] = p.beta.detach().cpu().numpy()
        out.append(d)
    return out


def lr_at(config: TrainConfig, iteration: int) -> float:
    """Piecewise-constant schedule (training.py:92-95)."""
    starts = [s for s, _ in config.lr_schedule]
    return config.lr_schedule[bisect_right(starts, iteration) - 1][1]


def sgd_step(params, lr: float, momentum: float, weight_decay: float, lr_dev=None) -> None:
    """v = m v + (g + wd w); w -= lr v; zero grads -- weight decay on linear
    weights only (training.py:98-117).  Flat-slab params: 2 launches."""
    if isinstance(params, ParamList):
        nw = params.n_weight
        total = params.values.numel()
        V, G, Vel = params.values, params.grads, params.vels
        N.call("qt_sgd", N.ptr(V), N.ptr(G), N.ptr(Vel), nw, float(lr), N.ptr(lr_dev),
               float(momentum), float(weight_decay))
        if total > nw:
            N.call("qt_sgd", N.ptr(V[nw:]), N.ptr(G[nw:]), N.ptr(Vel[nw:]), total - nw, float(lr),
                   N.ptr(lr_dev), float(momentum), 0.0)
        return
    for p in params:
        slots = [(p.weight, p.grad_weight, p.vel_weight, weight_decay)]
        if p.preact:
            slots += [(p.gamma, p.grad_gamma, p.vel_gamma, 0.0),
                      (p.beta, p.grad_beta, p.vel_beta, 0.0)]
        for v, g, m, wd in slots:
            N.call("qt_sgd", N.ptr(v), N.ptr(g), N.ptr(m), v.numel(), float(lr), N.ptr(lr_dev),
                   float(momentum), float(wd))


def softmax_xent(logits: torch.Tensor, labels, loss_buf=None, grad_out=None, check=True):
    """Mean cross-entropy with max-subtraction (training.py:120-134).

    Returns (loss, grad).  With ``check`` (default) the loss is a Python
    float and out-of-range labels raise DataError (both synchronise); the
    captured step passes ``check=False`` and gets the device loss slot."""
    n, c = logits.shape
    dev = logits.device
    if not isinstance(labels, torch.Tensor):
        labels = torch.as_tensor(np.asarray(labels), dtype=torch.int64)
    if labels.device != dev or labels.dtype != torch.int64:
        labels = labels.to(device=dev, dtype=torch.int64)
    if loss_buf is None:
        loss_buf = torch.empty(1 + n, dtype=torch.float64, device=dev)
    grad = grad_out if grad_out is not None else torch.empty((n, c), dtype=torch.float32,
                                                             device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev) if check else None
    N.call("qt_softmax_xent", N.ptr(logits.contiguous()), N.ptr(labels.contiguous()), n, c,
           N.ptr(loss_buf), N.ptr(grad), N.ptr(bad))
    if check:
        if int(bad.item()):
            raise DataError(f"labels must lie in [0, {c})")
        return float(loss_buf[0].item()), grad
    return loss_buf[:1], grad


def _dp_overlap() -> bool:
    """Bucketed all-reduce overlapped with backward inside the captured step
    (default); QTAPE_DP_OVERLAP=0 falls back to one all-reduce of the whole
    slab between two graph replays."""
    return os.environ.get("QTAPE_DP_OVERLAP", "1") not in ("", "0")


def _capture_priority() -> int:
    """Stream priority of the captured step (QTAPE_CAPTURE_PRIORITY, default 0
    = the default priority; torch clamps to the device's range)."""
    return int(os.environ.get("QTAPE_CAPTURE_PRIORITY", "0"))


class Trainer:
    """Preallocated, CUDA-graph-captured training iteration.

    ``step(images, labels)`` is the public end-to-end call: host batch ->
    pinned staging -> H2D copy -> graph replay (forward, xent, backward,
    all-reduce, SGD) -> D2H loss.  ``step_device()`` replays with the inputs
    already resident (the throughput number)."""

    def __init__(self, spec: NetworkSpec, batch_size: int, mode: str = "approx", bits=4,
                 lr: float = 0.1, momentum: float = 0.9, weight_decay: float = 2e-4,
                 seed: int = 0, params: Optional[ParamList] = None, device=None,
                 use_graph: bool = True, process_group=None):
        self.spec = spec
        self.n = int(batch_size)
        self.mode, self.bits = mode, bits
        self.momentum, self.weight_decay = float(momentum), float(weight_decay)
        self.device = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        self.params = params if params is not None else init_params(spec, seed, device=self.device)
        self.group = process_group
        shapes = spec.layer_shapes(self.n)
        self.pool = BufferPool(spec.width() + 1, device=self.device)
        self.pool.reserve(max(max(_numel(i), _numel(o)) for i, o in shapes))
        self.arena = TapeArena(spec, self.n, mode, bits, self.device)
        self.pool.cache[("ws", id(spec), self.n)] = Workspace(spec, self.n, self.device)
        self.x = torch.empty((self.n,) + tuple(spec.input_shape), dtype=torch.float32,
                             device=self.device)
        self.labels = torch.zeros(self.n, dtype=torch.int64, device=self.device)
        self.loss_buf = torch.zeros(1 + self.n, dtype=torch.float64, device=self.device)
        self.lr = torch.full((1,), float(lr), dtype=torch.float32, device=self.device)
        self.x_host = torch.empty(self.x.shape, dtype=torch.float32, pin_memory=True)
        self.labels_host = torch.empty(self.n, dtype=torch.int64, pin_memory=True)
        self.loss_host = torch.empty(1, dtype=torch.float64, pin_memory=True)
        self.num_classes = spec.num_classes
        self.graph = None
        self.use_graph = use_graph
        self.tapes = None
        self._build_weight_prep()
        self.buckets = None
        if process_group is not None and _dp_overlap():
            from .dist import GradBuckets
            self.buckets = GradBuckets(self.params, process_group)

    # one iteration of training.py:192-199 on the static buffers, in two
    # parts so the (optional) gradient all-reduce sits between them
    def _build_weight_prep(self):
        """Tensor-core conv layers get persistent prepared weight operands,
        refreshed by ONE qt_conv_prepare_weights launch at the start of every
        step (instead of one re-layout per conv call).  They live in this
        Trainer's workspace (``Workspace.prep``), never on the shared
        LayerParams, so an eager forward on ``self.params`` after a step
        lays out the current weights itself."""
        descs = []
        self._prep_max = 0
        prep = self.pool.cache[("ws", id(self.spec), self.n)].prep
        prep.clear()
        for li, (p, (ins, _)) in enumerate(zip(self.params, self.spec.layer_shapes(self.n))):
            if p.kind != "conv":
                continue
            n, ci, h, w = ins
            co, _, kh, kw = p.weight.shape
            elems = co * ci * kh * kw
            ent = [None, None]
            for dgrad in (0, 1):
                if not N.query("qt_conv_uses_tc", n, ci, h, w, co, kh, kw, p.stride, p.pad, dgrad):
                    continue
                if dgrad and li == 0:
                    continue          # the stem needs no input gradient
                buf = torch.empty(2 * elems, dtype=torch.float32, device=self.device)
                rows, cols = (ci, co) if dgrad else (co, ci)
                descs.append((p.weight.data_ptr(), buf.data_ptr(), rows, cols, kh, kw, dgrad, 0))
                ent[dgrad] = buf
                self._prep_max = max(self._prep_max, elems)
            if ent[0] is not None or ent[1] is not None:
                prep[id(p)] = ent
        dt = np.dtype([("w", "<u8"), ("out", "<u8"), ("rows", "<i4"), ("cols", "<i4"),
                       ("kh", "<i4"), ("kw", "<i4"), ("flip", "<i4"), ("pad", "<i4")])
        arr = np.array(descs, dtype=dt)
        self._prep_descs = torch.from_numpy(arr.view(np.uint8).copy()).to(self.device)
        self._prep_count = len(descs)

    def _prepare_weights(self):
        if self._prep_count:
            N.call("qt_conv_prepare_weights", N.ptr(self._prep_descs), self._prep_count,
                   self._prep_max)

    def _fwd_bwd(self):
        self._prepare_weights()
        logits, tapes = network_forward(self.spec, self.params, self.x, mode=self.mode,
                                        bits=self.bits, pool=self.pool, arena=self.arena)
        _, g = softmax_xent(logits, self.labels, loss_buf=self.loss_buf, check=False)
        hook = None
        if self.buckets is not None:
            self.buckets.reset()
            hook = self.buckets.layer_done
        network_backward(self.spec, self.params, tapes, g, self.x, mode=self.mode, pool=self.pool,
                         grad_ready=hook)
        self.tapes = tapes

    def _update(self):
        sgd_step(self.params, 0.0, self.momentum, self.weight_decay, lr_dev=self.lr)

    def _allreduce(self):
        if self.group is None:
            return
        if self.buckets is not None:      # buckets already issued during backward
            self.buckets.finish()
        else:
            from .dist import allreduce_mean_
            allreduce_mean_(self.params.grads, self.group)

    def _body(self):
        self._fwd_bwd()
        self._allreduce()
        self._update()

    def _state(self):
        rs = [t for p in self.params if p.preact for t in (p.running_mean, p.running_var)]
        return [self.params.values, self.params.vels] + rs

    def capture(self, warmup: int = 2):
        """Warm up eagerly on a side stream, then capture the step (one CUDA
        graph; two around an all-reduce when data-parallel).  The model
        state is restored afterwards, so capture has no visible effect."""
        snapshot = [t.clone() for t in self._state()]
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self._body()
        torch.cuda.current_stream(self.device).wait_stream(s)
        if self.use_graph:
            # capture stream priority (QTAPE_CAPTURE_PRIORITY): equal to the
            # side stream's by default -- measured, giving either the
            # input-gradient chain or the side-stream weight gradients the
            # higher priority costs 0.3 ms/step at C2
            cap = torch.cuda.Stream(device=self.device, priority=_capture_priority())
            if self.group is None or self.buckets is not None:
                # one graph: forward, backward with the bucketed all-reduce
                # on the communication stream, join, SGD
                self.graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(self.graph, stream=cap):
                    self._body()
            else:
                self.graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(self.graph, stream=cap):
                    self._fwd_bwd()
                self.graph_update = torch.cuda.CUDAGraph()
                with torch.cuda.graph(self.graph_update, stream=cap):
                    self._update()
        for t, v in zip(self._state(), snapshot):
            t.copy_(v)
        self.params.grads.zero_()
        torch.cuda.synchronize(self.device)

    def set_lr(self, lr: float):
        self.lr.fill_(float(lr))

    def step_device(self):
        """Replay one step on the resident inputs (no host traffic)."""
        if self.graph is None:
            self._body()
        elif self.group is None or self.buckets is not None:
            self.graph.replay()
        else:
            self.graph.replay()
            self._allreduce()
            self.graph_update.replay()

    def load_batch(self, images, labels):
        """Host -> device (non-blocking): straight from the caller's tensors
        when they are already pinned, contiguous and of the step's dtype and
        size, else through the Trainer's pinned staging buffers."""
        if isinstance(images, np.ndarray):
            images = torch.from_numpy(np.ascontiguousarray(images, dtype=np.float32))
        if isinstance(labels, np.ndarray):
            labels = torch.from_numpy(np.ascontiguousarray(labels, dtype=np.int64))
        lab = labels.reshape(-1)
        if int(lab.min()) < 0 or int(lab.max()) >= self.num_classes:
            raise DataError(f"labels must lie in [0, {self.num_classes})")

        def direct(t, like):
            return (t.device.type == "cpu" and t.is_pinned() and t.is_contiguous()
                    and t.dtype == like.dtype and t.numel() == like.numel())

        if direct(images, self.x):
            self.x.copy_(images.reshape(self.x.shape), non_blocking=True)
        else:
            self.x_host.copy_(images)
            self.x.copy_(self.x_host, non_blocking=True)
        if direct(lab, self.labels):
            self.labels.copy_(lab.reshape(self.labels.shape), non_blocking=True)
        else:
            self.labels_host.copy_(lab)
            self.labels.copy_(self.labels_host, non_blocking=True)

    def step(self, images, labels) -> float:
        """End-to-end iteration through the public API; returns the loss."""
        self.load_batch(images, labels)
        return self.step_loaded()

    def step_loaded(self) -> float:
        """One iteration on the batch already in ``self.x`` / ``self.labels``
        (the device input pipeline writes them); returns the loss."""
        self.step_device()
        self.loss_host.copy_(self.loss_buf[:1], non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return float(self.loss_host[0])

    @property
    def h2d_bytes(self) -> int:
        return self.x.numel() * 4 + self.labels.numel() * 8

    @property
    def d2h_bytes(self) -> int:
        return 8


def _numel(shape) -> int:
    r = 1
    for s in shape:
        r *= int(s)
    return r


@dataclass
class TrainResult:
    records: list
    params: list
    pool: BufferPool

    def losses(self) -> np.ndarray:
        return np.array([r[1] for r in self.records])


def iterate_indices(n: int, batch_size: int, total_iters: int, seed: int):
    """(iteration, epoch, sample indices): seeded epoch permutations, the
    partial last batch dropped -- the reference's batch order
    (training.py:147-166) as indices, so a device-resident dataset is
    gathered on the GPU."""
    per_epoch = n // batch_size
    if per_epoch == 0:
        raise ConfigError("batch_size larger than dataset")
    rng = np.random.default_rng(seed)
    it = epoch = 0
    while it < total_iters:
        order = rng.permutation(n)
        for b in range(per_epoch):
            if it >= total_iters:
                return
            yield it, epoch, order[b * batch_size:(b + 1) * batch_size]
            it += 1
        epoch += 1


def iterate_batches(dataset, batch_size: int, total_iters: int, seed: int):
    """(iteration, epoch, images, labels) in the reference's order
    (training.py:147-166); images are host copies (or device gathers for a
    device-resident dataset)."""
    for it, epoch, idx in iterate_indices(len(dataset.labels), batch_size, total_iters, seed):
        if isinstance(dataset.images, torch.Tensor):
            from .data import gather_batch
            images = gather_batch(dataset.images, idx)
        else:
            images = dataset.images[idx].copy()
        yield it, epoch, images, dataset.labels[idx]


def write_log(path: str, records: list) -> None:
    """CSV training log (training.py:206-212)."""
    with open(path, "w") as f:
        f.write("iter,loss,lr,elapsed_ms\n")
        for it, loss, lr, ms in records:
            f.write(f"{it},{loss:.17g},{lr:.17g},{ms:.3f}\n")


def train(spec: NetworkSpec, config: TrainConfig, dataset, params=None) -> TrainResult:
    """Training loop with the reference's seeding, augmentation and CSV log
    (training.py:169-212) on the captured Trainer step.

    Every batch is gathered and augmented on the device straight into the
    step's input buffer (qt_gather_augment): a device-resident dataset
    (data.load_cifar10) never leaves HBM; a host dataset is uploaded per
    batch.  The flips / crop offsets come from the per-batch generator
    keyed by (seed, epoch, iteration) with the reference's draws, so runs
    augment exactly as the reference does."""
    from .data import gather_batch
    if params is None:
        params = init_params(spec, config.seed)
    tr = Trainer(spec, config.batch_size, mode=config.mode, bits=config.bits,
                 lr=lr_at(config, 0), momentum=config.momentum,
                 weight_decay=config.weight_decay, params=params)
    tr.capture()
    records = []
    t0 = time.perf_counter()
    augment = (config.hflip or config.translate) and len(tr.x.shape) == 4
    dev_images = isinstance(dataset.images, torch.Tensor)
    staging = None
    for it, epoch, idx in iterate_indices(len(dataset.labels), config.batch_size,
                                          config.total_iters, config.seed):
        rng = (np.random.default_rng(np.random.SeedSequence((config.seed, epoch, it)))
               if augment else None)
        if dev_images:
            src, gidx = dataset.images, idx
        else:                          # host dataset: upload the batch, augment on the device
            if staging is None:
                staging = torch.empty_like(tr.x)
            tr.x_host.copy_(torch.from_numpy(np.ascontiguousarray(dataset.images[idx],
                                                                   dtype=np.float32)))
            staging.copy_(tr.x_host, non_blocking=True)
            src, gidx = staging, None
        if augment or dev_images:
            gather_batch(src, gidx, rng, config.hflip, config.translate, out=tr.x,
                         n=config.batch_size)
        else:
            tr.x.copy_(src)
        tr.labels_host.copy_(torch.from_numpy(np.asarray(dataset.labels[idx], dtype=np.int64)))
        tr.labels.copy_(tr.labels_host, non_blocking=True)
        lr = lr_at(config, it)
        tr.set_lr(lr)
        loss = tr.step_loaded()
        records.append((it, loss, lr, (time.perf_counter() - t0) * 1e3))
    if config.log_path:
        write_log(config.log_path, records)
    return TrainResult(records=records, params=tr.params, pool=tr.pool)


def evaluate(spec: NetworkSpec, params, dataset, batch_size: int = 256) -> float:
    """Top-1 error with running statistics (training.py:215-225)."""
    n = len(dataset.labels)
    wrong = 0
    dev = params[0].weight.device
    for s in range(0, n, batch_size):
        if isinstance(dataset.images, torch.Tensor):      # device-resident dataset
            x = dataset.images[s:s + batch_size].contiguous()
        else:
            x = torch.as_tensor(np.ascontiguousarray(dataset.images[s:s + batch_size],
                                                     dtype=np.float32)).to(dev)
        logits, _ = network_forward(spec, params, x, training=False)
        pred = logits.argmax(dim=1).cpu().numpy()
        wrong += int(np.count_nonzero(pred != np.asarray(dataset.labels[s:s + batch_size])))
    return wrong / n
