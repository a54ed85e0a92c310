"""One pre-activation layer (BN -> scale/bias -> ReLU -> linear) on the GPU.

Drop-in for /root/reference/pkg/src/qtape/layer.py: the same modes
(exact / approx / naive), the same tape semantics (frozen gamma/beta, sigma2,
identity bypass with bits=None, plain stem layers keep a reference to their
input) and the same gradient accumulation (``+=`` into LayerParams.grad_*).

Forward per pre-activation layer = 3 launches:
  qt_bn_stats          (float64 moments + running-stat update)
  qt_bn_relu_forward   (BN apply -> K-bit codes / exact copy -> ReLU; K1)
  qt_conv_forward      (implicit GEMM; optional fused shortcut add)
Backward = qt_conv_wgrad (activation operand decoded from the codes inside
the GEMM's operand staging) + qt_conv_dgrad + qt_bn_backward_reduce/apply
(mask, Eq. 5-8 and the shortcut adjoint from the same codes).  No
full-precision activation is re-materialised for approx tapes.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional

import torch

from . import _native as N
from . import ops
from .codec import QuantizedTape, _nch_hw, packed_nbytes
from .errors import ConfigError, ShapeError, StateError

MODES = ("exact", "approx", "naive")          # layer.py:32
RUNNING_STAT_MOMENTUM = 0.9                   # layer.py:34
_NATIVE_MODE = {"exact": 0, "approx": 1, "naive": 2}


def _dev_f32(t, name):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise ConfigError(f"{name} must be a torch tensor")
    N.require_cuda(t, name)
    if t.dtype != torch.float32:
        raise ConfigError(f"{name}: device layers are float32 only (got {t.dtype})")
    return t


@dataclass
class LayerParams:
    """Learnable state of one layer plus gradient / momentum / running-stat
    slots (layer.py:37-103).  ``kind`` is conv | dense | gap_dense; dense
    weights are (Din, Dout), conv weights (Cout, Cin, kh, kw)."""

    kind: str
    weight: torch.Tensor
    stride: int = 1
    pad: int = 0
    gamma: Optional[torch.Tensor] = None
    beta: Optional[torch.Tensor] = None
    bn_epsilon: float = 1e-5
    grad_weight: torch.Tensor = None
    grad_gamma: Optional[torch.Tensor] = None
    grad_beta: Optional[torch.Tensor] = None
    vel_weight: torch.Tensor = None
    vel_gamma: Optional[torch.Tensor] = None
    vel_beta: Optional[torch.Tensor] = None
    running_mean: Optional[torch.Tensor] = None
    running_var: Optional[torch.Tensor] = None

    def __post_init__(self):
        _dev_f32(self.weight, "weight")
        z = torch.zeros_like
        if self.grad_weight is None:
            self.grad_weight = z(self.weight)
        if self.vel_weight is None:
            self.vel_weight = z(self.weight)
        if self.preact:
            _dev_f32(self.gamma, "gamma")
            _dev_f32(self.beta, "beta")
            c = self.gamma.numel()
            if self.beta.numel() != c:
                raise ShapeError("gamma/beta length mismatch")
            for name in ("grad_gamma", "vel_gamma"):
                if getattr(self, name) is None:
                    setattr(self, name, z(self.gamma))
            for name in ("grad_beta", "vel_beta"):
                if getattr(self, name) is None:
                    setattr(self, name, z(self.beta))
            dev = self.gamma.device
            if self.running_mean is None:
                self.running_mean = torch.zeros(c, dtype=torch.float64, device=dev)
            if self.running_var is None:
                self.running_var = torch.ones(c, dtype=torch.float64, device=dev)

    @property
    def preact(self) -> bool:
        return self.gamma is not None

    @property
    def dtype(self):
        return self.weight.dtype

    def zero_grads(self) -> None:
        self.grad_weight.zero_()
        if self.preact:
            self.grad_gamma.zero_()
            self.grad_beta.zero_()

    def param_nbytes(self) -> int:
        n = self.weight.numel() * 4
        if self.preact:
            n += (self.gamma.numel() + self.beta.numel()) * 4
        return n


@dataclass
class LayerTape:
    """Per-layer state retained for the backward pass (layer.py:106-129)."""

    mode: str
    stored: object                          # fp32 tensor, QuantizedTape or None
    sigma2: Optional[torch.Tensor] = None   # float64 [C]
    gamma: Optional[torch.Tensor] = None    # frozen copies (layer.py:253-255)
    beta: Optional[torch.Tensor] = None
    bn_epsilon: float = 1e-5
    identity: bool = False
    input_ref: Optional[torch.Tensor] = None

    @property
    def is_quantized(self) -> bool:
        return isinstance(self.stored, QuantizedTape)

    @property
    def shape(self):
        return tuple(self.stored.shape)

    def stored_nbytes(self) -> int:
        if isinstance(self.stored, QuantizedTape):
            return self.stored.nbytes_codes()
        if isinstance(self.stored, torch.Tensor):
            return self.stored.numel() * self.stored.element_size()
        return 0

    def as_native(self):
        if self.is_quantized:
            return self.stored.as_native()
        return N.make_tape(a2=self.stored)


class TapeSlot:
    """Preallocated device storage for one layer's tape (engine arenas and
    CUDA-graph capture reuse it across steps)."""

    def __init__(self, shape, c, bits, exact, device, codes=None, a2=None, clip=None):
        self.shape = tuple(shape)
        self.bits = bits
        self.mean = torch.empty(c, dtype=torch.float64, device=device)
        self.var = torch.empty(c, dtype=torch.float64, device=device)
        self.gamma = torch.empty(c, dtype=torch.float32, device=device)
        self.beta = torch.empty(c, dtype=torch.float32, device=device)
        self.consts = torch.empty(c * 48, dtype=torch.uint8, device=device)  # BnConst[C]
        if exact:
            self.a2 = a2 if a2 is not None else torch.empty(shape, dtype=torch.float32,
                                                             device=device)
            self.codes = None
        else:
            numel = 1
            for s in shape:
                numel *= int(s)
            self.a2 = None
            self.codes = codes if codes is not None else torch.empty(
                packed_nbytes(numel, bits), dtype=torch.uint8, device=device)
        if exact:
            self.step = self.offset = self.clip = None
        else:
            self.step = torch.empty(c, dtype=torch.float64, device=device)
            self.offset = torch.empty(c, dtype=torch.int64, device=device)
            self.clip = clip if clip is not None else torch.zeros(1, dtype=torch.int64,
                                                                  device=device)


def safe_gamma(gamma: torch.Tensor) -> torch.Tensor:
    """gamma with magnitude floored, sign kept (layer.py:132-135) -- diagnostics."""
    mag = torch.clamp_min(gamma.abs(), 1e-8)
    return torch.where(gamma < 0, -mag, mag)


def linear_out_shape(p: LayerParams, in_shape: tuple) -> tuple:
    """layer.py:188-195."""
    if p.kind == "conv":
        return ops.conv2d_out_shape(in_shape, tuple(p.weight.shape), p.stride, p.pad)
    if p.kind in ("dense", "gap_dense"):
        return (in_shape[0], p.weight.shape[1])
    raise StateError(f"unknown layer kind {p.kind!r}")


def _gap(a3: torch.Tensor) -> torch.Tensor:
    """(N,C,H,W) -> (N,C) float64 mean (layer.py:154-157)."""
    n, c, hw = ops.nchw(a3)
    out = torch.empty((n, c), dtype=torch.float32, device=a3.device)
    N.call("qt_gap", N.ptr(a3), n, c, hw, N.ptr(out))
    return out


def _bn_fused(n: int, c: int, hw: int) -> bool:
    """qt_bn_forward_fused takes this shape and is enabled (QTAPE_BN_FUSED=1).

    Off by default: measured on the C2 step the one-launch form is slower
    (2.18-2.27 vs 0.92 + 1.05 ms/step for the two launches; 3.36 with 512
    threads): its apply pass is confined to the statistics partition (one
    cluster of <= 8 blocks per channel), while qt_bn_relu_forward spreads the
    elementwise work over the whole GPU."""
    if os.environ.get("QTAPE_BN_FUSED", "0") in ("", "0"):
        return False
    return bool(N.query("qt_bn_forward_fused_ok", n, c, hw))


def _prepared(ws, p: LayerParams, dgrad: int):
    """Tensor-core weight operand of ``p`` prepared by the Trainer for this
    step (Workspace.prep, keyed by the LayerParams object), else None: the
    conv call then lays out the operand from ``p.weight`` itself.  The
    prepared copies live in the Trainer's workspace only, so eager calls on
    the same parameters never see a stale (pre-SGD) operand."""
    prep = getattr(ws, "prep", None)
    if not prep:
        return None
    ent = prep.get(id(p))
    return None if ent is None else ent[dgrad]


def _linear_forward(a3, p: LayerParams, out, residual=None, ws=None, epilogue=None):
    """layer.py:138-151; ``residual`` fuses the block-end shortcut add,
    ``epilogue`` (engine) the next layer's BN statistics."""
    if p.kind == "conv":
        if epilogue is not None:
            return ops.conv2d_forward_fused(a3, p.weight, p.stride, p.pad, out, residual,
                                            ws=ws.conv, prepared=_prepared(ws, p, 0),
                                            epilogue=epilogue)
        return ops.conv2d_forward(a3, p.weight, p.stride, p.pad, out=out, residual=residual,
                                  ws=None if ws is None else ws.conv, prepared=_prepared(ws, p, 0))
    if p.kind == "dense":
        src = a3
    elif p.kind == "gap_dense":
        src = _gap(a3) if a3.dim() == 4 else a3
    else:
        raise StateError(f"unknown layer kind {p.kind!r}")
    r = ops.matmul(src, p.weight, out=out)
    if residual is not None:
        raise StateError("shortcut add needs a conv layer at the block end")
    return r


def layer_forward(a_in: torch.Tensor, p: LayerParams, mode: str = "exact",
                  bits: Optional[int] = 8, training: bool = True,
                  out: Optional[torch.Tensor] = None, work: Optional[torch.Tensor] = None,
                  slot: Optional[TapeSlot] = None, residual: Optional[torch.Tensor] = None,
                  ws=None, fuse: Optional[dict] = None):
    """Run the layer forward; returns (a_out, tape) (layer.py:208-266).

    ``work`` receives the ReLU'd activations and may not alias ``a_in``;
    ``out`` may share storage with ``a_in``.  ``slot``/``residual``/``ws`` are
    engine hooks (preallocated tape storage, fused shortcut add, scratch).

    ``fuse`` (engine hook, DESIGN.md section 3 "layer fusion"):
      stats_done -- this layer's statistics and constants were already
                    written into ``slot`` by the previous conv's epilogue;
      pro        -- the conv applies BN + ReLU and writes the K-bit tape in
                    its operand staging (no qt_bn_relu_forward, no ``work``);
      epi        -- N.BnStatsEpilogue: the conv's epilogue computes the NEXT
                    layer's statistics."""
    if mode not in MODES:
        raise StateError(f"unknown mode {mode!r}")
    if bits is not None and bits not in (1, 2, 4, 8):
        raise ConfigError(f"bits must be one of (1, 2, 4, 8), got {bits}")
    _dev_f32(a_in, "a_in")
    fz = fuse or {}
    if not p.preact:
        a_out = _linear_forward(a_in, p, out, residual, ws, epilogue=fz.get("epi"))
        return a_out, LayerTape(mode="plain", stored=None, input_ref=a_in)

    n, c, hw = ops.nchw(a_in)
    if p.gamma.numel() != c:
        raise ShapeError(f"layer expects {p.gamma.numel()} channels, got {c}")
    a_in = a_in.contiguous()
    dev = a_in.device
    quantized = training and mode != "exact" and bits is not None
    fused_in = bool(fz.get("pro")) and quantized and mode == "approx" and p.kind == "conv"
    if fused_in:
        if slot is None or ws is None:
            raise StateError("the fused BN prologue is an engine path (slot and ws required)")
    elif work is None:
        work = torch.empty_like(a_in)
    elif work.data_ptr() == a_in.data_ptr():
        raise StateError("work may not alias a_in")

    a2_tape = codes = step = offset = clip = consts = None
    bn_done = False
    kbits = 0
    nmode = 0
    if training:
        if slot is None:
            slot = TapeSlot(a_in.shape, c, bits, not quantized, dev)
        if quantized:
            codes, step, offset, clip = slot.codes, slot.step, slot.offset, slot.clip
            kbits = bits
            nmode = _NATIVE_MODE[mode]
        else:
            a2_tape = slot.a2
        # one launch: moments + running stats + K1 constants + frozen gamma/beta
        # + tape step/offset + clip-counter reset (layer.py:236-255)
        mean, var, consts = slot.mean, slot.var, slot.consts
        if not fz.get("stats_done") and not fused_in and _bn_fused(n, c, hw):
            # statistics + BN apply + tape + ReLU in one launch; its clip
            # count accumulates into a counter that is zero here (a fresh
            # slot, or the engine zeroed the arena's counters this pass)
            N.call("qt_bn_forward_fused", N.ptr(a_in), n, c, hw, float(p.bn_epsilon),
                   N.ptr(p.gamma), N.ptr(p.beta), nmode, kbits, N.ptr(mean), N.ptr(var),
                   N.ptr(p.running_mean), N.ptr(p.running_var), N.ptr(slot.gamma),
                   N.ptr(slot.beta), N.ptr(step), N.ptr(offset), N.ptr(clip), N.ptr(consts),
                   N.ptr(work), N.ptr(a2_tape), N.ptr(codes))
            bn_done = True
        elif not fz.get("stats_done"):
            if ws is not None:
                sws = ws.stats
            else:
                sws = ops.workspace(N.query("qt_bn_stats_workspace", n, c, hw), dev, "stats")
            N.call("qt_bn_stats_prep", N.ptr(a_in), n, c, hw, float(p.bn_epsilon),
                   N.ptr(p.gamma), N.ptr(p.beta), kbits, N.ptr(mean), N.ptr(var),
                   N.ptr(p.running_mean), N.ptr(p.running_var), N.ptr(slot.gamma),
                   N.ptr(slot.beta), N.ptr(step), N.ptr(offset), N.ptr(clip), N.ptr(consts),
                   N.ptr(sws))
    else:
        mean, var = p.running_mean, p.running_var
    if not fused_in and not bn_done:
        N.call("qt_bn_relu_forward", N.ptr(a_in), n, c, hw, N.ptr(mean), N.ptr(var),
               float(p.bn_epsilon), N.ptr(p.gamma), N.ptr(p.beta), nmode, kbits, N.ptr(work),
               N.ptr(a2_tape), N.ptr(codes), N.ptr(step), N.ptr(offset), N.ptr(clip),
               N.ptr(consts))

    tape = None
    if training:
        if quantized:
            stored = QuantizedTape(codes=codes, bits=bits, shape=tuple(a_in.shape),
                                   dtype=torch.float32, step=step, offset=offset, sigma2=var,
                                   clip_counter=clip)
        else:
            stored = a2_tape
        tape = LayerTape(mode=mode, stored=stored, sigma2=var, gamma=slot.gamma,
                         beta=slot.beta, bn_epsilon=p.bn_epsilon,
                         identity=(bits is None and mode != "exact"))
    if fused_in:   # BN apply + ReLU + tape inside the conv's operand staging
        pro = N.BnPrologue(N.ptr(consts), N.ptr(codes), N.ptr(clip), int(bits))
        a_out = ops.conv2d_forward_fused(a_in, p.weight, p.stride, p.pad, out, residual,
                                         ws=ws.conv, prepared=_prepared(ws, p, 0),
                                         prologue=pro, epilogue=fz.get("epi"))
    else:
        a_out = _linear_forward(work, p, out, residual, ws, epilogue=fz.get("epi"))
    ops._check_finite(a_out)
    return a_out, tape


def reconstruct_from_tape(tape: LayerTape):
    """(normalized a1, pre-ReLU a2, rectified a3) from a tape (layer.py:269-283)."""
    if tape is None or tape.mode == "plain":
        raise StateError("plain layer tapes hold no activations")
    shape = tape.shape
    n, c, hw = _nch_hw(shape)
    dev = tape.gamma.device
    a1, a2, a3 = (torch.empty(shape, dtype=torch.float32, device=dev) for _ in range(3))
    N.call("qt_reconstruct", tape.as_native(), n, c, hw, N.ptr(tape.gamma), N.ptr(tape.beta),
           N.ptr(a1), N.ptr(a2), N.ptr(a3))
    return a1, a2, a3


def bn_input_gradient(a1: torch.Tensor, g1: torch.Tensor, sigma2: torch.Tensor, eps: float,
                      variance_a1: Optional[torch.Tensor] = None,
                      out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """inv * [g1 - mean(g1) - a1v * mean(a1v * g1)] (layer.py:286-308).

    Standalone utility (the engine's backward runs the fused
    qt_bn_backward_reduce/apply kernels instead); float64 channel means come
    from the native reduction, the elementwise steps keep the reference's
    fp32 rounding points."""
    a1v = a1 if variance_a1 is None else variance_a1
    shp = (1, -1) + (1,) * (g1.dim() - 2)
    t2 = ops.channel_mean(g1).float()
    t3 = ops.channel_mean(a1v * g1).float()
    inv = (1.0 / torch.sqrt(sigma2.double() + eps)).float()
    if out is None:
        out = torch.empty_like(g1)
    torch.sub(g1, t2.reshape(shp), out=out)
    out -= a1v * t3.reshape(shp)
    out *= inv.reshape(shp)
    return out


def _apply_adjoint(g_in, res_g):
    """engine.py:272-279 as a standalone kernel."""
    n, c, h, w = g_in.shape
    N.call("qt_shortcut_adjoint", N.ptr(g_in), N.ptr(res_g), n, c, h, w, res_g.shape[1],
           h // res_g.shape[2])


def _on_side(ws, fn) -> None:
    """Run a weight-gradient launch on the engine's side stream when it has
    one: it forks after everything queued so far on the current stream and
    leaves its completion event in ``ws.wgrad_done`` (the engine fences the
    g_out buffer with it and joins before SGD)."""
    side = getattr(ws, "side", None)
    if side is None:
        fn()
        return
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    ev = torch.cuda.Event()
    ev.record(side)
    ws.wgrad_done = ev


def layer_backward(g_out: torch.Tensor, tape: LayerTape, p: LayerParams,
                   out: Optional[torch.Tensor] = None, need_input_grad: bool = True,
                   variance_a1: Optional[torch.Tensor] = None,
                   internals: Optional[dict] = None, residual_grad: Optional[torch.Tensor] = None,
                   ws=None):
    """Backward through the layer (layer.py:311-381): accumulates parameter
    gradients into ``p`` and returns the input gradient (into ``out``).

    ``residual_grad`` (engine hook) fuses the block-start shortcut adjoint
    add into the final elementwise kernel."""
    if tape is None:
        raise StateError("no tape: layer was run in evaluation mode")
    _dev_f32(g_out, "g_out")
    g_out = g_out.contiguous()
    if tape.mode == "plain":
        a_in = tape.input_ref
        if p.kind != "conv":
            ops.matmul(a_in, g_out, out=p.grad_weight, ta=True, accumulate=True)
            if not need_input_grad:
                return None
            g_in = ops.matmul(g_out, p.weight, out=out, tb=True)
        else:
            x_plain = a_in.contiguous()
            _on_side(ws, lambda: ops.conv2d_wgrad(g_out, tuple(p.weight.shape), p.stride, p.pad,
                                                  p.grad_weight, x_plain=x_plain,
                                                  ws=None if ws is None else ws.wgrad))
            if not need_input_grad:
                return None
            g_in = out if out is not None else torch.empty_like(a_in)
            ops.conv2d_dgrad(g_out, p.weight, tuple(a_in.shape), p.stride, p.pad, g_in,
                             ws=None if ws is None else ws.conv, prepared=_prepared(ws, p, 1))
        if residual_grad is not None:
            _apply_adjoint(g_in, residual_grad)
        return g_in

    if tape.gamma is None or tape.gamma.numel() != p.gamma.numel():
        raise StateError("tape does not match layer parameters")
    in_shape = tape.shape
    if linear_out_shape(p, in_shape) != tuple(g_out.shape):
        raise StateError(f"g_out shape {tuple(g_out.shape)} inconsistent with tape {in_shape}")
    nt = tape.as_native()
    dev = g_out.device
    g3 = out if out is not None else torch.empty(in_shape, dtype=torch.float32, device=dev)

    # linear transform backward (layer.py:353-362)
    if p.kind == "conv":
        _on_side(ws, lambda: ops.conv2d_wgrad(g_out, tuple(p.weight.shape), p.stride, p.pad,
                                              p.grad_weight, tape=nt, in_shape=in_shape,
                                              ws=None if ws is None else ws.wgrad))
        ops.conv2d_dgrad(g_out, p.weight, in_shape, p.stride, p.pad, g3,
                         ws=None if ws is None else ws.conv, prepared=_prepared(ws, p, 1))
    else:
        _, _, a3 = reconstruct_from_tape(tape)
        if p.kind == "dense":
            ops.matmul(a3, g_out, out=p.grad_weight, ta=True, accumulate=True)
            ops.matmul(g_out, p.weight, out=g3, tb=True)
        elif p.kind == "gap_dense":
            pooled = _gap(a3)
            ops.matmul(pooled, g_out, out=p.grad_weight, ta=True, accumulate=True)
            g_pool = ops.matmul(g_out, p.weight, tb=True)
            n, c, hw = ops.nchw(a3)
            N.call("qt_gap_backward", N.ptr(g_pool), n, c, hw, N.ptr(g3))
        else:
            raise StateError(f"unknown layer kind {p.kind!r}")

    if internals is not None:
        a1_i, a2_i, _ = reconstruct_from_tape(tape)
        mask = a2_i > 0
        internals["mask"] = mask
        internals["grad_linear_in"] = g3.clone()

    n, c, hw = ops.nchw(g3)
    if ws is not None:
        bws, stats = ws.bnb, ws.bn_stats[: 3 * c]
    else:
        bws = ops.workspace(N.query("qt_bn_backward_workspace", n, c, hw), dev, "bnb")
        stats = torch.empty(3 * c, dtype=torch.float32, device=dev)
    N.call("qt_bn_backward_reduce", N.ptr(g3), nt, n, c, hw, N.ptr(tape.gamma), N.ptr(tape.beta),
           N.ptr(tape.sigma2), float(tape.bn_epsilon), N.ptr(variance_a1), N.ptr(p.grad_gamma),
           N.ptr(p.grad_beta), N.ptr(stats), N.ptr(bws))

    if internals is not None:
        shp = (1, -1) + (1,) * (g3.dim() - 2)
        gm = g3 * internals["mask"]
        internals["grad_pre_relu"] = gm.clone()
        internals["grad_normalized"] = gm * tape.gamma.reshape(shp)
        internals["a1"] = a1_i

    if not need_input_grad:
        return None
    h, w = (g3.shape[2], g3.shape[3]) if g3.dim() == 4 else (1, 1)
    cr, sc = 0, 1
    if residual_grad is not None:
        cr = residual_grad.shape[1]
        sc = h // residual_grad.shape[2] if g3.dim() == 4 else 1
    N.call("qt_bn_backward_apply", N.ptr(g3), nt, n, c, h, w, N.ptr(tape.gamma), N.ptr(tape.beta),
           N.ptr(variance_a1), N.ptr(stats), N.ptr(residual_grad), cr, sc, N.ptr(bws), N.ptr(g3))
    ops._check_finite(g3)
    return g3
