"""Dense tensor primitives on the GPU (drop-in for qtape.ops).

Same names/signatures as /root/reference/pkg/src/qtape/ops.py, operating on
``torch.cuda`` float32 tensors (rank 2 (N,C) or rank 4 NCHW, contiguous).

Precision contract (stated, and tested in tests/test_ops_gpu.py and, at network
level, tests/test_parity_gpu.py):
  * matmul: float64 ascending-k accumulation -> bit-identical to ops.matmul.
  * conv2d_forward / conv2d_backward: fp32-faithful implicit GEMMs (CUDA-core
    FFMA or tcgen05 split-precision); the reference accumulates in float64,
    so these match within ~1e-6 normwise relative error, not bitwise.
  * channel_moments / channel_sum / channel_mean: float64 deterministic
    reductions (a fixed partition, not numpy's pairwise order).
"""

from __future__ import annotations

import ctypes

import os
from typing import Optional

import torch

from . import _native as N
from .errors import ConfigError, ShapeError

DEBUG_CHECKS = bool(os.environ.get("QTAPE_DEBUG"))    # ops.py:21-35


def set_debug_checks(enabled: bool) -> None:
    global DEBUG_CHECKS
    DEBUG_CHECKS = bool(enabled)


def _check_finite(*ts):
    if DEBUG_CHECKS:
        for t in ts:
            if t is not None and not bool(torch.isfinite(t).all()):
                raise FloatingPointError("non-finite values in op result")


def reduce_axes(x) -> tuple:
    if x.dim() == 2:
        return (0,)
    if x.dim() == 4:
        return (0, 2, 3)
    raise ShapeError(f"expected rank 2 or 4 tensor, got rank {x.dim()}")


def channel_shape(vec, ndim: int):
    return vec.reshape(1, -1) if ndim == 2 else vec.reshape(1, -1, 1, 1)


def _dense(t, name):
    if not isinstance(t, torch.Tensor):
        raise ShapeError(f"{name} must be a torch tensor")
    N.require_cuda(t, name)
    if t.dtype != torch.float32:
        raise ConfigError(f"{name}: only float32 is implemented on the device (got {t.dtype})")
    return t if t.is_contiguous() else t.contiguous()


def nchw(x):
    """(n, c, hw) of a rank-2/4 tensor."""
    if x.dim() == 2:
        return x.shape[0], x.shape[1], 1
    if x.dim() == 4:
        return x.shape[0], x.shape[1], x.shape[2] * x.shape[3]
    raise ShapeError(f"expected rank 2 or 4 tensor, got rank {x.dim()}")


def matmul(a: torch.Tensor, b: torch.Tensor, out: Optional[torch.Tensor] = None,
           ta: bool = False, tb: bool = False, accumulate: bool = False) -> torch.Tensor:
    """C = A @ B with float64 ascending-k accumulation (ops.py:54-77).

    ``ta``/``tb`` read A/B as stored transposed (no copy); ``accumulate``
    adds the fp32-rounded product into ``out`` (``grad += matmul(..)``)."""
    if a.dim() != 2 or b.dim() != 2:
        raise ShapeError("matmul expects rank-2 operands")
    a, b = _dense(a, "a"), _dense(b, "b")
    m, k = (a.shape[1], a.shape[0]) if ta else (a.shape[0], a.shape[1])
    kb, n = (b.shape[1], b.shape[0]) if tb else (b.shape[0], b.shape[1])
    if k != kb:
        raise ShapeError(f"inner extents disagree: {tuple(a.shape)} x {tuple(b.shape)}")
    if out is None:
        if accumulate:
            raise ShapeError("accumulate needs out")
        out = torch.empty((m, n), dtype=torch.float32, device=a.device)
    N.call("qt_matmul", N.ptr(a), N.ptr(b), N.ptr(out), m, k, n, int(ta), int(tb),
           int(accumulate))
    _check_finite(out)
    return out


def conv2d_out_shape(in_shape: tuple, k_shape: tuple, stride: int, pad: int) -> tuple:
    """Integral-extent output shape or ShapeError (ops.py:80-94)."""
    n, ci, h, w = (int(v) for v in in_shape)
    co, kci, kh, kw = (int(v) for v in k_shape)
    if kci != ci:
        raise ShapeError(f"kernel expects {kci} input channels, got {ci}")
    if (h + 2 * pad - kh) % stride or (w + 2 * pad - kw) % stride:
        raise ShapeError(f"non-integral output extent for input {h}x{w}, kernel {kh}x{kw}, "
                         f"stride {stride}, pad {pad}")
    oh = (h + 2 * pad - kh) // stride + 1
    ow = (w + 2 * pad - kw) // stride + 1
    if oh <= 0 or ow <= 0:
        raise ShapeError("kernel larger than padded input")
    return n, co, oh, ow


def _conv_ws(k, ws, in_shape=None, stride=1, pad=0):
    co, ci, kh, kw = k.shape
    if in_shape is not None:
        n, _, h, w = in_shape
        need = N.query("qt_conv_workspace_ex", n, ci, h, w, co, kh, kw, stride, pad)
    else:
        need = N.query("qt_conv_workspace", ci, co, kh, kw)
    if ws is None or ws.numel() < need:
        ws = workspace(need, k.device, "conv")
    return ws


def conv2d_forward(x: torch.Tensor, k: torch.Tensor, stride: int = 1, pad: int = 0,
                   out: Optional[torch.Tensor] = None, residual: Optional[torch.Tensor] = None,
                   ws=None, prepared=None) -> torch.Tensor:
    """Cross-correlation with zero padding (ops.py:106-138).

    ``residual`` (engine use) fuses the parameter-free shortcut add of
    engine.py:262-269 into the epilogue; ``prepared`` (engine use) is the
    tensor-core weight operand already laid out by qt_conv_prepare_weights."""
    if x.dim() != 4 or k.dim() != 4:
        raise ShapeError("conv2d expects rank-4 input and kernel")
    x, k = _dense(x, "x"), _dense(k, "k")
    n, co, oh, ow = conv2d_out_shape(tuple(x.shape), tuple(k.shape), stride, pad)
    ci, kh, kw = k.shape[1:]
    if out is None:
        out = torch.empty((n, co, oh, ow), dtype=torch.float32, device=x.device)
    elif tuple(out.shape) != (n, co, oh, ow) or not out.is_contiguous():
        raise ShapeError("out has the wrong shape")
    cr, sr = 0, 1
    if residual is not None:
        cr = residual.shape[1]
        sr = residual.shape[2] // oh
    wp, wsp = (None, prepared) if prepared is not None else \
        (k, _conv_ws(k, ws, tuple(x.shape), stride, pad))
    N.call("qt_conv_forward", N.ptr(x), N.ptr(wp), N.ptr(out), n, ci, x.shape[2], x.shape[3], co,
           kh, kw, stride, pad, N.ptr(residual), cr, sr, N.ptr(wsp))
    _check_finite(out)
    return out


def conv2d_forward_fused(x: torch.Tensor, k: torch.Tensor, stride: int, pad: int,
                         out: torch.Tensor, residual=None, ws=None, prepared=None,
                         prologue=None, epilogue=None) -> torch.Tensor:
    """Engine form of the forward conv with layer fusion (qt_conv_forward_fused):
    ``prologue`` (N.BnPrologue) makes ``x`` the layer's pre-BN input and the
    conv apply BN + ReLU and write the K-bit tape in its operand staging;
    ``epilogue`` (N.BnStatsEpilogue) computes the next layer's BN statistics
    from the output.  Shapes must pass qt_conv_fused_support."""
    n, co, oh, ow = conv2d_out_shape(tuple(x.shape), tuple(k.shape), stride, pad)
    ci, kh, kw = k.shape[1:]
    cr, sr = 0, 1
    if residual is not None:
        cr = residual.shape[1]
        sr = residual.shape[2] // oh
    wp, wsp = (None, prepared) if prepared is not None else \
        (k, _conv_ws(k, ws, tuple(x.shape), stride, pad))
    N.call("qt_conv_forward_fused", N.ptr(x), N.ptr(wp), N.ptr(out), n, ci, x.shape[2],
           x.shape[3], co, kh, kw, stride, pad, N.ptr(residual), cr, sr,
           None if prologue is None else ctypes.byref(prologue),
           None if epilogue is None else ctypes.byref(epilogue), N.ptr(wsp))
    return out


_WS = {}


def workspace(nbytes: int, device, slot: str = "default") -> torch.Tensor:
    """Grow-only scratch buffer shared by standalone op calls (zero-filled:
    the reduction kernels keep their per-channel counters in it)."""
    key = (slot, str(device))
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.zeros(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        _WS[key] = buf
    return buf


def conv2d_wgrad(g_out, k_shape, stride, pad, grad_w, x_plain=None, tape=None, in_shape=None,
                 ws=None):
    """grad_w += weight gradient; the activation comes from ``x_plain`` or a
    native tape descriptor (relu(decode(codes)) fused into the operand load)."""
    n, ci, h, w = in_shape if in_shape is not None else x_plain.shape
    co, _, kh, kw = k_shape
    need = N.query("qt_conv_wgrad_workspace", n, ci, h, w, co, kh, kw, stride, pad)
    if ws is None or ws.numel() < need:
        ws = workspace(need, g_out.device, "wgrad")
    tp = tape if tape is not None else N.make_tape()
    N.call("qt_conv_wgrad", N.ptr(g_out), tp, N.ptr(x_plain), N.ptr(grad_w), n, ci, h, w, co, kh,
           kw, stride, pad, N.ptr(ws))


def conv2d_dgrad(g_out, k, in_shape, stride, pad, g_x_out, ws=None, prepared=None):
    n, ci, h, w = in_shape
    co, _, kh, kw = k.shape
    wp, wsp = (None, prepared) if prepared is not None else \
        (k, _conv_ws(k, ws, tuple(in_shape), stride, pad))
    N.call("qt_conv_dgrad", N.ptr(g_out), N.ptr(wp), N.ptr(g_x_out), n, ci, h, w, co, kh, kw,
           stride, pad, N.ptr(wsp))


def conv2d_backward(x: torch.Tensor, k: torch.Tensor, g_out: torch.Tensor, stride: int = 1,
                    pad: int = 0, g_x_out: Optional[torch.Tensor] = None, need_g_x: bool = True):
    """(g_x, g_k) adjoints of conv2d_forward (ops.py:141-183)."""
    x, k, g_out = _dense(x, "x"), _dense(k, "k"), _dense(g_out, "g_out")
    shape = conv2d_out_shape(tuple(x.shape), tuple(k.shape), stride, pad)
    if tuple(g_out.shape) != shape:
        raise ShapeError(f"gradient shape {tuple(g_out.shape)} != expected {shape}")
    g_k = torch.zeros_like(k)
    conv2d_wgrad(g_out, tuple(k.shape), stride, pad, g_k, x_plain=x)
    if not need_g_x:
        _check_finite(g_k)
        return None, g_k
    if g_x_out is None:
        g_x_out = torch.empty_like(x)
    conv2d_dgrad(g_out, k, tuple(x.shape), stride, pad, g_x_out)
    _check_finite(g_x_out, g_k)
    return g_x_out, g_k


def channel_moments(x: torch.Tensor, running=None, out=None, ws=None):
    """Per-channel population (mean, var), float64 (ops.py:186-196).

    ``running`` = (running_mean, running_var) additionally applies the
    layer.py:237-241 momentum update inside the same kernel."""
    x = _dense(x, "x")
    n, c, hw = nchw(x)
    if out is None:
        out = (torch.empty(c, dtype=torch.float64, device=x.device),
               torch.empty(c, dtype=torch.float64, device=x.device))
    need = N.query("qt_bn_stats_workspace", n, c, hw)
    if ws is None or ws.numel() < need:
        ws = workspace(need, x.device, "stats")
    rm, rv = running if running is not None else (None, None)
    N.call("qt_bn_stats", N.ptr(x), n, c, hw, N.ptr(out[0]), N.ptr(out[1]), N.ptr(rm), N.ptr(rv),
           N.ptr(ws))
    return out


def channel_sum(x: torch.Tensor) -> torch.Tensor:
    """Per-channel float64 sum over batch and spatial axes (ops.py:199-201)."""
    x = _dense(x, "x")
    n, c, hw = nchw(x)
    out = torch.empty(c, dtype=torch.float64, device=x.device)
    ws = workspace(N.query("qt_bn_stats_workspace", n, c, hw), x.device, "stats")
    N.call("qt_channel_sum", N.ptr(x), n, c, hw, N.ptr(out), N.ptr(ws))
    return out


def channel_mean(x: torch.Tensor) -> torch.Tensor:
    """Per-channel float64 mean (ops.py:204-206)."""
    n, c, hw = nchw(x)
    return channel_sum(x) / float(n * hw)
