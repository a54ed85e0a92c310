"""numpy restatement of the reference approximate-activation training step.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Every function cites
the reference ``/root/reference/pkg/src/qtape`` file:line whose arithmetic it
restates.  Arithmetic that the reference defines bit-exactly (codec, BN
apply, fixed-order conv forward / matmul, SGD) is restated with the same
operation order and rounding points; BLAS-ordered backward contractions are
restated with float64 BLAS as well and are compared with a tolerance.

Data model: a network is the reference's JSON spec dict
(``NetworkSpec.to_json``, engine.py:166-170); parameters are plain dicts.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

__all__ = [
    "BITS", "GAMMA_FLOOR", "code_constants", "raw_codes", "quantize", "pack",
    "unpack", "dequantize", "decode_threshold", "conv_out_shape", "conv_fwd",
    "conv_bwd", "moments", "chan_sum", "chan_mean", "matmul_fixed", "safe_gamma",
    "new_params", "layer_fwd", "layer_bwd", "net_shapes", "net_width",
    "net_fwd", "net_bwd", "softmax_xent", "sgd", "init_params", "train_step",
    "ref_kernels_available",
]

BITS = (1, 2, 4, 8)              # codec.py:20
GAMMA_FLOOR = 1e-8               # codec.py:24
RUN_MOMENTUM = 0.9               # layer.py:34
DEFAULT_EPS = 1e-5               # layer.py:53


def _b(v, ndim):
    """Per-channel broadcast on axis 1 (ops.py:47-51)."""
    return np.asarray(v).reshape((1, -1) + (1,) * (ndim - 2))


def _axes(ndim):
    """Reduction axes: everything but channels (ops.py:38-44)."""
    if ndim == 2:
        return (0,)
    if ndim == 4:
        return (0, 2, 3)
    raise ValueError(f"rank {ndim} unsupported")


# ---------------------------------------------------------------- codec ---

def code_constants(gamma, beta, bits):
    """(scale, step, offset) per channel.

    codec.py:27-29 (|gamma| floored), :101-104 (scale 2^K/(6g), step 6g*2^-K),
    :117 / :137 (offset = floor(beta*scale) as int64).
    """
    if bits not in BITS:
        raise ValueError(f"bits {bits}")
    g6 = 6.0 * np.maximum(np.abs(np.asarray(gamma).astype(np.float64)), GAMMA_FLOOR)
    scale = (2.0 ** bits) / g6
    step = g6 * (2.0 ** -bits)
    with np.errstate(invalid="ignore"):
        offset = np.floor(np.asarray(beta).astype(np.float64) * scale).astype(np.int64)
    return scale, step, offset


def raw_codes(a, gamma, beta, bits):
    """Unclipped int64 codes, codec.py:107-120 (float64 math, x86 int cast)."""
    scale, _, offset = code_constants(gamma, beta, bits)
    with np.errstate(invalid="ignore", over="ignore"):
        u = np.floor(np.asarray(a).astype(np.float64) * _b(scale, a.ndim))
        return u.astype(np.int64) + (1 << (bits - 1)) - _b(offset, a.ndim)


def pack(codes, bits):
    """Little-endian K-bit packing in flat C order, codec.py:59-78."""
    c = np.asarray(codes)
    if c.size and (c.min() < 0 or c.max() >= (1 << bits)):
        raise ValueError("code out of range")
    c = c.astype(np.uint8).ravel()
    if bits == 8:
        return c.copy()
    per = 8 // bits
    c = np.concatenate([c, np.zeros((-c.size) % per, np.uint8)]).reshape(-1, per)
    out = np.zeros(c.shape[0], np.uint8)
    for j in range(per):
        out |= (c[:, j] << np.uint8(j * bits)).astype(np.uint8)
    return out


def unpack(packed, bits, count):
    """Inverse of ``pack``; byte-count check as codec.py:86-90."""
    p = np.asarray(packed, dtype=np.uint8).ravel()
    if p.size != (count * bits + 7) // 8:
        raise ValueError("wrong byte count")
    if bits == 8:
        return p[:count].copy()
    per = 8 // bits
    sh = np.arange(per, dtype=np.uint8) * np.uint8(bits)
    return ((p[:, None] >> sh[None, :]) & np.uint8((1 << bits) - 1)).reshape(-1)[:count]


def quantize(a, gamma, beta, bits, sigma2=None):
    """codec.py:123-143 -> dict mirroring QuantizedTape (codec.py:32-56)."""
    raw = raw_codes(a, gamma, beta, bits)
    top = (1 << bits) - 1
    clip = int(np.count_nonzero((raw < 0) | (raw > top)))
    _, step, offset = code_constants(gamma, beta, bits)
    c = a.shape[1]
    return {
        "codes": pack(np.clip(raw, 0, top), bits), "bits": bits,
        "shape": tuple(a.shape), "dtype": a.dtype, "step": step,
        "offset": offset.astype(np.int64),
        "sigma2": (np.zeros(c) if sigma2 is None else np.asarray(sigma2, np.float64)),
        "clip_count": clip,
    }


def dequantize(t):
    """Interval medians with frozen constants, codec.py:146-156."""
    shape = t["shape"]
    codes = unpack(t["codes"], t["bits"], int(np.prod(shape))).reshape(shape)
    half = float(1 << (t["bits"] - 1))
    inner = codes.astype(np.float64) + (0.5 - half)
    inner = inner + _b(t["offset"].astype(np.float64), len(shape))
    return (_b(t["step"], len(shape)) * inner).astype(t["dtype"])


def decode_threshold(t):
    """Smallest positive code per channel, codec.py:165-173."""
    return ((1 << (t["bits"] - 1)) - t["offset"]).astype(np.int64)


# ------------------------------------------------------------------ ops ---

_REF_LIB = None
_REF_TRIED = False


def _ref_lib():
    """oracle/_ref/libqtape_ref_kernels.so: the reference's own _kernels.c
    compiled by oracle/Makefile with _native.py:26-29's flags."""
    global _REF_LIB, _REF_TRIED
    if _REF_TRIED:
        return _REF_LIB
    _REF_TRIED = True
    so = Path(__file__).parent / "_ref" / "libqtape_ref_kernels.so"
    if so.exists() and not os.environ.get("QTAPE_ORACLE_NO_REF"):
        lib = ctypes.CDLL(str(so))
        lib.conv_fwd_f32.restype = None
        lib.conv_fwd_f64.restype = None
        _REF_LIB = lib
    return _REF_LIB


def ref_kernels_available() -> bool:
    return _ref_lib() is not None


def conv_out_shape(in_shape, k_shape, stride, pad):
    """Integral-extent rule, ops.py:80-94."""
    n, ci, h, w = in_shape
    co, kci, kh, kw = k_shape
    if kci != ci:
        raise ValueError("channel mismatch")
    if (h + 2 * pad - kh) % stride or (w + 2 * pad - kw) % stride:
        raise ValueError("non-integral output extent")
    oh = (h + 2 * pad - kh) // stride + 1
    ow = (w + 2 * pad - kw) // stride + 1
    if oh <= 0 or ow <= 0:
        raise ValueError("kernel larger than padded input")
    return n, co, oh, ow


def _padded(x, pad):
    if not pad:
        return np.ascontiguousarray(x)
    n, c, h, w = x.shape
    xp = np.zeros((n, c, h + 2 * pad, w + 2 * pad), x.dtype)
    xp[:, :, pad:pad + h, pad:pad + w] = x
    return xp


def conv_fwd(x, k, stride=1, pad=0):
    """Cross-correlation, float64 accumulation over (ci,u,v) ascending,
    one multiply and one add rounding per term (ops.py:106-138,
    _kernels.c:10-49).  Uses the reference C kernel when built."""
    n, co, oh, ow = conv_out_shape(x.shape, k.shape, stride, pad)
    ci, kh, kw = k.shape[1:]
    xp = _padded(x, pad)
    k = np.ascontiguousarray(k, dtype=x.dtype)
    acc = np.zeros((n, co, oh, ow), np.float64)
    lib = _ref_lib()
    if lib is not None and x.dtype in (np.float32, np.float64):
        fn = lib.conv_fwd_f32 if x.dtype == np.float32 else lib.conv_fwd_f64
        fn(xp.ctypes.data_as(ctypes.c_void_p), k.ctypes.data_as(ctypes.c_void_p),
           acc.ctypes.data_as(ctypes.c_void_p),
           *(ctypes.c_long(int(v)) for v in
             (n, ci, xp.shape[2], xp.shape[3], co, kh, kw, oh, ow, stride)))
    else:
        k64 = k.astype(np.float64)
        term = np.empty_like(acc)
        for c in range(ci):
            for u in range(kh):
                for v in range(kw):
                    win = xp[:, c, u:u + stride * oh:stride, v:v + stride * ow:stride]
                    np.multiply(win[:, None].astype(np.float64),
                                k64[None, :, c, u, v, None, None], out=term)
                    acc += term
    return acc.astype(x.dtype)


def conv_bwd(x, k, g, stride=1, pad=0, need_gx=True):
    """(g_x, g_k) adjoints in float64 BLAS, ops.py:141-183."""
    n, co, oh, ow = conv_out_shape(x.shape, k.shape, stride, pad)
    ci, kh, kw = k.shape[1:]
    h, w = x.shape[2:]
    xp = _padded(x, pad).astype(np.float64)
    g64 = g.astype(np.float64)
    k64 = k.astype(np.float64)
    gk = np.empty((co, ci, kh, kw))
    gxp = np.zeros_like(xp) if need_gx else None
    for u in range(kh):
        for v in range(kw):
            sl = (slice(None), slice(None), slice(u, u + stride * oh, stride),
                  slice(v, v + stride * ow, stride))
            gk[:, :, u, v] = np.tensordot(g64, xp[sl], axes=([0, 2, 3], [0, 2, 3]))
            if need_gx:
                gxp[sl] += np.tensordot(g64, k64[:, :, u, v],
                                        axes=([1], [0])).transpose(0, 3, 1, 2)
    gk = gk.astype(k.dtype)
    if not need_gx:
        return None, gk
    gx = gxp[:, :, pad:pad + h, pad:pad + w] if pad else gxp
    return gx.astype(x.dtype), gk


def moments(x):
    """Two-pass population mean/var in float64, ops.py:186-196."""
    ax = _axes(x.ndim)
    x64 = x.astype(np.float64)
    mean = x64.mean(axis=ax)
    var = np.square(x64 - _b(mean, x.ndim)).mean(axis=ax)
    return mean, var


def chan_sum(x):
    """ops.py:199-201."""
    return x.astype(np.float64).sum(axis=_axes(x.ndim))


def chan_mean(x):
    """ops.py:204-206."""
    return x.astype(np.float64).mean(axis=_axes(x.ndim))


def matmul_fixed(a, b):
    """Ascending-k float64 accumulation, one rounding per mul/add
    (ops.py:54-77)."""
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    acc = np.zeros((a.shape[0], b.shape[1]))
    for kk in range(a.shape[1]):
        acc += a64[:, kk, None] * b64[None, kk, :]
    return acc.astype(a.dtype)


# ---------------------------------------------------------------- layer ---

def safe_gamma(gamma):
    """layer.py:132-135."""
    mag = np.maximum(np.abs(gamma), gamma.dtype.type(GAMMA_FLOOR))
    return np.where(gamma < 0, -mag, mag)


def new_params(kind, weight, stride=1, pad=0, gamma=None, beta=None, eps=DEFAULT_EPS):
    """LayerParams equivalent (layer.py:37-103)."""
    p = {"kind": kind, "weight": weight, "stride": stride, "pad": pad,
         "gamma": gamma, "beta": beta, "eps": eps,
         "grad_weight": np.zeros_like(weight), "vel_weight": np.zeros_like(weight)}
    if gamma is not None:
        c = len(gamma)
        p.update(grad_gamma=np.zeros_like(gamma), grad_beta=np.zeros_like(beta),
                 vel_gamma=np.zeros_like(gamma), vel_beta=np.zeros_like(beta),
                 running_mean=np.zeros(c), running_var=np.ones(c))
    return p


def _gap(a3):
    """layer.py:154-157."""
    return a3.astype(np.float64).mean(axis=tuple(range(2, a3.ndim))).astype(a3.dtype)


def _lin_fwd(a3, p):
    """layer.py:138-151."""
    if p["kind"] == "conv":
        return conv_fwd(a3, p["weight"], p["stride"], p["pad"])
    if p["kind"] == "dense":
        return matmul_fixed(a3, p["weight"])
    return matmul_fixed(_gap(a3), p["weight"])


def _lin_bwd(a3, g, p, need_gx=True):
    """layer.py:160-185; accumulates into grad_weight."""
    if p["kind"] == "conv":
        gx, gk = conv_bwd(a3, p["weight"], g, p["stride"], p["pad"], need_gx)
        p["grad_weight"] += gk
        return gx
    if p["kind"] == "dense":
        p["grad_weight"] += matmul_fixed(a3.T.copy(), g)
        return matmul_fixed(g, p["weight"].T.copy()) if need_gx else None
    hw = int(np.prod(a3.shape[2:])) if a3.ndim == 4 else 1
    p["grad_weight"] += matmul_fixed(_gap(a3).T.copy(), g)
    gp = matmul_fixed(g, p["weight"].T.copy())
    return np.ascontiguousarray(np.broadcast_to(
        (gp / a3.dtype.type(hw)).reshape(a3.shape[:2] + (1,) * (a3.ndim - 2)),
        a3.shape))


def layer_fwd(a_in, p, mode="exact", bits=8, training=True, keep_a2=False):
    """layer.py:208-266 -> (a_out, tape dict or None).

    ``keep_a2`` (test instrumentation, not in the reference) also keeps the
    pre-ReLU A2 of a quantized tape as ``tape["a2_pre"]`` (and the layer
    input as ``tape["a_in"]``) so a parity test can locate each code's
    distance to its quantization boundary."""
    if p["gamma"] is None:
        return _lin_fwd(a_in, p), {"mode": "plain", "input": a_in}
    dt = a_in.dtype
    nd = a_in.ndim
    if training:
        mean, var = moments(a_in)
        p["running_mean"] *= RUN_MOMENTUM
        p["running_mean"] += (1.0 - RUN_MOMENTUM) * mean
        p["running_var"] *= RUN_MOMENTUM
        p["running_var"] += (1.0 - RUN_MOMENTUM) * var
    else:
        mean, var = p["running_mean"], p["running_var"]
    inv = 1.0 / np.sqrt(var + p["eps"])
    # four separately rounded storage-dtype ops (layer.py:246-249)
    w = np.empty_like(a_in)
    np.subtract(a_in, _b(mean.astype(dt), nd), out=w)
    np.multiply(w, _b(inv.astype(dt), nd), out=w)
    np.multiply(w, _b(p["gamma"], nd), out=w)
    np.add(w, _b(p["beta"], nd), out=w)
    tape = None
    if training:
        tape = {"mode": mode, "sigma2": var, "gamma": p["gamma"].copy(),
                "beta": p["beta"].copy(), "eps": p["eps"],
                "identity": bits is None and mode != "exact"}
        if mode == "exact" or bits is None:
            tape["a2"] = w.copy()
        else:
            tape["q"] = quantize(w, p["gamma"], p["beta"], bits, sigma2=var)
            if keep_a2:
                tape["a2_pre"] = w.copy()
                tape["a_in"] = a_in
            if mode == "naive":
                w = dequantize(tape["q"])
    w = np.maximum(w, dt.type(0))
    return _lin_fwd(w, p), tape


def _decoded(tape):
    return dequantize(tape["q"]) if "q" in tape else tape["a2"].copy()


def bn_input_grad(a1, g1, sigma2, eps, variance_a1=None):
    """layer.py:286-308."""
    dt = g1.dtype
    nd = g1.ndim
    a1v = a1 if variance_a1 is None else variance_a1
    t2 = chan_mean(g1).astype(dt)
    t3 = chan_mean(a1v * g1).astype(dt)
    inv = (1.0 / np.sqrt(sigma2 + eps)).astype(dt)
    out = g1 - _b(t2, nd)
    out = out - a1v * _b(t3, nd)
    return out * _b(inv, nd)


def layer_bwd(g_out, tape, p, need_input_grad=True, variance_a1=None, internals=None):
    """layer.py:311-381; accumulates grads into p, returns g_in."""
    if tape["mode"] == "plain":
        a_in = tape["input"]
        if p["kind"] != "conv":
            p["grad_weight"] += matmul_fixed(a_in.T.copy(), g_out)
            return matmul_fixed(g_out, p["weight"].T.copy()) if need_input_grad else None
        gx, gk = conv_bwd(a_in, p["weight"], g_out, p["stride"], p["pad"], need_input_grad)
        p["grad_weight"] += gk
        return gx
    dt = g_out.dtype
    a3 = _decoded(tape)
    nd = a3.ndim
    mask = a3 > 0
    a3 = np.maximum(a3, dt.type(0))
    g3 = _lin_bwd(a3, g_out, p)
    if internals is not None:
        internals["mask"] = mask.copy()
        internals["grad_linear_in"] = g3.copy()
    a1 = _decoded(tape)
    a1 = (a1 - _b(tape["beta"], nd)) / _b(safe_gamma(tape["gamma"]), nd)
    g3 = g3 * mask
    p["grad_beta"] += chan_sum(g3)
    p["grad_gamma"] += chan_sum(a1 * g3)
    g3 = g3 * _b(tape["gamma"], nd)
    if internals is not None:
        internals["grad_pre_relu"] = g3.copy()
        internals["a1"] = a1.copy()
    if not need_input_grad:
        return None
    return bn_input_grad(a1, g3, tape["sigma2"], tape["eps"], variance_a1)


# --------------------------------------------------------------- engine ---

def net_shapes(spec, batch):
    """Per-layer (in, out) shapes, engine.py:119-138."""
    shapes = []
    cur = (batch,) + tuple(spec["input_shape"])
    for l in spec["layers"]:
        if l["kind"] == "conv":
            out = conv_out_shape(cur, (l["out_channels"], cur[1], l["kernel"], l["kernel"]),
                                 l["stride"], l["pad"])
        else:
            out = (batch, l["out_channels"])
        shapes.append((cur, out))
        cur = out
    return shapes


def net_width(spec):
    """engine.py:140-156."""
    n = len(spec["layers"])
    last = {v: v + 1 for v in range(-1, n - 1)}
    for first, lst in spec["blocks"]:
        last[first - 1] = max(last[first - 1], lst)
    return max([1] + [1 + sum(1 for v in range(-1, i) if last.get(v, -1) > i)
                      for i in range(n)])


def _block_starts_ends(spec):
    return ({b[0]: tuple(b) for b in spec["blocks"]},
            {b[1]: tuple(b) for b in spec["blocks"]})


def _shortcut_add(cur, res):
    """engine.py:262-269."""
    if cur.shape == res.shape:
        return cur + res
    s = res.shape[2] // cur.shape[2]
    out = cur.copy()
    out[:, :res.shape[1]] += res[:, :, ::s, ::s]
    return out


def _shortcut_adj(g_in, g_res):
    """engine.py:272-279."""
    if g_in.shape == g_res.shape:
        return g_in + g_res
    s = g_in.shape[2] // g_res.shape[2]
    out = g_in.copy()
    out[:, :, ::s, ::s] += g_res[:, :g_in.shape[1]]
    return out


def net_fwd(spec, params, batch, mode="exact", bits=8, training=True, keep_a2=False):
    """engine.py:282-329 (values only; pool reuse does not change values)."""
    starts, ends = _block_starts_ends(spec)
    head = len(spec["layers"]) - 1
    cur, res, tapes = batch, None, []
    for i, p in enumerate(params):
        if i in starts:
            res = cur.copy()
        cur, tape = layer_fwd(cur, p, "exact" if i == head else mode, bits, training, keep_a2)
        tapes.append(tape)
        if i in ends:
            cur = _shortcut_add(cur, res)
    return cur.copy(), tapes


def net_bwd(spec, params, tapes, loss_grad):
    """engine.py:332-376."""
    starts, ends = _block_starts_ends(spec)
    g, res_g = loss_grad.copy(), None
    for i in range(len(spec["layers"]) - 1, -1, -1):
        if i in ends:
            res_g = g.copy()
        g = layer_bwd(g, tapes[i], params[i], need_input_grad=(i != 0))
        if i in starts and g is not None:
            g = _shortcut_adj(g, res_g)


# ------------------------------------------------------------- training ---

def softmax_xent(logits, labels):
    """training.py:120-134."""
    n = logits.shape[0]
    z = logits.astype(np.float64)
    z = z - z.max(axis=1, keepdims=True)
    ez = np.exp(z)
    den = ez.sum(axis=1)
    nll = -(z[np.arange(n), labels] - np.log(den))
    grad = ez / ez.sum(axis=1, keepdims=True)
    grad[np.arange(n), labels] -= 1.0
    grad /= n
    return float(nll.mean()), grad.astype(logits.dtype)


def sgd(params, lr, momentum, weight_decay):
    """training.py:98-117 (fp32 in-place arithmetic, then zero grads)."""
    for p in params:
        groups = [("weight", weight_decay)]
        if p["gamma"] is not None:
            groups += [("gamma", 0.0), ("beta", 0.0)]
        for name, wd in groups:
            val, grad, vel = p[name], p["grad_" + name], p["vel_" + name]
            t = val.dtype.type
            vel *= t(momentum)
            vel += (grad + t(wd) * val) if wd else grad
            val -= t(lr) * vel
            grad[...] = 0


def init_params(spec, seed, dtype=np.float32):
    """He init, gamma=1, beta=0 (training.py:64-89)."""
    dtype = np.dtype(dtype)
    rng = np.random.default_rng(seed)
    out = []
    for l, (ins, _) in zip(spec["layers"], net_shapes(spec, 1)):
        cin = ins[1]
        if l["kind"] == "conv":
            fan = cin * l["kernel"] ** 2
            w = rng.standard_normal((l["out_channels"], cin, l["kernel"], l["kernel"]))
        else:
            fan = cin
            w = rng.standard_normal((cin, l["out_channels"]))
        w = (w * np.sqrt(2.0 / fan)).astype(dtype)
        if l.get("preact", True):
            out.append(new_params(l["kind"], w, l["stride"], l["pad"],
                                  np.ones(cin, dtype), np.zeros(cin, dtype)))
        else:
            out.append(new_params(l["kind"], w, l["stride"], l["pad"]))
    return out


def train_step(spec, params, x, labels, mode, bits, lr=0.1, momentum=0.9, wd=2e-4):
    """One iteration of training.py:192-199 (no augmentation)."""
    logits, tapes = net_fwd(spec, params, x, mode, bits)
    loss, g = softmax_xent(logits, labels)
    net_bwd(spec, params, tapes, g)
    sgd(params, lr, momentum, wd)
    return loss, logits, tapes
