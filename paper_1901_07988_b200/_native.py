"""ctypes binding of libqtape_b200.so (include/qtape_b200.h).

Mirrors the reference's FFI pattern (``ctypes.CDLL`` of a native shared
object, /root/reference/pkg/src/qtape/_native.py:45-98) with two deliberate
differences: the library is prebuilt in-tree by ``build.py`` for sm_100a, and
there is NO fallback -- a missing library, a missing GPU or a nonzero status
raises.  Every call is enqueued on the caller's current torch CUDA stream.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

from .errors import StateError, raise_for_status

_SO = Path(__file__).resolve().parent / "libqtape_b200.so"

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int
F32 = ctypes.c_float
F64 = ctypes.c_double


class Tape(ctypes.Structure):
    """qt_tape_t: fp32 pre-ReLU tape or packed codes + frozen constants."""
    _fields_ = [("a2", P), ("codes", P), ("step", P), ("offset", P), ("bits", I32)]


class BnPrologue(ctypes.Structure):
    """qt_bn_prologue_t: BN-apply + ReLU + K-bit tape in the conv operand staging."""
    _fields_ = [("consts", P), ("codes", P), ("clip_count", P), ("bits", I32)]


class BnStatsEpilogue(ctypes.Structure):
    """qt_bn_stats_epilogue_t: the next layer's BN statistics in the conv epilogue."""
    _fields_ = [("eps", F64), ("gamma", P), ("beta", P), ("bits", I32), ("mean", P),
                ("var", P), ("running_mean", P), ("running_var", P), ("gamma_copy", P),
                ("beta_copy", P), ("step", P), ("offset", P), ("clip_count", P),
                ("consts", P), ("ws", P)]


# name -> (restype, argtypes); keep in sync with include/qtape_b200.h
SIGNATURES = {
    "qt_version": (I32, []),
    "qt_error_string": (ctypes.c_char_p, [I32]),
    "qt_num_sms": (I32, []),
    "qt_set_concurrent_backward": (I32, [I32]),
    "qt_codec_constants": (I32, [P, P, I64, I32, P, P, P]),
    "qt_quantize_pack": (I32, [P, I64, I64, I64, P, P, I32, P, P, P, P, P]),
    "qt_unpack_dequant": (I32, [P, I64, I64, I64, I32, P, P, I32, P, P]),
    "qt_pack_codes": (I32, [P, I64, I32, P, P, P]),
    "qt_unpack_codes": (I32, [P, I64, I32, P, P]),
    "qt_bn_stats_workspace": (I64, [I64, I64, I64]),
    "qt_bn_stats": (I32, [P, I64, I64, I64, P, P, P, P, P, P]),
    "qt_channel_sum": (I32, [P, I64, I64, I64, P, P, P]),
    "qt_bn_relu_forward": (I32, [P, I64, I64, I64, P, P, F64, P, P, I32, I32,
                                 P, P, P, P, P, P, P, P]),
    "qt_bn_stats_prep": (I32, [P, I64, I64, I64, F64, P, P, I32, P, P, P, P, P, P, P, P, P,
                               P, P, P]),
    "qt_bn_forward_fused_ok": (I32, [I64, I64, I64]),
    "qt_bn_forward_fused": (I32, [P, I64, I64, I64, F64, P, P, I32, I32, P, P, P, P, P, P, P, P,
                                  P, P, P, P, P, P]),
    "qt_reconstruct": (I32, [Tape, I64, I64, I64, P, P, P, P, P, P]),
    "qt_bn_backward_workspace": (I64, [I64, I64, I64]),
    "qt_bn_backward_reduce": (I32, [P, Tape, I64, I64, I64, P, P, P, F64, P, P, P,
                                    P, P, P]),
    "qt_bn_backward_apply": (I32, [P, Tape, I64, I64, I64, I64, P, P, P, P, P, I64,
                                   I64, P, P, P]),
    "qt_conv_forward": (I32, [P, P, P, I64, I64, I64, I64, I64, I64, I64, I64, I64,
                              P, I64, I64, P, P]),
    "qt_conv_stats_workspace": (I64, [I64]),
    "qt_conv_fused_support": (I32, [I64] * 10 + [I32]),
    "qt_conv_forward_fused": (I32, [P, P, P, I64, I64, I64, I64, I64, I64, I64, I64, I64,
                                    P, I64, I64, ctypes.POINTER(BnPrologue),
                                    ctypes.POINTER(BnStatsEpilogue), P, P]),
    "qt_conv_dgrad": (I32, [P, P, P, I64, I64, I64, I64, I64, I64, I64, I64, I64, P, P]),
    "qt_conv_workspace": (I64, [I64, I64, I64, I64]),
    "qt_conv_workspace_ex": (I64, [I64] * 9),
    "qt_conv_prepare_weights": (I32, [P, I64, I64, P]),
    "qt_conv_uses_tc": (I32, [I64] * 9 + [I32]),
    "qt_conv_wgrad_workspace": (I64, [I64] * 9),
    "qt_conv_wgrad": (I32, [P, Tape, P, P, I64, I64, I64, I64, I64, I64, I64, I64,
                            I64, P, P]),
    "qt_matmul": (I32, [P, P, P, I64, I64, I64, I32, I32, I32, P]),
    "qt_gap": (I32, [P, I64, I64, I64, P, P]),
    "qt_gap_backward": (I32, [P, I64, I64, I64, P, P]),
    "qt_softmax_xent": (I32, [P, P, I64, I64, P, P, P, P]),
    "qt_sgd": (I32, [P, P, P, I64, F32, P, F32, F32, P]),
    "qt_cifar_decode": (I32, [P, I64, P, P, P, P]),
    "qt_standardize": (I32, [P, I64, I64, I64, P, P, P]),
    "qt_gather_augment": (I32, [P, P, I64, I64, I64, I64, P, P, I32, P, P]),
    "qt_copy": (I32, [P, P, I64, P]),
    "qt_shortcut_add": (I32, [P, P, I64, I64, I64, I64, I64, I64, P]),
    "qt_shortcut_adjoint": (I32, [P, P, I64, I64, I64, I64, I64, I64, P]),
}

# kernels launched per call (for the bench's gpu_launches claim)
LAUNCHES_PER_CALL = {"qt_conv_wgrad": 2, "qt_bn_relu_forward": 1}
launch_count = [0]
# optional instrumentation hook: object with before(name, args) / after(name, args)
hook = None

_lib = None


def lib():
    """Load (once) the in-tree CUDA library; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    from . import build as _build
    if not _build.is_current():
        # stale or missing: rebuild in-tree when nvcc is available, else fail
        try:
            _build.build()
        except Exception as exc:  # noqa: BLE001
            if not _SO.exists():
                raise StateError(
                    f"{_SO.name} is not built and the build failed ({exc}); "
                    "there is no CPU fallback") from exc
            raise StateError(f"{_SO.name} is stale and could not be rebuilt: {exc}") from exc
    so = ctypes.CDLL(str(_SO))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(so, name)
        fn.restype = res
        fn.argtypes = args
    _lib = so
    return _lib


def library_path() -> str:
    return str(_SO)


def exported_symbols():
    return list(SIGNATURES)


def require_cuda(t: torch.Tensor, name: str = "tensor") -> None:
    if not t.is_cuda:
        raise StateError(f"{name} must be a CUDA tensor (no CPU path)")


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def call(name: str, *args) -> None:
    """Invoke qt_<name> with the current stream appended; raise on error."""
    L = lib()
    fn = getattr(L, name)
    h = hook
    if h is not None:
        h.before(name, args)
    status = fn(*args, stream())
    if h is not None:
        h.after(name, args)
    launch_count[0] += LAUNCHES_PER_CALL.get(name, 1)
    if status:
        msg = L.qt_error_string(status)
        raise_for_status(status, name, msg.decode() if msg else "")


def query(name: str, *args) -> int:
    """Invoke a host-side size query (no stream argument)."""
    return int(getattr(lib(), name)(*args))


def make_tape(a2=None, codes=None, step=None, offset=None, bits=0) -> Tape:
    return Tape(ptr(a2), ptr(codes), ptr(step), ptr(offset), int(bits or 0))


def debug_sync() -> None:
    """QTAPE_SYNC=1: synchronise after every call (error localisation)."""
    if os.environ.get("QTAPE_SYNC"):
        torch.cuda.synchronize()
