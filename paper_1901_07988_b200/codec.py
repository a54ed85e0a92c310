"""K-bit per-channel activation codec on the GPU (drop-in for qtape.codec).

Same public names and semantics as /root/reference/pkg/src/qtape/codec.py:
clip to beta +/- 3|gamma|, 2^K uniform intervals, decode to the interval
median with constants frozen at encode time, codes bit-packed little-endian
in flat NCHW order.  Tensors are ``torch.cuda`` float32; the packed bytes are
byte-identical to the reference's ``pack_codes`` output.  All arithmetic runs
in the CUDA library (csrc/codec.cu); nothing here computes on the host.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import torch

from . import _native as N
from .errors import CodecError, ConfigError, ShapeError

SUPPORTED_BITS = (1, 2, 4, 8)       # codec.py:20
GAMMA_FLOOR = 1e-8                  # codec.py:24


def _check_bits(bits):
    if bits not in SUPPORTED_BITS:
        raise ConfigError(f"bits must be one of {SUPPORTED_BITS}, got {bits}")


def _nch_hw(shape):
    """(n, c, hw) view of a rank-2 (N,C) or rank-4 (N,C,H,W) shape."""
    if len(shape) == 2:
        return int(shape[0]), int(shape[1]), 1
    if len(shape) == 4:
        return int(shape[0]), int(shape[1]), int(shape[2]) * int(shape[3])
    raise ShapeError(f"expected rank 2 or 4 tensor, got rank {len(shape)}")


def _f32(t, name):
    if not isinstance(t, torch.Tensor):
        raise ShapeError(f"{name} must be a torch tensor")
    N.require_cuda(t, name)
    if t.dtype != torch.float32:
        raise ConfigError(f"{name} must be float32 (got {t.dtype})")
    return t.contiguous()


def gamma_magnitude(gamma: torch.Tensor) -> torch.Tensor:
    """|gamma| floored away from zero, float64 (codec.py:27-29)."""
    return torch.clamp_min(gamma.double().abs(), GAMMA_FLOOR)


@dataclass
class QuantizedTape:
    """Packed K-bit codes plus frozen decode constants, all device-resident.

    Mirrors codec.QuantizedTape (codec.py:32-56).  ``clip_count`` is kept as
    a device int64 counter and read lazily (reading it synchronises).
    """

    codes: torch.Tensor              # uint8, ceil(K*numel/8) bytes
    bits: int
    shape: tuple
    dtype: torch.dtype
    step: torch.Tensor               # float64 [C]
    offset: torch.Tensor             # int64 [C]
    sigma2: torch.Tensor             # float64 [C]
    clip_counter: torch.Tensor = field(repr=False, default=None)  # int64 [1]

    @property
    def numel(self) -> int:
        n = 1
        for s in self.shape:
            n *= int(s)
        return n

    @property
    def clip_count(self) -> int:
        return int(self.clip_counter.item()) if self.clip_counter is not None else 0

    def nbytes_codes(self) -> int:
        return int(self.codes.numel())

    def as_native(self):
        return N.make_tape(codes=self.codes, step=self.step, offset=self.offset, bits=self.bits)


def packed_nbytes(count: int, bits: int) -> int:
    return (int(count) * int(bits) + 7) // 8


def pack_codes(codes: torch.Tensor, bits: int) -> torch.Tensor:
    """Pack integer codes < 2^bits (codec.py:59-78); CodecError if out of range."""
    _check_bits(bits)
    N.require_cuda(codes, "codes")
    c = codes.reshape(-1)
    if c.dtype != torch.uint8:
        if c.numel() and (int(c.min()) < 0 or int(c.max()) >= (1 << bits)):
            raise CodecError(f"code out of range for {bits}-bit packing")
        c = c.to(torch.uint8)
    c = c.contiguous()
    out = torch.empty(packed_nbytes(c.numel(), bits), dtype=torch.uint8, device=c.device)
    bad = torch.zeros(1, dtype=torch.int32, device=c.device)
    N.call("qt_pack_codes", N.ptr(c), c.numel(), bits, N.ptr(out), N.ptr(bad))
    if int(bad.item()):
        raise CodecError(f"code out of range for {bits}-bit packing")
    return out


def unpack_codes(packed: torch.Tensor, bits: int, count: int) -> torch.Tensor:
    """Inverse of pack_codes (codec.py:81-98); CodecError on a wrong byte count."""
    _check_bits(bits)
    N.require_cuda(packed, "packed")
    p = packed.reshape(-1).contiguous()
    expected = packed_nbytes(count, bits)
    if p.numel() != expected:
        raise CodecError(f"need {expected} bytes for {count} {bits}-bit codes, got {p.numel()}")
    out = torch.empty(int(count), dtype=torch.uint8, device=p.device)
    N.call("qt_unpack_codes", N.ptr(p), int(count), bits, N.ptr(out))
    return out


def codec_constants(gamma: torch.Tensor, beta: torch.Tensor, bits: int):
    """(step float64[C], offset int64[C]) -- codec._scales + offset (codec.py:101-117)."""
    _check_bits(bits)
    gamma, beta = _f32(gamma, "gamma"), _f32(beta, "beta")
    c = gamma.numel()
    step = torch.empty(c, dtype=torch.float64, device=gamma.device)
    offset = torch.empty(c, dtype=torch.int64, device=gamma.device)
    N.call("qt_codec_constants", N.ptr(gamma), N.ptr(beta), c, bits, N.ptr(step), N.ptr(offset))
    return step, offset


def raw_codes(a: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, bits: int) -> torch.Tensor:
    """Unclipped int64 codes (codec.py:107-120) -- diagnostics helper.

    Evaluated on the device in float64 with torch ops (not on the hot path;
    the hot path computes codes inside csrc/codec.cu)."""
    _check_bits(bits)
    scale = (2.0 ** bits) / (6.0 * gamma_magnitude(gamma))
    shp = (1, -1) + (1,) * (a.dim() - 2)
    off = torch.floor(beta.double() * scale)
    u = torch.floor(a.double() * scale.reshape(shp))

    def cast(x):  # x86 numpy int64 cast: out-of-range / NaN -> INT64_MIN
        ok = torch.isfinite(x) & (x >= -2.0 ** 63) & (x < 2.0 ** 63)
        return torch.where(ok, x, torch.zeros_like(x)).to(torch.int64).masked_fill(
            ~ok, -2 ** 63)

    return cast(u) + (1 << (bits - 1)) - cast(off).reshape(shp)


def quantize(a: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, bits: int,
             sigma2: Optional[torch.Tensor] = None, codes_out: Optional[torch.Tensor] = None
             ) -> QuantizedTape:
    """Encode a tensor into a K-bit tape with frozen constants (codec.py:123-143)."""
    _check_bits(bits)
    a = _f32(a, "a")
    n, c, hw = _nch_hw(a.shape)
    if gamma.numel() != c or beta.numel() != c:
        raise ConfigError(f"gamma/beta length must match channel extent {c}")
    gamma, beta = _f32(gamma, "gamma"), _f32(beta, "beta")
    dev = a.device
    nbytes = packed_nbytes(a.numel(), bits)
    codes = codes_out if codes_out is not None else torch.empty(nbytes, dtype=torch.uint8, device=dev)
    step = torch.empty(c, dtype=torch.float64, device=dev)
    offset = torch.empty(c, dtype=torch.int64, device=dev)
    clip = torch.zeros(1, dtype=torch.int64, device=dev)
    N.call("qt_quantize_pack", N.ptr(a), n, c, hw, N.ptr(gamma), N.ptr(beta), bits,
           N.ptr(codes), N.ptr(step), N.ptr(offset), N.ptr(clip))
    s2 = (torch.zeros(c, dtype=torch.float64, device=dev) if sigma2 is None
          else sigma2.to(device=dev, dtype=torch.float64))
    return QuantizedTape(codes=codes, bits=bits, shape=tuple(a.shape), dtype=a.dtype, step=step,
                         offset=offset, sigma2=s2, clip_counter=clip)


def dequantize(t: QuantizedTape, out: Optional[torch.Tensor] = None, relu: bool = False
               ) -> torch.Tensor:
    """Decode a tape to interval medians with its frozen constants (codec.py:146-156)."""
    n, c, hw = _nch_hw(t.shape)
    if t.codes.numel() != packed_nbytes(t.numel, t.bits):
        raise CodecError("tape byte count does not match its shape")
    if out is None:
        out = torch.empty(t.shape, dtype=torch.float32, device=t.codes.device)
    elif tuple(out.shape) != tuple(t.shape) or not out.is_contiguous():
        raise ShapeError("out must be contiguous with the tape's shape")
    N.call("qt_unpack_dequant", N.ptr(t.codes), n, c, hw, t.bits, N.ptr(t.step),
           N.ptr(t.offset), int(relu), N.ptr(out))
    return out


def error_bound(gamma: torch.Tensor, bits: int) -> torch.Tensor:
    """Worst-case absolute error for unclipped entries, 3|gamma|2^-K (codec.py:159-162)."""
    return 3.0 * gamma_magnitude(gamma) * (2.0 ** -bits)


def decode_threshold(t: QuantizedTape) -> torch.Tensor:
    """Smallest code decoding to a positive value, per channel (codec.py:165-173)."""
    return ((1 << (t.bits - 1)) - t.offset).to(torch.int64)
