"""Codec parity on the GPU: bit-exact against the reference's golden
vectors (tests/golden/codec.npz) and the oracle restatement."""

import numpy as np
import pytest
import torch

import oracle as O
from gpu_util import dev, host

pytestmark = pytest.mark.gpu

from paper_1901_07988_b200 import codec as Q  # noqa: E402
from paper_1901_07988_b200.errors import CodecError, ConfigError  # noqa: E402


def one_channel(values, gamma=1.0, beta=0.0, bits=4):
    a = dev(np.asarray(values, np.float32).reshape(1, 1, -1, 1))
    return Q.quantize(a, dev(np.array([gamma], np.float32)), dev(np.array([beta], np.float32)),
                      bits)


def codes_of(t):
    return host(Q.unpack_codes(t.codes, t.bits, t.numel))


def test_known_answers():
    # reference tests/test_quantize.py:20-87
    t = one_channel([0.1])
    assert codes_of(t)[0] == 8 and t.clip_count == 0
    t = one_channel([10.0])
    assert codes_of(t)[0] == 15 and t.clip_count == 1
    assert codes_of(one_channel([-0.01], bits=8))[0] == 127
    assert host(Q.dequantize(one_channel([0.1])))[0, 0, 0, 0] == np.float32(0.1875)
    assert host(Q.dequantize(one_channel([10.0])))[0, 0, 0, 0] == np.float32(2.8125)
    assert host(Q.dequantize(one_channel([-0.01], bits=8)))[0, 0, 0, 0] == np.float32(-0.01171875)
    t = one_channel([0.5], gamma=0.0)
    assert host(t.step)[0] == pytest.approx(6e-8 / 16)
    assert host(Q.pack_codes(dev(np.array([3, 7, 0, 15], np.uint8)), 4)).tolist() == [0x73, 0xF0]
    assert host(Q.pack_codes(dev(np.array([1, 0, 1, 1, 0, 0, 0, 0], np.uint8)), 1)).tolist() == [0x0D]
    assert host(Q.pack_codes(dev(np.array([1, 2, 3, 0, 3], np.uint8)), 2)).tolist() == [0x39, 0x03]
    assert host(Q.unpack_codes(dev(np.array([0x73, 0xF0], np.uint8)), 4, 4)).tolist() == [3, 7, 0, 15]


def test_errors():
    with pytest.raises(ConfigError):
        one_channel([0.0], bits=3)
    with pytest.raises(CodecError):
        Q.pack_codes(dev(np.array([4], np.uint8)), 2)
    with pytest.raises(CodecError):
        Q.unpack_codes(dev(np.zeros(3, np.uint8)), 4, 4)


def test_golden_vectors_bit_exact(golden_codec):
    g = golden_codec
    for i in range(int(g["n_codec"])):
        k = f"c{i}"
        bits = int(g[k + "_bits"])
        t = Q.quantize(dev(g[k + "_a"]), dev(g[k + "_gamma"]), dev(g[k + "_beta"]), bits)
        assert np.array_equal(host(t.codes), g[k + "_codes"]), k
        assert np.array_equal(host(t.step), g[k + "_step"]), k
        assert np.array_equal(host(t.offset), g[k + "_offset"]), k
        assert t.clip_count == int(g[k + "_clip"]), k
        d = host(Q.dequantize(t))
        assert np.array_equal(d.view(np.uint32), g[k + "_deq"].view(np.uint32)), k


@pytest.mark.parametrize("bits", [1, 2, 4, 8])
@pytest.mark.parametrize("shape", [(3, 5, 7, 7), (2, 16, 32, 32), (5, 3, 1, 1), (7, 13),
                                   (1, 1, 3, 3), (4, 64, 8, 8)])
def test_random_vs_oracle(bits, shape):
    rng = np.random.default_rng(hash((bits,) + shape) % 2**32)
    c = shape[1]
    a = (rng.standard_normal(shape) * 3 + 1).astype(np.float32)
    gamma = rng.uniform(0.5, 2.0, c).astype(np.float32)
    beta = rng.uniform(-1, 1, c).astype(np.float32)
    want = O.quantize(a, gamma, beta, bits)
    t = Q.quantize(dev(a), dev(gamma), dev(beta), bits)
    assert np.array_equal(host(t.codes), want["codes"])
    assert t.clip_count == want["clip_count"]
    assert np.array_equal(host(Q.dequantize(t)), O.dequantize(want))
    relu = host(Q.dequantize(t, relu=True))
    assert np.array_equal(relu, np.maximum(O.dequantize(want), np.float32(0)))


def test_edge_values():
    # NaN / inf / huge / subnormal follow x86 numpy's int64 cast
    vals = np.array([np.nan, np.inf, -np.inf, 1e19, -1e19, 5e18, np.float32(-1.4e-45),
                     np.float32(1.4e-45), -0.0, 0.0, 3.0, -3.0], np.float32)
    for bits in (1, 2, 4, 8):
        a = vals.reshape(1, 1, -1, 1)
        want = O.quantize(a, np.ones(1, np.float32), np.zeros(1, np.float32), bits)
        t = Q.quantize(dev(a), dev(np.ones(1, np.float32)), dev(np.zeros(1, np.float32)), bits)
        assert np.array_equal(host(t.codes), want["codes"]), bits
        assert t.clip_count == want["clip_count"], bits


@pytest.mark.parametrize("bits", [1, 2, 4, 8])
def test_pack_roundtrip(bits):
    rng = np.random.default_rng(bits)
    codes = rng.integers(0, 1 << bits, size=1237).astype(np.uint8)
    p = Q.pack_codes(dev(codes), bits)
    assert np.array_equal(host(p), O.pack(codes, bits))
    assert np.array_equal(host(Q.unpack_codes(p, bits, 1237)), codes)


def test_frozen_constants():
    a = dev(np.linspace(-2, 2, 16, dtype=np.float32).reshape(1, 1, 4, 4))
    gamma, beta = dev(np.array([0.8], np.float32)), dev(np.array([0.3], np.float32))
    t = Q.quantize(a, gamma, beta, 8)
    before = host(Q.dequantize(t))
    gamma.fill_(99.0)
    beta.fill_(-5.0)
    assert np.array_equal(host(Q.dequantize(t)), before)


def test_storage_size():
    for bits in (1, 2, 4, 8):
        t = Q.quantize(torch.zeros((3, 2, 5, 7), device="cuda"), torch.ones(2, device="cuda"),
                       torch.zeros(2, device="cuda"), bits)
        assert t.nbytes_codes() == (bits * 210 + 7) // 8


def test_large_tensor_roundtrip_property():
    """Size-independent property at a C2-sized layer: unclipped decode error
    <= 3|gamma|2^-K with the sign preserved (test_acceptance.py:85-95)."""
    rng = np.random.default_rng(7)
    shape = (128, 64, 32, 32)
    c = shape[1]
    gamma = rng.uniform(0.5, 2.0, c).astype(np.float32)
    beta = rng.uniform(-1, 1, c).astype(np.float32)
    a = (torch.randn(shape, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
         * 3 + 1)
    g, b = dev(gamma), dev(beta)
    for bits in (2, 4, 8):
        t = Q.quantize(a, g, b, bits)
        d = Q.dequantize(t)
        raw = Q.raw_codes(a, g, b, bits)
        unclipped = (raw >= 0) & (raw <= (1 << bits) - 1)
        bound = Q.error_bound(g, bits).reshape(1, -1, 1, 1).float()
        err = (d - a).abs()
        # decoded values are rounded to fp32: allow that rounding on top of the bound
        assert bool(((err <= bound + 1e-6 * (a.abs() + 1)) | ~unclipped).all())
        sg = (a >= 0) == (d >= 0)
        assert bool((sg | ~unclipped).all())
        assert t.clip_count == int((~unclipped).sum())


@pytest.mark.parametrize("hw", [64, 196, 12, 4])
@pytest.mark.parametrize("bits", [1, 2, 4, 8])
def test_stream_kernel_codes_at_interval_boundaries(bits, hw):
    """The fused BN-apply + quantize stream kernel (per-channel constant table,
    fp32 fast path for floor(a*scale) with a float64 fallback near integers)
    against the oracle at exact code boundaries k*step, their fp32
    neighbours, huge / non-finite / subnormal values and tiny gammas, on
    planes of hw % 8 == 0 and hw % 8 == 4 pixels."""
    from paper_1901_07988_b200 import _native as N
    rng = np.random.default_rng(bits)
    n, c = 3, 6   # hw % 8 == 4: 8-element groups straddle two channels
    gamma = np.array([1.0, 0.37, -2.5, 1e-9, 0.0, 3.0], np.float32)
    beta = np.array([0.0, 0.11, -0.7, 0.2, 1e-3, 25.0], np.float32)
    scale, step, off = O.code_constants(gamma, beta, bits)
    x = np.empty((n, c, hw), np.float32)
    for ch in range(c):
        k = rng.integers(-(1 << bits) - 4, (1 << bits) + 4, n * hw).astype(np.float64)
        base = ((k + off[ch] - (1 << (bits - 1))) / scale[ch]).astype(np.float32)   # a*scale ~ k
        jitter = rng.integers(-2, 3, n * hw)
        vals = np.nextafter(base, np.where(jitter > 0, np.inf, -np.inf).astype(np.float32))
        vals = np.where(jitter == 0, base, vals)
        vals[:12] = [np.nan, np.inf, -np.inf, 1e30, -1e30, 1.4e-45, -1.4e-45, 0.0, -0.0,
                     5e18, -5e18, 3.4e38]
        x[:, ch, :] = vals.reshape(n, hw)
    # constants with mean 0, inv 1: A2 = x*gamma + beta in fp32 (layer.py:246-249)
    ct = np.zeros(c, dtype=[("m32", "<f4"), ("inv32", "<f4"), ("g", "<f4"), ("b", "<f4"),
                            ("scale", "<f8"), ("step", "<f8"), ("off", "<i8"), ("s1", "<f4"),
                            ("s2", "<f4")])
    ct["inv32"], ct["g"], ct["b"] = 1.0, gamma, beta
    ct["scale"], ct["step"], ct["off"] = scale, step, off
    ct["s1"] = scale.astype(np.float32)
    ct["s2"] = (scale - ct["s1"].astype(np.float64)).astype(np.float32)
    assert ct.dtype.itemsize == 48
    with np.errstate(invalid="ignore", over="ignore"):
        a2 = (((x - np.float32(0)) * np.float32(1)) * gamma[None, :, None]) + beta[None, :, None]
        raw = O.raw_codes(a2, gamma, beta, bits)
    codes_ref = O.pack(np.clip(raw, 0, (1 << bits) - 1), bits)
    clips_ref = int(((raw < 0) | (raw > (1 << bits) - 1)).sum())
    xd, consts = dev(x), torch.from_numpy(ct.view(np.uint8).copy()).cuda()
    a3 = torch.empty_like(xd)
    codes = torch.empty((bits * x.size + 7) // 8, dtype=torch.uint8, device="cuda")
    stp = torch.empty(c, dtype=torch.float64, device="cuda")
    offd = torch.empty(c, dtype=torch.int64, device="cuda")
    clip = torch.zeros(1, dtype=torch.int64, device="cuda")
    dummy = torch.zeros(c, dtype=torch.float64, device="cuda")
    gd, bd = dev(gamma), dev(beta)
    N.call("qt_bn_relu_forward", N.ptr(xd), n, c, hw, N.ptr(dummy), N.ptr(dummy), 1e-5,
           N.ptr(gd), N.ptr(bd), 1, bits, N.ptr(a3), None, N.ptr(codes), N.ptr(stp), N.ptr(offd),
           N.ptr(clip), N.ptr(consts))
    assert np.array_equal(host(codes), codes_ref)
    assert int(clip.item()) == clips_ref
    with np.errstate(invalid="ignore"):
        assert np.array_equal(host(a3), np.maximum(a2, np.float32(0)), equal_nan=True)
