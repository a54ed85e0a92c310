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
