"""Conv / matmul / moment parity against the oracle (tolerances in gpu_util)."""

import numpy as np
import pytest
import torch

import oracle as O
from gpu_util import CONV_TOL, MOMENT_TOL, dev, host, norm_err

pytestmark = pytest.mark.gpu

from paper_1901_07988_b200 import ops  # noqa: E402
from paper_1901_07988_b200.errors import ShapeError  # noqa: E402

GEOS = [  # (n, ci, h, co, k, s, p)
    (2, 3, 9, 4, 3, 1, 1), (2, 5, 8, 6, 3, 1, 1), (3, 4, 8, 8, 2, 2, 0), (2, 16, 8, 16, 1, 1, 0),
    (2, 3, 16, 8, 4, 4, 0), (2, 8, 7, 5, 3, 2, 0), (1, 32, 16, 64, 1, 1, 0), (4, 64, 8, 16, 1, 1, 0),
    (2, 16, 16, 16, 3, 1, 1), (2, 12, 14, 24, 2, 2, 0), (3, 7, 5, 9, 3, 1, 2), (2, 4, 12, 4, 4, 2, 1),
    # tensor-core (tcgen05) shapes: rows of 8/16/32 px, ci % 8 == 0, co % 16 == 0
    (4, 16, 32, 16, 3, 1, 1), (2, 32, 32, 64, 1, 1, 0), (2, 64, 8, 256, 1, 1, 0),
    (4, 256, 8, 64, 1, 1, 0), (2, 64, 8, 64, 3, 1, 1), (2, 128, 16, 32, 1, 1, 0),
    (2, 32, 16, 32, 3, 1, 1), (2, 16, 32, 64, 1, 1, 0), (6, 8, 8, 16, 3, 1, 1),
    # kernel == stride transitions: space-to-depth + tensor-core 1x1
    (2, 32, 32, 32, 2, 2, 0), (4, 64, 16, 64, 2, 2, 0),
    # 1x1 on any plane (flattened 128-pixel runs; last run partial): ImageNet
    # widths 56/28/14, a 12-wide plane, 7x7 (SIMT: plane not 16-byte aligned),
    # and the 4x4/s4 stem / 2x2/s2 transitions landing on them via s2d
    (2, 64, 14, 32, 1, 1, 0), (2, 32, 28, 64, 1, 1, 0), (1, 16, 56, 16, 1, 1, 0),
    (3, 48, 12, 16, 1, 1, 0), (2, 32, 7, 32, 1, 1, 0), (2, 16, 56, 32, 2, 2, 0),
    (1, 3, 64, 16, 4, 4, 0),
    # 3x3 "same" convs on other plane widths: segmented copy (rows padded to
    # 8/16/32 px, or 30-column segments with a one-column halo above 32 px)
    # + tensor-core rows: ImageNet 56/28/14/7, odd widths, an odd batch
    (2, 16, 56, 16, 3, 1, 1), (2, 32, 28, 32, 3, 1, 1), (2, 64, 14, 32, 3, 1, 1),
    (2, 64, 7, 64, 3, 1, 1), (3, 16, 7, 16, 3, 1, 1), (1, 16, 40, 32, 3, 1, 1),
    (2, 16, 3, 16, 3, 1, 1), (1, 32, 61, 16, 3, 1, 1),
    # kernel == stride convs whose (space-to-depth) plane is not 16-byte
    # aligned (7x7 = 49 px): zero-padded flat plane + tensor-core 1x1
    (2, 64, 7, 32, 1, 1, 0), (2, 32, 14, 64, 2, 2, 0), (3, 16, 5, 48, 1, 1, 0),
]


def test_tensor_core_path_is_selected():
    from paper_1901_07988_b200 import _native as N
    assert N.query("qt_conv_uses_tc", 128, 16, 32, 32, 16, 3, 3, 1, 1, 0) == 1
    assert N.query("qt_conv_uses_tc", 128, 16, 32, 32, 16, 3, 3, 1, 1, 1) == 1
    assert N.query("qt_conv_uses_tc", 128, 64, 8, 8, 256, 1, 1, 1, 0, 0) == 1
    assert N.query("qt_conv_uses_tc", 128, 3, 32, 32, 16, 3, 3, 1, 1, 0) == 0   # stem
    assert N.query("qt_conv_uses_tc", 128, 32, 32, 32, 32, 2, 2, 2, 0, 0) == 0  # 2x2/s2


@pytest.mark.parametrize("geo", GEOS)
def test_conv_forward(geo):
    n, ci, h, co, k, s, p = geo
    rng = np.random.default_rng(sum(geo))
    x = rng.standard_normal((n, ci, h, h)).astype(np.float32)
    w = rng.standard_normal((co, ci, k, k)).astype(np.float32)
    want = O.conv_fwd(x, w, s, p)
    got = host(ops.conv2d_forward(dev(x), dev(w), s, p))
    assert got.shape == want.shape
    assert norm_err(got, want) < CONV_TOL


@pytest.mark.parametrize("geo", GEOS)
def test_conv_backward(geo):
    n, ci, h, co, k, s, p = geo
    rng = np.random.default_rng(100 + sum(geo))
    x = rng.standard_normal((n, ci, h, h)).astype(np.float32)
    w = rng.standard_normal((co, ci, k, k)).astype(np.float32)
    g = rng.standard_normal(O.conv_out_shape(x.shape, w.shape, s, p)).astype(np.float32)
    gx_w, gk_w = O.conv_bwd(x, w, g, s, p)
    gx, gk = ops.conv2d_backward(dev(x), dev(w), dev(g), s, p)
    assert norm_err(host(gx), gx_w) < CONV_TOL
    assert norm_err(host(gk), gk_w) < CONV_TOL
    none, gk2 = ops.conv2d_backward(dev(x), dev(w), dev(g), s, p, need_g_x=False)
    assert none is None and np.array_equal(host(gk2), host(gk))


def test_conv_adjoint_identity():
    rng = np.random.default_rng(3)
    x = dev(rng.standard_normal((2, 3, 8, 8)).astype(np.float32))
    w = dev(rng.standard_normal((4, 3, 3, 3)).astype(np.float32))
    y = dev(rng.standard_normal((2, 4, 8, 8)).astype(np.float32))
    gx, _ = ops.conv2d_backward(x, w, y, 1, 1)
    lhs = float((ops.conv2d_forward(x, w, 1, 1).double() * y.double()).sum())
    rhs = float((x.double() * gx.double()).sum())
    assert abs(lhs - rhs) / abs(lhs) < 1e-5


def test_conv_residual_fused():
    rng = np.random.default_rng(4)
    x = rng.standard_normal((2, 8, 8, 8)).astype(np.float32)
    w = rng.standard_normal((16, 8, 2, 2)).astype(np.float32)
    res = rng.standard_normal((2, 4, 8, 8)).astype(np.float32)
    y = O.conv_fwd(x, w, 2, 0)
    want = y.copy()
    want[:, :4] += res[:, :, ::2, ::2]
    got = host(ops.conv2d_forward(dev(x), dev(w), 2, 0, residual=dev(res)))
    assert norm_err(got, want) < CONV_TOL


@pytest.mark.parametrize("geo", [(2, 16, 28, 32, 1), (2, 32, 14, 64, 2), (2, 16, 56, 32, 2)])
def test_conv_residual_flat_1x1(geo):
    _residual_case(geo, 1)


@pytest.mark.parametrize("geo", [(2, 16, 56, 32, 1), (2, 32, 14, 32, 2), (2, 16, 7, 16, 1)])
def test_conv_residual_segmented_3x3(geo):
    """Residual add in the unsegment pass of the segmented 3x3 path."""
    _residual_case(geo, 3)


def _residual_case(geo, k):
    """Residual add on the flattened 1x1 path: same-resolution (fused, one TMA
    box per 128-pixel run) and strided (standalone add after the conv)."""
    n, ci, h, co, sr = geo
    rng = np.random.default_rng(sum(geo))
    x = rng.standard_normal((n, ci, h, h)).astype(np.float32)
    w = rng.standard_normal((co, ci, k, k)).astype(np.float32)
    cr = co // 2
    res = rng.standard_normal((n, cr, h * sr, h * sr)).astype(np.float32)
    want = O.conv_fwd(x, w, 1, k // 2)
    want[:, :cr] += res[:, :, ::sr, ::sr]
    got = host(ops.conv2d_forward(dev(x), dev(w), 1, k // 2, residual=dev(res)))
    assert norm_err(got, want) < CONV_TOL


def test_shape_errors():
    with pytest.raises(ShapeError):
        ops.conv2d_forward(torch.zeros((1, 3, 8, 8), device="cuda"),
                           torch.zeros((4, 3, 3, 3), device="cuda"), 2, 1)
    with pytest.raises(ShapeError):
        ops.conv2d_forward(torch.zeros((1, 3, 8, 8), device="cuda"),
                           torch.zeros((4, 2, 3, 3), device="cuda"), 1, 1)


@pytest.mark.parametrize("shape", [(5, 7, 3), (64, 256, 10), (16, 2048, 1000), (1, 1, 1)])
def test_matmul_bit_exact(shape):
    n, k, m = shape
    rng = np.random.default_rng(n + k + m)
    a = rng.standard_normal((n, k)).astype(np.float32)
    b = rng.standard_normal((k, m)).astype(np.float32)
    got = host(ops.matmul(dev(a), dev(b)))
    assert np.array_equal(got, O.matmul_fixed(a, b))
    # transposed operands read in place
    assert np.array_equal(host(ops.matmul(dev(a.T.copy()), dev(b), ta=True)), got)
    assert np.array_equal(host(ops.matmul(dev(a), dev(b.T.copy()), tb=True)), got)


@pytest.mark.parametrize("shape", [(8, 4, 12, 12), (128, 64, 8, 8), (6, 7), (3, 5, 7, 7),
                                   (2, 16, 112, 112)])
def test_moments(shape):
    rng = np.random.default_rng(len(shape))
    x = (rng.standard_normal(shape) * 3 + 1).astype(np.float32)
    m, v = ops.channel_moments(dev(x))
    mw, vw = O.moments(x)
    assert np.max(np.abs(host(m) - mw) / (np.abs(mw) + 1e-3)) < MOMENT_TOL
    assert np.max(np.abs(host(v) - vw) / vw) < MOMENT_TOL
    s = host(ops.channel_sum(dev(x)))
    assert np.max(np.abs(s - O.chan_sum(x)) / (np.abs(O.chan_sum(x)) + 1)) < 1e-12


def test_moments_constant_and_two_point():
    x = torch.full((4, 3, 5, 5), 2.5, device="cuda")
    m, v = ops.channel_moments(x)
    assert np.all(host(m) == 2.5) and np.all(host(v) == 0.0)
    x = dev(np.array([[1.0], [3.0]], np.float32))
    m, v = ops.channel_moments(x)
    assert host(m)[0] == 2.0 and host(v)[0] == 1.0


def test_prepared_weights_match_per_call_preparation():
    """qt_conv_prepare_weights (one launch for many layers) + w == NULL gives
    the same bits as the per-call re-layout, forward and data gradient."""
    from paper_1901_07988_b200 import _native as N
    rng = np.random.default_rng(3)
    cases = [(2, 16, 32, 16, 3, 1), (2, 64, 8, 256, 1, 0), (2, 32, 16, 32, 3, 1)]
    descs, keep = [], []
    for n, ci, h, co, k, p in cases:
        w = dev((rng.standard_normal((co, ci, k, k)) * 0.2).astype(np.float32))
        pf = torch.empty(2 * w.numel(), dtype=torch.float32, device="cuda")
        pd = torch.empty(2 * w.numel(), dtype=torch.float32, device="cuda")
        descs += [(w.data_ptr(), pf.data_ptr(), co, ci, k, k, 0, 0),
                  (w.data_ptr(), pd.data_ptr(), ci, co, k, k, 1, 0)]
        keep.append((w, pf, pd))
    dt = np.dtype([("w", "<u8"), ("out", "<u8"), ("rows", "<i4"), ("cols", "<i4"),
                   ("kh", "<i4"), ("kw", "<i4"), ("flip", "<i4"), ("pad", "<i4")])
    assert dt.itemsize == 40
    d = torch.from_numpy(np.array(descs, dtype=dt).view(np.uint8).copy()).cuda()
    N.call("qt_conv_prepare_weights", N.ptr(d), len(descs), max(w.numel() for w, _, _ in keep))
    for (n, ci, h, co, k, p), (w, pf, pd) in zip(cases, keep):
        x = dev(rng.standard_normal((n, ci, h, h)).astype(np.float32))
        a = ops.conv2d_forward(x, w, 1, p)
        b = ops.conv2d_forward(x, w, 1, p, prepared=pf)
        assert torch.equal(a, b)
        g = dev(rng.standard_normal(tuple(a.shape)).astype(np.float32))
        ga, gb = torch.empty_like(x), torch.empty_like(x)
        ops.conv2d_dgrad(g, w, tuple(x.shape), 1, p, ga)
        ops.conv2d_dgrad(g, w, tuple(x.shape), 1, p, gb, prepared=pd)
        assert torch.equal(ga, gb)


def test_wgrad_column_tap_form_matches(tmp_path):
    """The opt-in 3x3 wgrad with the column taps in N (QTAPE_WG_TAP=1, read
    once per process) against a float64 reference, FAST and GENERIC CTAs."""
    import os
    import subprocess
    import sys
    code = r'''
import torch
from paper_1901_07988_b200 import codec, ops
torch.manual_seed(0)
for regime in ("narrow", "wide"):
    for n, ci, hw, co in ((2, 16, 32, 16), (2, 32, 16, 32)):
        x = torch.randn(n, ci, hw, hw, device="cuda")
        if regime == "narrow":
            gamma, beta = torch.rand(ci, device="cuda") + 0.5, torch.randn(ci, device="cuda") * 0.1
        else:
            gamma, beta = torch.rand(ci, device="cuda") * 0.05 + 0.05, torch.rand(ci, device="cuda") + 1.5
        t = codec.quantize(x, gamma, beta, 4)
        act = codec.dequantize(t, relu=True)
        g = torch.randn(n, co, hw, hw, device="cuda")
        gw = torch.zeros(co, ci, 3, 3, device="cuda")
        ops.conv2d_wgrad(g, (co, ci, 3, 3), 1, 1, gw, tape=t.as_native(), in_shape=(n, ci, hw, hw))
        ref = torch.nn.grad.conv2d_weight(act.double(), (co, ci, 3, 3), g.double(), padding=1)
        err = ((gw.double() - ref).norm() / ref.norm()).item()
        assert err < 1e-5, (regime, ci, err)
print("ok")
'''
    env = dict(os.environ, QTAPE_WG_TAP="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_wgrad_direct_pieces_form_matches():
    """The opt-in pre-split g_out pieces on unsegmented planes
    (QTAPE_WG_PRE_DIRECT=1, read once per process): 1x1 / 3x3 on 8/16/32-px
    rows and a 56x56 flat plane, 2- and 4-bit tapes, narrow / wide / mixed
    channels, against float64."""
    import os
    import subprocess
    import sys
    code = r'''
import torch
from paper_1901_07988_b200 import codec, ops
torch.manual_seed(1)
for bits in (1, 2, 4):
    for regime in ("narrow", "wide", "mixed"):
        for n, ci, hw, co, k in ((2, 16, 32, 64, 1), (2, 32, 16, 32, 3), (4, 256, 8, 64, 1),
                                 (2, 64, 8, 256, 1), (1, 64, 56, 128, 1)):
            x = torch.randn(n, ci, hw, hw, device="cuda")
            gamma, beta = torch.rand(ci, device="cuda") + 0.5, torch.randn(ci, device="cuda") * 0.1
            if regime != "narrow":
                wide = torch.arange(ci, device="cuda") % (1 if regime == "wide" else 3) == 0
                gamma = torch.where(wide, torch.rand(ci, device="cuda") * 0.05 + 0.05, gamma)
                beta = torch.where(wide, torch.rand(ci, device="cuda") + 1.5, beta)
            t = codec.quantize(x, gamma, beta, bits)
            act = codec.dequantize(t, relu=True)
            g = torch.randn(n, co, hw, hw, device="cuda")
            gw = torch.zeros(co, ci, k, k, device="cuda")
            ops.conv2d_wgrad(g, (co, ci, k, k), 1, k // 2, gw, tape=t.as_native(), in_shape=(n, ci, hw, hw))
            ref = torch.nn.grad.conv2d_weight(act.double(), (co, ci, k, k), g.double(), padding=k // 2)
            err = ((gw.double() - ref).norm() / ref.norm()).item()
            assert err < 1e-5, (bits, regime, ci, co, k, err)
print("ok")
'''
    env = dict(os.environ, QTAPE_WG_PRE_DIRECT="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("bits", [1, 2, 4, 8])
@pytest.mark.parametrize("shape", [(2, 32, 32, 32), (4, 64, 16, 64), (2, 16, 8, 16),
                                   (2, 32, 56, 64), (2, 64, 14, 32), (2, 3, 224, 64, 4),
                                   (2, 3, 32, 16, 4), (2, 48, 28, 32, 4)])
def test_transition_wgrad_from_codes(shape, bits):
    """2x2/s2 weight gradient from a packed tape (rearranged space-to-depth
    codes + the 1x1 tensor-core path where eligible, else the SIMT GEMM)
    against a float64 reference on the dequantized activation."""
    from paper_1901_07988_b200 import codec
    n, ci, hw, co, sd = shape + (2,) if len(shape) == 4 else shape
    torch.manual_seed(bits + ci)
    for regime in ("narrow", "wide"):
        x = torch.randn(n, ci, hw, hw, device="cuda")
        if regime == "narrow":
            gamma, beta = torch.rand(ci, device="cuda") + 0.5, torch.randn(ci, device="cuda") * 0.1
        else:
            gamma, beta = torch.rand(ci, device="cuda") * 0.05 + 0.05, torch.rand(ci, device="cuda") + 1.5
        t = codec.quantize(x, gamma, beta, bits)
        act = codec.dequantize(t, relu=True)
        g = torch.randn(n, co, hw // sd, hw // sd, device="cuda")
        gw = torch.full((co, ci, sd, sd), 0.25, device="cuda")    # accumulates into gw
        ops.conv2d_wgrad(g, (co, ci, sd, sd), sd, 0, gw, tape=t.as_native(), in_shape=(n, ci, hw, hw))
        ref = torch.nn.grad.conv2d_weight(act.double(), (co, ci, sd, sd), g.double(), stride=sd) + 0.25
        err = ((gw.double() - ref).norm() / ref.norm()).item()
        assert err < CONV_TOL, (regime, err)


@pytest.mark.parametrize("shape", [(2, 64, 8, 256, 1), (2, 32, 16, 512, 1), (2, 16, 32, 128, 3),
                                   (2, 64, 8, 320, 1), (2, 16, 56, 32, 1), (1, 64, 24, 64, 1),
                                   (2, 16, 56, 32, 3), (2, 64, 14, 64, 3), (2, 64, 7, 128, 3),
                                   (2, 32, 28, 32, 3), (2, 64, 14, 64, 1), (2, 32, 7, 64, 1),
                                   (2, 16, 28, 32, 1), (2, 256, 14, 256, 1), (2, 128, 7, 256, 3),
                                   (1, 512, 7, 128, 1)])
@pytest.mark.parametrize("bits", [1, 2, 4, 8])
def test_wgrad_from_codes_channel_blocks(shape, bits):
    """Weight gradient from a 2-/4-bit tape for outputs wider than one
    64-channel block (grid z) -- FAST and GENERIC CTAs, and on the segmented
    planes (14/7/28 px) the pre-split g_out pieces path (FAST-PRE and
    GENERIC-PRE) -- against float64."""
    from paper_1901_07988_b200 import codec
    n, ci, hw, co, k = shape
    torch.manual_seed(co + k + bits)
    for regime in ("narrow", "nonpos", "wide", "mixed"):
        x = torch.randn(n, ci, hw, hw, device="cuda")
        gamma, beta = torch.rand(ci, device="cuda") + 0.5, torch.randn(ci, device="cuda") * 0.1
        if regime == "nonpos":   # offsets <= 0: the 8-bit FAST range too (K < 8: 0,
            beta = -beta.abs() if bits == 8 else torch.zeros_like(beta)   # else all decode <= 0)
        elif regime != "narrow":
            wide = torch.arange(ci, device="cuda") % (1 if regime == "wide" else 7) == 0
            gamma = torch.where(wide, torch.rand(ci, device="cuda") * 0.05 + 0.05, gamma)
            beta = torch.where(wide, torch.rand(ci, device="cuda") + 1.5, beta)
        t = codec.quantize(x, gamma, beta, bits)
        act = codec.dequantize(t, relu=True)
        g = torch.randn(n, co, hw, hw, device="cuda")
        gw = torch.zeros(co, ci, k, k, device="cuda")
        ops.conv2d_wgrad(g, (co, ci, k, k), 1, k // 2, gw, tape=t.as_native(), in_shape=(n, ci, hw, hw))
        ref = torch.nn.grad.conv2d_weight(act.double(), (co, ci, k, k), g.double(), padding=k // 2)
        err = ((gw.double() - ref).norm() / ref.norm()).item()
        assert err < CONV_TOL, (regime, err)


@pytest.mark.parametrize("bits", [1, 2, 8])
@pytest.mark.parametrize("shape", [(2, 32, 14, 32), (1, 16, 40, 16), (2, 16, 7, 32)])
def test_segmented_3x3_wgrad_from_codes(shape, bits):
    """3x3 weight gradient on planes of other widths from a packed tape:
    segmented codes (padding pixels = code 0) + the exact padding correction
    for channels whose every code decodes positive ("wide" regime)."""
    from paper_1901_07988_b200 import codec
    n, ci, hw, co = shape
    torch.manual_seed(bits + hw)
    for regime in ("narrow", "wide"):
        x = torch.randn(n, ci, hw, hw, device="cuda")
        if regime == "narrow":
            gamma, beta = torch.rand(ci, device="cuda") + 0.5, torch.randn(ci, device="cuda") * 0.1
        else:
            gamma, beta = torch.rand(ci, device="cuda") * 0.05 + 0.05, torch.rand(ci, device="cuda") + 1.5
        t = codec.quantize(x, gamma, beta, bits)
        act = codec.dequantize(t, relu=True)
        g = torch.randn(n, co, hw, hw, device="cuda")
        gw = torch.full((co, ci, 3, 3), -0.5, device="cuda")
        ops.conv2d_wgrad(g, (co, ci, 3, 3), 1, 1, gw, tape=t.as_native(), in_shape=(n, ci, hw, hw))
        ref = torch.nn.grad.conv2d_weight(act.double(), (co, ci, 3, 3), g.double(), padding=1) - 0.5
        err = ((gw.double() - ref).norm() / ref.norm()).item()
        assert err < CONV_TOL, (regime, err)


@pytest.mark.parametrize("bits", [1, 2, 4, 8])
@pytest.mark.parametrize("shape", [(2, 16, 32, 16, 3), (2, 32, 16, 32, 3), (4, 64, 8, 64, 3),
                                   (2, 16, 32, 64, 1), (2, 64, 8, 256, 1), (4, 128, 16, 32, 1),
                                   (3, 64, 8, 16, 1)])
def test_wgrad_from_codes_row_tiles(shape, bits):
    """Row-tiled (8/16/32-px rows) weight gradient from 1-, 2-, 4- and 8-bit
    tapes: the FAST decode (integer bf16 operand; the 1- and 2-bit forms
    regroup each byte's / halfword's pixel pairs, the 8-bit form pairs bytes
    of two words) for narrow channels (8-bit: offsets <= 0), GENERIC for wide
    ones (8-bit over wide channel blocks: decoded inline, no table), mixed
    channels in one CTA -- against float64 on the dequantized tape."""
    from paper_1901_07988_b200 import codec
    n, ci, hw, co, k = shape
    torch.manual_seed(bits * 100 + ci + k)
    for regime in ("narrow", "nonpos", "wide", "mixed"):
        x = torch.randn(n, ci, hw, hw, device="cuda")
        gamma = torch.rand(ci, device="cuda") + 0.5
        beta = torch.randn(ci, device="cuda") * 0.3
        if regime == "nonpos":
            beta = -beta.abs() if bits == 8 else torch.zeros_like(beta)
        elif regime != "narrow":
            wide = torch.arange(ci, device="cuda") % (1 if regime == "wide" else 5) == 0
            gamma = torch.where(wide, torch.rand(ci, device="cuda") * 0.05 + 0.05, gamma)
            beta = torch.where(wide, torch.rand(ci, device="cuda") + 1.5, beta)
        t = codec.quantize(x, gamma, beta, bits)
        act = codec.dequantize(t, relu=True)
        g = torch.randn(n, co, hw, hw, device="cuda")
        gw = torch.full((co, ci, k, k), 0.125, device="cuda")
        ops.conv2d_wgrad(g, (co, ci, k, k), 1, k // 2, gw, tape=t.as_native(), in_shape=(n, ci, hw, hw))
        ref = torch.nn.grad.conv2d_weight(act.double(), (co, ci, k, k), g.double(), padding=k // 2)
        ref = ref + 0.125
        err = ((gw.double() - ref).norm() / ref.norm()).item()
        assert err < CONV_TOL, (regime, err)


_DUAL_SHAPES = [(128, 16, 32, 16, 3), (128, 16, 32, 64, 1), (128, 64, 32, 16, 1), (128, 32, 16, 32, 3),
                (128, 128, 16, 32, 1), (128, 64, 8, 64, 3)]

_DUAL_CODE = r'''
import sys, torch
from paper_1901_07988_b200 import ops
out = []
for n, ci, hw, co, k in SHAPES:
    g = torch.Generator(device="cuda").manual_seed(ci * 1000 + co + k)
    x = torch.randn(n, ci, hw, hw, device="cuda", generator=g)
    w = torch.randn(co, ci, k, k, device="cuda", generator=g) * 0.1
    gy = torch.randn(n, co, hw, hw, device="cuda", generator=g)
    y = ops.conv2d_forward(x, w, 1, k // 2)
    gx = torch.empty_like(x)
    ops.conv2d_dgrad(gy, w, tuple(x.shape), 1, k // 2, gx)
    out.append((y.cpu(), gx.cpu()))
torch.save(out, sys.argv[1])
'''


def test_two_cta_conv_form_bit_identical(tmp_path):
    """The two-CTAs-per-SM conv form (CIFAR-sized layers with more tiles than
    SMs) against the single-CTA form (QTAPE_FWD_DUAL=0, read once per
    process): forward and data gradient bit-identical (the same per-output
    summation), and within CONV_TOL of float64."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = "SHAPES = " + repr(_DUAL_SHAPES) + "\n" + _DUAL_CODE
    res = {}
    for dual in ("1", "0"):
        path = tmp_path / f"dual{dual}.pt"
        r = subprocess.run([sys.executable, "-c", code, str(path)], cwd=root, capture_output=True,
                           text=True, timeout=300, env=dict(os.environ, QTAPE_FWD_DUAL=dual))
        assert r.returncode == 0, r.stderr[-2000:]
        res[dual] = torch.load(path)
    for (n, ci, hw, co, k), (y1, gx1), (y0, gx0) in zip(_DUAL_SHAPES, res["1"], res["0"]):
        assert torch.equal(y1, y0) and torch.equal(gx1, gx0), (ci, co, k)
        g = torch.Generator(device="cuda").manual_seed(ci * 1000 + co + k)
        x = torch.randn(n, ci, hw, hw, device="cuda", generator=g)
        w = torch.randn(co, ci, k, k, device="cuda", generator=g) * 0.1
        ref = torch.nn.functional.conv2d(x.double(), w.double(), padding=k // 2).cpu()
        assert ((y1.double() - ref).norm() / ref.norm()).item() < CONV_TOL



_MODE_CODE = r'''
import ctypes, sys, torch
from paper_1901_07988_b200 import _native as N, codec, ops
bits, regime, k, ci = int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
n, hw, co = 4, 16, 64
torch.manual_seed(bits * 10 + k)
x = torch.randn(n, ci, hw, hw, device="cuda")
gamma = torch.rand(ci, device="cuda") + 0.5
if regime == "narrow":   # 8-bit FAST: offsets <= 0 (K < 8: zero, else every decode <= 0)
    beta = -torch.rand(ci, device="cuda") * 0.3 if bits == 8 else torch.zeros(ci, device="cuda")
else:   # offsets beta * 2^K / (6 gamma) in [130, 800] (past FAST, inside INT: m < 2048)
    lo, hi = (130, 800) if regime == "wide" else (3000, 5000)   # "huge": past INT too
    beta = (torch.rand(ci, device="cuda") * (hi - lo) + lo + 0.5) * 6 * gamma / 2 ** bits
t = codec.quantize(x, gamma, beta, bits)
act = codec.dequantize(t, relu=True)
g = torch.randn(n, co, hw, hw, device="cuda")
gw = torch.zeros(co, ci, k, k, device="cuda")
fn = N.lib().qt_debug_wgrad_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = torch.zeros(4000, dtype=torch.int64, device="cuda")
fn(buf.data_ptr(), 0)
ops.conv2d_wgrad(g, (co, ci, k, k), 1, k // 2, gw, tape=t.as_native(), in_shape=(n, ci, hw, hw))
torch.cuda.synchronize()
fn(None, 0)
ref = torch.nn.grad.conv2d_weight(act.double(), (co, ci, k, k), g.double(), padding=k // 2)
err = ((gw.double() - ref).norm() / ref.norm()).item()
print("MODE", int(buf[525].item()), int(buf[526].item()), int(buf[527].item()), "ERR", err)
'''


@pytest.mark.parametrize("bits", [1, 2, 4, 8])
@pytest.mark.parametrize("k,ci", [(3, 64), (1, 128)])
def test_wgrad_decode_mode_selected(bits, k, ci):
    """Which operand decode a CTA takes, read from the kernel's debug
    timeline (trace slots 525 FAST, 526 INT, 527 FAST2), and its accuracy:
    FAST (one bf16 integer A piece) for narrow channels at every code width
    (8-bit: offsets <= 0), for wide ones FAST2 (two bf16 pieces of m < 2048)
    at 8 bits and INT (TF32 integer A, two passes) below 8 bits or with
    QTAPE_WG_FAST2=0, the table GENERIC
    past m = 2048 or with QTAPE_WG_INT=0 (8-bit over 128 channels: the
    table decoded inline)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    wide = "MODE 0 0 1" if bits == 8 else "MODE 0 1 0"   # FAST2 is compiled for 8-bit only
    cases = (("narrow", {}, "MODE 1 0 0"), ("wide", {}, wide),
             ("wide", {"QTAPE_WG_FAST2": "0"}, "MODE 0 1 0"), ("huge", {}, "MODE 0 0 0"),
             ("wide", {"QTAPE_WG_INT": "0"}, "MODE 0 0 0"))
    for regime, env, want in cases:
        r = subprocess.run([sys.executable, "-c", _MODE_CODE, str(bits), regime, str(k), str(ci)],
                           cwd=root, capture_output=True, text=True, timeout=300,
                           env={**os.environ, **env})
        assert r.returncode == 0, r.stderr[-2000:]
        assert want in r.stdout, (bits, regime, env, r.stdout)
        err = float(r.stdout.split("ERR")[1])
        assert err < CONV_TOL, (bits, regime, env, err)
