"""Layer forward/backward parity (reference golden vectors + oracle)."""

import numpy as np
import pytest
import torch

import oracle as O
from gpu_util import LAYER_TOL, code_flips, dev, host, norm_err

pytestmark = pytest.mark.gpu

import paper_1901_07988_b200 as P  # noqa: E402
from paper_1901_07988_b200 import _native as N  # noqa: E402
from paper_1901_07988_b200 import layer as L  # noqa: E402
from paper_1901_07988_b200.errors import StateError  # noqa: E402


def _bits(v):
    v = int(v)
    return None if v < 0 else v


def _params(g, k):
    kind = str(g[k + "_kind"])
    kind = "conv" if kind == "plain_conv" else kind
    gamma = g.get(k + "_gamma")
    return L.LayerParams(kind=kind, weight=dev(g[k + "_w"]), stride=int(g[k + "_stride"]),
                         pad=int(g[k + "_pad"]),
                         gamma=None if gamma is None else dev(gamma),
                         beta=None if gamma is None else dev(g[k + "_beta"]))


def test_bn_relu_forward_bit_exact_given_moments():
    """K1 fed the oracle's float64 moments reproduces the reference's A2,
    codes and ReLU output bit for bit (layer.py:245-264, codec.py:107-143)."""
    rng = np.random.default_rng(11)
    for shape, bits in [((4, 5, 8, 8), 4), ((3, 16, 7, 7), 8), ((6, 7), 2), ((2, 3, 5, 5), 1),
                        ((8, 64, 16, 16), 4)]:
        c = shape[1]
        x = (rng.standard_normal(shape) * 2 + 0.5).astype(np.float32)
        gamma = rng.uniform(0.5, 1.5, c).astype(np.float32)
        beta = rng.uniform(-0.3, 0.3, c).astype(np.float32)
        mean, var = O.moments(x)
        kind, wshape = ("dense", (c, 1)) if len(shape) == 2 else ("conv", (1, c, 1, 1))
        p = O.new_params(kind, np.zeros(wshape, np.float32), gamma=gamma, beta=beta)
        for mode in ("approx", "naive", "exact"):
            _, tape = O.layer_fwd(x, dict(p, running_mean=np.zeros(c), running_var=np.ones(c)),
                                  mode, bits)
            a2w = ((((x - O.qtape_oracle._b(mean.astype(np.float32), x.ndim))
                     * O.qtape_oracle._b((1.0 / np.sqrt(var + 1e-5)).astype(np.float32), x.ndim))
                    * O.qtape_oracle._b(gamma, x.ndim)) + O.qtape_oracle._b(beta, x.ndim))
            n_, c_, hw = P.ops.nchw(torch.empty(shape, device="meta"))
            a3 = torch.empty(shape, device="cuda")
            a2 = torch.empty(shape, device="cuda")
            nb = (bits * x.size + 7) // 8
            codes = torch.empty(nb, dtype=torch.uint8, device="cuda")
            step = torch.empty(c, dtype=torch.float64, device="cuda")
            off = torch.empty(c, dtype=torch.int64, device="cuda")
            clip = torch.zeros(1, dtype=torch.int64, device="cuda")
            nm = {"exact": 0, "approx": 1, "naive": 2}[mode]
            kb = 0 if mode == "exact" else bits
            keep = [dev(x), dev(mean), dev(var), dev(gamma), dev(beta)]   # keep alive
            N.call("qt_bn_relu_forward", N.ptr(keep[0]), n_, c_, hw, N.ptr(keep[1]),
                   N.ptr(keep[2]), 1e-5, N.ptr(keep[3]), N.ptr(keep[4]), nm, kb, N.ptr(a3),
                   N.ptr(a2 if mode == "exact" else None), N.ptr(codes if kb else None),
                   N.ptr(step if kb else None), N.ptr(off if kb else None),
                   N.ptr(clip if kb else None), None)
            if mode == "exact":
                assert np.array_equal(host(a2), tape["a2"])
                assert np.array_equal(host(a3), np.maximum(a2w, np.float32(0)))
            else:
                assert np.array_equal(host(codes), tape["q"]["codes"]), (shape, bits, mode)
                assert int(clip.item()) == tape["q"]["clip_count"]
                pre = O.dequantize(tape["q"]) if mode == "naive" else a2w
                assert np.array_equal(host(a3), np.maximum(pre, np.float32(0))), (shape, mode)


def test_golden_layers(golden_layers):
    g = golden_layers
    for i in range(int(g["n_layer"])):
        k = f"l{i}"
        p = _params(g, k)
        mode, bits = str(g[k + "_mode"]), _bits(g[k + "_bits"])
        y, tape = L.layer_forward(dev(g[k + "_x"]), p, mode=mode, bits=bits)
        assert norm_err(host(y), g[k + "_y"]) < LAYER_TOL, k
        if p.preact:
            assert norm_err(host(tape.sigma2), g[k + "_sigma2"]) < 1e-12, k
            assert norm_err(host(p.running_mean), g[k + "_rmean"]) < 1e-12, k
            if tape.is_quantized:
                # the moments may differ from numpy's pairwise sums in the
                # last ulp, which moves A2 by an ulp: any differing code must
                # sit within FLIP_TAU of its boundary (oracle A2, pinned: its
                # codes == the golden codes)
                rp = O.new_params(kind=p.kind, weight=g[k + "_w"], stride=int(g[k + "_stride"]),
                                  pad=int(g[k + "_pad"]), gamma=g[k + "_gamma"],
                                  beta=g[k + "_beta"])
                _, rt = O.layer_fwd(g[k + "_x"], rp, mode, bits, keep_a2=True)
                assert np.array_equal(rt["q"]["codes"], g[k + "_codes"]), k
                f = code_flips(host(tape.stored.codes), rt, bits)
                assert f["bad"] == 0 and f["flips"] <= f["near"], (k, f)
                assert np.array_equal(host(tape.stored.offset), g[k + "_offset"]), k
                assert np.array_equal(host(tape.stored.step), g[k + "_step"]), k
            else:
                assert norm_err(host(tape.stored), g[k + "_a2"]) < LAYER_TOL, k
        gin = L.layer_backward(dev(g[k + "_g"]), tape, p)
        assert norm_err(host(gin), g[k + "_gin"]) < LAYER_TOL, k
        assert norm_err(host(p.grad_weight), g[k + "_gw"]) < LAYER_TOL, k
        if p.preact:
            assert norm_err(host(p.grad_gamma), g[k + "_ggamma"]) < LAYER_TOL, k
            assert norm_err(host(p.grad_beta), g[k + "_gbeta"]) < LAYER_TOL, k


def _conv_params(ci, co, seed, gamma=None, beta=None):
    rng = np.random.default_rng(seed)
    w = (rng.standard_normal((co, ci, 3, 3)) * 0.3).astype(np.float32)
    gamma = np.ones(ci, np.float32) if gamma is None else gamma.astype(np.float32)
    beta = np.zeros(ci, np.float32) if beta is None else beta.astype(np.float32)
    return L.LayerParams(kind="conv", weight=dev(w), stride=1, pad=1, gamma=dev(gamma),
                         beta=dev(beta))


def test_approx_forward_equals_exact_forward_bitwise():
    rng = np.random.default_rng(2)
    x = dev(rng.standard_normal((4, 3, 8, 8)).astype(np.float32))
    ye, _ = L.layer_forward(x, _conv_params(3, 5, 1), mode="exact")
    ya, ta = L.layer_forward(x, _conv_params(3, 5, 1), mode="approx", bits=4)
    assert torch.equal(ye, ya) and ta.is_quantized


def test_identity_bypass_bitwise():
    rng = np.random.default_rng(1)
    x = dev(rng.standard_normal((2, 2, 5, 5)).astype(np.float32))
    ye, te = L.layer_forward(x, _conv_params(2, 3, 4), mode="exact")
    ya, ta = L.layer_forward(x, _conv_params(2, 3, 4), mode="approx", bits=None)
    yn, _ = L.layer_forward(x, _conv_params(2, 3, 4), mode="naive", bits=None)
    assert torch.equal(ye, ya) and torch.equal(ye, yn)
    assert torch.equal(te.stored, ta.stored) and ta.identity


def test_naive_uses_reconstruction():
    rng = np.random.default_rng(3)
    x = dev(rng.standard_normal((4, 3, 8, 8)).astype(np.float32))
    p = _conv_params(3, 5, 7)
    ye, _ = L.layer_forward(x, _conv_params(3, 5, 7), mode="exact")
    yn, tn = L.layer_forward(x, p, mode="naive", bits=4)
    assert not torch.equal(ye, yn)
    _, _, a3 = L.reconstruct_from_tape(tn)
    assert torch.equal(yn, P.ops.conv2d_forward(a3, p.weight, 1, 1))


def test_exactness_decomposition():
    """reference tests/test_layer.py:173-202 on the device."""
    rng = np.random.default_rng(9)
    gamma, beta = rng.uniform(0.8, 1.2, 3), rng.uniform(-0.2, 0.2, 3)
    x = dev(rng.standard_normal((4, 3, 8, 8)).astype(np.float32))
    p = _conv_params(3, 4, 9, gamma, beta)
    out, te = L.layer_forward(x, p, mode="exact")
    _, ta = L.layer_forward(x, p, mode="approx", bits=8)
    g = dev(rng.standard_normal(tuple(out.shape)).astype(np.float32))
    ie, ia = {}, {}
    pe, pa = _conv_params(3, 4, 9, gamma, beta), _conv_params(3, 4, 9, gamma, beta)
    gin_e = L.layer_backward(g, te, pe, internals=ie)
    gin_a = L.layer_backward(g, ta, pa, internals=ia)
    assert torch.equal(ie["mask"], ia["mask"])
    assert torch.equal(ie["grad_linear_in"], ia["grad_linear_in"])
    assert torch.equal(pe.grad_beta, pa.grad_beta)
    assert torch.equal(ie["grad_normalized"], ia["grad_normalized"])
    assert not torch.equal(pe.grad_weight, pa.grad_weight)
    assert not torch.equal(pe.grad_gamma, pa.grad_gamma)
    assert not torch.equal(gin_e, gin_a)
    pa2 = _conv_params(3, 4, 9, gamma, beta)
    gin_sub = L.layer_backward(g, ta, pa2, variance_a1=ie["a1"])
    assert torch.equal(gin_sub, gin_e)


def test_eval_mode_and_errors():
    rng = np.random.default_rng(5)
    p = _conv_params(2, 2, 5)
    x = dev(rng.standard_normal((4, 2, 6, 6)).astype(np.float32))
    for _ in range(3):
        L.layer_forward(x, p, mode="exact")
    y1, tape = L.layer_forward(x, p, training=False)
    assert tape is None
    rm = p.running_mean.clone()
    y2, _ = L.layer_forward(x, p, training=False)
    assert torch.equal(y1, y2) and torch.equal(rm, p.running_mean)
    with pytest.raises(StateError):
        L.layer_backward(torch.zeros((1, 2, 4, 4), device="cuda"), None, p)
    _, t = L.layer_forward(x, p, mode="exact")
    with pytest.raises(StateError):
        L.layer_backward(torch.zeros((4, 2, 9, 9), device="cuda"), t, p)


def test_zero_gradient():
    rng = np.random.default_rng(6)
    p = _conv_params(2, 3, 6)
    x = dev(rng.standard_normal((2, 2, 5, 5)).astype(np.float32))
    out, tape = L.layer_forward(x, p, mode="approx", bits=4)
    gin = L.layer_backward(torch.zeros_like(out), tape, p)
    assert not bool(gin.any()) and not bool(p.grad_weight.any())
    assert not bool(p.grad_gamma.any()) and not bool(p.grad_beta.any())


@pytest.mark.parametrize("cfg", [
    # (n, ci, co, hw, k, pad, bits, mode) -- tensor-core shapes (wgrad decodes the codes in smem)
    (4, 16, 16, 32, 3, 1, 4, "approx"), (8, 64, 16, 8, 1, 0, 4, "approx"),
    (4, 16, 64, 16, 1, 0, 8, "approx"), (2, 32, 32, 16, 3, 1, 2, "approx"),
    (4, 16, 16, 32, 3, 1, 4, "exact"), (4, 32, 128, 8, 1, 0, 1, "approx"),
    # 4-bit offsets beyond the bf16 fast path (2^K-1+2*offset > 127): whole
    # launch generic, and one wide channel making one row group generic
    (4, 16, 16, 32, 3, 1, 4, "approx", "wide"), (2, 32, 32, 16, 3, 1, 4, "approx", "mixed"),
    (4, 64, 256, 8, 1, 0, 4, "approx", "mixed"), (4, 16, 64, 16, 1, 0, 4, "approx", "dead"),
    # ImageNet plane widths: segmented 3x3 (halo above 32 px), flat-padded
    # 1x1, 4-pixel BN-backward groups (14x14), scalar BN backward (7x7)
    (2, 32, 32, 14, 3, 1, 4, "approx"), (2, 16, 32, 7, 1, 0, 4, "approx"),
    (2, 16, 16, 14, 3, 1, 1, "approx"), (2, 16, 16, 28, 3, 1, 2, "approx", "wide"),
    (2, 32, 16, 14, 1, 0, 8, "exact"), (1, 16, 16, 56, 3, 1, 4, "approx", "mixed"),
])
def test_backward_given_device_tape(cfg):
    """Backward parity with the oracle fed OUR tape (codes, step, offset,
    sigma2, frozen gamma/beta): isolates the backward kernels (TC wgrad with
    fused decode, TC dgrad, BN/ReLU backward) from forward-moment ulps."""
    n, ci, co, hw, k, pad, bits, mode = cfg[:8]
    regime = cfg[8] if len(cfg) > 8 else "narrow"
    rng = np.random.default_rng(sum(cfg[:7]))
    w = (rng.standard_normal((co, ci, k, k)) * 0.3).astype(np.float32)
    gamma = rng.uniform(0.5, 1.5, ci).astype(np.float32)
    beta = rng.uniform(-0.3, 0.3, ci).astype(np.float32)
    if regime == "wide":      # offset = floor(beta * 2^K / (6 |gamma|)) ~ 60..200
        gamma = rng.uniform(0.05, 0.1, ci).astype(np.float32)
        beta = rng.uniform(1.5, 3.0, ci).astype(np.float32)
    elif regime == "mixed":   # the last channel alone is wide
        gamma[-1], beta[-1] = 0.05, 2.5
    elif regime == "dead":    # strongly negative offsets: all-zero ReLU channels
        beta[: ci // 2] = -40.0
    x = (rng.standard_normal((n, ci, hw, hw)) * 2 + 0.5).astype(np.float32)
    p = L.LayerParams(kind="conv", weight=dev(w), stride=1, pad=pad, gamma=dev(gamma),
                      beta=dev(beta))
    y, tape = L.layer_forward(dev(x), p, mode=mode, bits=bits)
    g = rng.standard_normal(tuple(y.shape)).astype(np.float32)
    gin = L.layer_backward(dev(g), tape, p)
    ot = {"mode": mode, "sigma2": host(tape.sigma2), "gamma": host(tape.gamma),
          "beta": host(tape.beta), "eps": 1e-5}
    if tape.is_quantized:
        q = tape.stored
        ot["q"] = {"codes": host(q.codes), "bits": bits, "shape": tuple(q.shape),
                   "dtype": np.dtype(np.float32), "step": host(q.step), "offset": host(q.offset)}
    else:
        ot["a2"] = host(tape.stored)
    op = O.new_params("conv", w, 1, pad, gamma.copy(), beta.copy())
    ogin = O.layer_bwd(g, ot, op)
    assert norm_err(host(gin), ogin) < LAYER_TOL
    assert norm_err(host(p.grad_weight), op["grad_weight"]) < LAYER_TOL
    assert norm_err(host(p.grad_gamma), op["grad_gamma"]) < LAYER_TOL
    assert norm_err(host(p.grad_beta), op["grad_beta"]) < LAYER_TOL


@pytest.mark.parametrize("bits", [1, 2, 4, 8, None])
def test_reconstruct_from_tape_matches_oracle(bits):
    """layer.reconstruct_from_tape (layer.py:269-283): A2 = decode(tape),
    A3 = max(A2, 0), A1 = (A2 - beta) / safe_gamma(gamma) with the frozen
    gamma / beta -- bit-exact against the oracle on the same tape, including
    a zero gamma (floored to 1e-8), negative gammas and exact (fp32) tapes."""
    rng = np.random.default_rng(0 if bits is None else bits)
    c = 6
    gamma = np.array([1.0, -0.7, 0.0, 2.5, -1e-9, 0.3], np.float32)
    beta = rng.uniform(-1, 1, c).astype(np.float32)
    x = dev((rng.standard_normal((3, c, 8, 8)) * 2 + 0.5).astype(np.float32))
    p = _conv_params(c, 4, 5, gamma, beta)
    _, t = L.layer_forward(x, p, mode="approx" if bits else "exact", bits=bits)
    a1, a2, a3 = (host(v) for v in L.reconstruct_from_tape(t))
    if t.is_quantized:
        q = {"codes": host(t.stored.codes), "bits": bits, "shape": t.shape, "dtype": np.float32,
             "step": host(t.stored.step), "offset": host(t.stored.offset)}
        want2 = O.dequantize(q)
    else:
        want2 = host(t.stored)
    want3 = np.maximum(want2, np.float32(0))
    gs = O.safe_gamma(host(t.gamma))
    want1 = (want2 - host(t.beta).reshape(1, -1, 1, 1)) / gs.reshape(1, -1, 1, 1)
    for got, want in ((a1, want1), (a2, want2), (a3, want3)):
        assert got.dtype == np.float32
        assert np.array_equal(got.view(np.uint32), want.astype(np.float32).view(np.uint32))


@pytest.mark.parametrize("bits", [1, 2, 4, 8])
def test_decode_threshold_is_the_sign_of_the_decode(bits):
    """codec.decode_threshold (codec.py:165-173) equals the oracle's, and a
    code is >= the threshold exactly when it decodes to a positive value --
    the mask primitive the BN backward uses (bn_bwd.cu's per-code tables)."""
    rng = np.random.default_rng(bits)
    c = 8
    gamma = rng.uniform(0.2, 3, c).astype(np.float32) * rng.choice([-1, 1], c).astype(np.float32)
    beta = np.concatenate([rng.uniform(-4, 4, c - 2), [50.0, -50.0]]).astype(np.float32)
    x = dev(rng.standard_normal((2, c, 4, 4)).astype(np.float32))
    _, t = L.layer_forward(x, _conv_params(c, 4, 1, gamma, beta), mode="approx", bits=bits)
    thr = host(P.codec.decode_threshold(t.stored))
    q = {"bits": bits, "offset": host(t.stored.offset)}
    assert np.array_equal(thr, O.decode_threshold(q))
    codes = np.arange(1 << bits)
    for ch in range(c):
        dec = host(t.stored.step)[ch] * ((codes + (0.5 - (1 << (bits - 1)))) + q["offset"][ch])
        assert np.array_equal(dec.astype(np.float32) > 0, codes >= thr[ch]), (bits, ch)
