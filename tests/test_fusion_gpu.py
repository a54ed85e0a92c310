"""Layer fusion around the forward GEMM (qt_conv_forward_fused).

  prologue  BN apply + ReLU + K-bit tape inside the conv's operand staging:
            output, packed codes and clip count are BIT-IDENTICAL to the
            unfused sequence qt_bn_relu_forward -> qt_conv_forward with the
            same constants (the rectified activation is the same fp32 value,
            produced by the same four rounded ops, fed to the same GEMM);
  epilogue  the next layer's batch statistics from the conv output (after
            the fused shortcut add): mean / var against the oracle's two-pass
            float64 moments within MOMENT_TOL, and every other output of
            qt_bn_stats_prep (running stats, BnConst, frozen gamma/beta,
            step/offset, clip counter reset) equal to what the standalone
            kernel writes from those moments.
Reference: layer.py:236-266, codec.py:107-143, ops.py:186-196.
"""

import numpy as np
import pytest
import torch

import oracle as O
from gpu_util import MOMENT_TOL, STEP_TOL, dev, host, norm_err

pytestmark = pytest.mark.gpu

import paper_1901_07988_b200 as P  # noqa: E402
from paper_1901_07988_b200 import _native as N  # noqa: E402
from paper_1901_07988_b200 import engine as E  # noqa: E402
from paper_1901_07988_b200 import ops  # noqa: E402
from paper_1901_07988_b200.layer import TapeSlot  # noqa: E402

# (n, ci, h, co, k, pad): row-tiled 32/16/8 px (8x8: two images per tile),
# 3x3 and 1x1, flat 1x1 on ImageNet planes (partial last run at 28x28)
PRO_GEOS = [(4, 16, 32, 16, 3, 1), (4, 16, 32, 64, 1, 0), (4, 64, 16, 32, 1, 0),
            (4, 32, 16, 32, 3, 1), (6, 64, 8, 64, 3, 1), (4, 256, 8, 64, 1, 0),
            (2, 64, 56, 64, 1, 0), (2, 128, 28, 32, 1, 0), (2, 48, 16, 16, 1, 0)]


def _bn_params(c, rng):
    gamma = (rng.uniform(0.5, 2.0, c) * rng.choice([-1, 1], c)).astype(np.float32)
    gamma[0] = 1.0
    beta = rng.uniform(-1, 1, c).astype(np.float32)
    return gamma, beta


def _stats_prep(x, gamma, beta, bits, slot, rmean, rvar):
    n, c, h, w = x.shape
    hw = h * w
    sws = ops.workspace(N.query("qt_bn_stats_workspace", n, c, hw), x.device, "stats")
    N.call("qt_bn_stats_prep", N.ptr(x), n, c, hw, 1e-5, N.ptr(gamma), N.ptr(beta), bits,
           N.ptr(slot.mean), N.ptr(slot.var), N.ptr(rmean), N.ptr(rvar), N.ptr(slot.gamma),
           N.ptr(slot.beta), N.ptr(slot.step), N.ptr(slot.offset), N.ptr(slot.clip),
           N.ptr(slot.consts), N.ptr(sws))


@pytest.mark.parametrize("geo", PRO_GEOS)
@pytest.mark.parametrize("bits", [4, 2, 8, 1])
def test_prologue_bitwise_equals_unfused(geo, bits):
    n, ci, h, co, k, pad = geo
    if N.query("qt_conv_fused_support", n, ci, h, h, co, k, k, 1, pad, 1, bits) & 1 == 0:
        pytest.skip("prologue not available for this shape / width")
    rng = np.random.default_rng(sum(geo) + bits)
    x = dev((rng.standard_normal((n, ci, h, h)) * 3 + 1).astype(np.float32))
    w = dev((rng.standard_normal((co, ci, k, k)) * 0.2).astype(np.float32))
    g_np, b_np = _bn_params(ci, rng)
    gamma, beta = dev(g_np), dev(b_np)
    outs = []
    for fused in (False, True):
        slot = TapeSlot(tuple(x.shape), ci, bits, False, x.device)
        rm = torch.zeros(ci, dtype=torch.float64, device="cuda")
        rv = torch.ones(ci, dtype=torch.float64, device="cuda")
        _stats_prep(x, gamma, beta, bits, slot, rm, rv)
        out = torch.empty((n, co, h + 2 * pad - k + 1, h + 2 * pad - k + 1), device="cuda")
        if fused:
            pro = N.BnPrologue(N.ptr(slot.consts), N.ptr(slot.codes), N.ptr(slot.clip), bits)
            ops.conv2d_forward_fused(x, w, 1, pad, out, prologue=pro)
        else:
            work = torch.empty_like(x)
            N.call("qt_bn_relu_forward", N.ptr(x), n, ci, h * h, N.ptr(slot.mean),
                   N.ptr(slot.var), 1e-5, N.ptr(gamma), N.ptr(beta), 1, bits, N.ptr(work), None,
                   N.ptr(slot.codes), N.ptr(slot.step), N.ptr(slot.offset), N.ptr(slot.clip),
                   N.ptr(slot.consts))
            ops.conv2d_forward(work, w, 1, pad, out=out)
        outs.append((host(out).copy(), host(slot.codes).copy(), int(slot.clip.item())))
    (o0, c0, k0), (o1, c1, k1) = outs
    assert np.array_equal(c0, c1), geo
    assert k0 == k1, (k0, k1)
    assert np.array_equal(o0.view(np.uint32), o1.view(np.uint32)), (geo, norm_err(o1, o0))


# (n, ci, h, co, k, stride, pad, res): the epilogue sees the shortcut sum
EPI_GEOS = [(4, 16, 32, 64, 1, 1, 0, "same"), (4, 16, 32, 16, 3, 1, 1, None),
            (6, 64, 8, 256, 1, 1, 0, "same"), (4, 32, 16, 128, 1, 1, 0, "half"),
            (2, 64, 56, 256, 1, 1, 0, "same"), (4, 32, 32, 32, 2, 2, 0, None),
            (2, 128, 28, 512, 1, 1, 0, None), (4, 64, 16, 32, 3, 1, 1, None)]


@pytest.mark.parametrize("geo", EPI_GEOS)
def test_stats_epilogue_matches_oracle_moments(geo):
    n, ci, h, co, k, s, pad, res_kind = geo
    oh = (h + 2 * pad - k) // s + 1
    rng = np.random.default_rng(sum(g for g in geo if isinstance(g, int)))
    x = (rng.standard_normal((n, ci, h, h))).astype(np.float32)
    w = (rng.standard_normal((co, ci, k, k)) * 0.3).astype(np.float32)
    res = None
    sr = 1
    if res_kind == "same":
        res = (rng.standard_normal((n, co // 2, oh, oh)) + 2).astype(np.float32)
    elif res_kind == "half":
        res = (rng.standard_normal((n, co // 4, 2 * oh, 2 * oh)) - 1).astype(np.float32)
        sr = 2
    sup = N.query("qt_conv_fused_support", n, ci, h, h, co, k, k, s, pad, sr, 4)
    if not sup & 2:
        pytest.skip("statistics epilogue not available for this shape")
    g_np, b_np = _bn_params(co, rng)
    gamma, beta = dev(g_np), dev(b_np)
    out = torch.empty((n, co, oh, oh), device="cuda")
    slot = TapeSlot((n, co, oh, oh), co, 4, False, out.device)
    slot.clip.fill_(12345)
    rm = dev(rng.standard_normal(co))
    rv = dev(rng.uniform(0.5, 2, co))
    rm0, rv0 = host(rm).copy(), host(rv).copy()
    fws = torch.zeros(N.query("qt_conv_stats_workspace", co), dtype=torch.uint8, device="cuda")
    epi = N.BnStatsEpilogue(1e-5, N.ptr(gamma), N.ptr(beta), 4, N.ptr(slot.mean), N.ptr(slot.var),
                            N.ptr(rm), N.ptr(rv), N.ptr(slot.gamma), N.ptr(slot.beta),
                            N.ptr(slot.step), N.ptr(slot.offset), N.ptr(slot.clip),
                            N.ptr(slot.consts), N.ptr(fws))
    resd = None if res is None else dev(res)
    for rep in range(2):     # twice: the counters must be re-armed by the kernel
        ops.conv2d_forward_fused(dev(x), dev(w), s, pad, out, residual=resd, epilogue=epi)
    y = host(out)
    want = O.conv_fwd(x, w, s, pad)
    if res is not None:
        from oracle import qtape_oracle as OQ
        want = OQ._shortcut_add(want, res)
    assert norm_err(y, want) < 1e-5
    mean, var = O.moments(y.astype(np.float32))
    assert norm_err(host(slot.mean), mean) < MOMENT_TOL
    assert norm_err(host(slot.var), var) < MOMENT_TOL
    assert not bool(fws[:8].any())          # counters left at zero
    # everything else equals the standalone qt_bn_stats_prep on the same output
    ref = TapeSlot((n, co, oh, oh), co, 4, False, out.device)
    rm2, rv2 = dev(rm0), dev(rv0)
    for _ in range(2):
        _stats_prep(out, gamma, beta, 4, ref, rm2, rv2)
    assert norm_err(host(rm), host(rm2)) < MOMENT_TOL and norm_err(host(rv), host(rv2)) < MOMENT_TOL
    assert np.array_equal(host(slot.gamma), g_np) and np.array_equal(host(slot.beta), b_np)
    assert np.array_equal(host(slot.step), host(ref.step))
    assert np.array_equal(host(slot.offset), host(ref.offset))
    assert int(slot.clip.item()) == 0
    # BnConst: the code constants are exact, mean32 / inv32 agree to fp32
    bc = host(slot.consts).view(np.uint32).reshape(co, 12)
    br = host(ref.consts).view(np.uint32).reshape(co, 12)
    assert np.array_equal(bc[:, 2:], br[:, 2:])
    assert np.allclose(bc[:, :2].view(np.float32), br[:, :2].view(np.float32), rtol=2e-7, atol=0)


@pytest.mark.parametrize("bits", [4, 2])
def test_fused_engine_matches_unfused(bits, monkeypatch):
    """The fused engine (prologue + epilogue statistics) against the unfused
    sequence on ResNet-164 at batch 8: logits, loss and gradients agree to
    fp32 level; codes may differ only where the two (both float64) moment
    computations round mean32 / inv32 differently, which the network parity
    test bounds against the oracle."""
    spec = E.resnet164_spec()
    rng = np.random.default_rng(bits)
    x = dev(rng.standard_normal((8, 3, 32, 32)).astype(np.float32))
    y = rng.integers(0, 10, 8)
    monkeypatch.setenv("QTAPE_FUSE", "1")
    pro, epi = E.fusion_plan(spec, 8, "approx", bits)
    assert sum(pro) > 100 and sum(epi) > 100
    res = []
    for fuse in ("0", "1"):
        monkeypatch.setenv("QTAPE_FUSE", fuse)
        params = P.init_params(spec, 0)
        logits, tapes = E.network_forward(spec, params, x, mode="approx", bits=bits)
        loss, g = P.softmax_xent(logits, y)
        E.network_backward(spec, params, tapes, g, x, mode="approx")
        codes = np.concatenate([host(t.stored.codes) for t in tapes if t is not None and
                                t.is_quantized])
        rm = np.concatenate([host(p.running_mean) for p in params if p.preact])
        res.append((host(logits), loss, host(params.grads).copy(), codes, rm))
    (l0, s0, g0, c0, r0), (l1, s1, g1, c1, r1) = res
    assert norm_err(l1, l0) < 1e-5
    assert abs(s1 - s0) < STEP_TOL * abs(s0)
    assert norm_err(r1, r0) < 1e-9
    assert np.mean(c0 == c1) > 0.9999
    assert norm_err(g1, g0) < 5e-2      # a flipped code moves its activation a whole step


@pytest.mark.parametrize("mode,bits", [("approx", 4), ("approx", 2), ("approx", 8), ("approx", 1),
                                       ("naive", 4), ("exact", None), ("approx", None)])
def test_fused_bn_forward_bitwise(mode, bits, monkeypatch):
    """qt_bn_forward_fused (statistics + BN apply + tape + ReLU in one
    launch) against the two-launch path on ResNet-164 at batch 8."""
    spec = E.resnet164_spec()
    rng = np.random.default_rng(7)
    x = dev(rng.standard_normal((8, 3, 32, 32)).astype(np.float32))
    y = rng.integers(0, 10, 8)
    res = []
    for fused in ("0", "1"):
        monkeypatch.setenv("QTAPE_BN_FUSED", fused)     # 1: the one-launch form (opt-in)
        params = P.init_params(spec, 0)
        logits, tapes = E.network_forward(spec, params, x, mode=mode, bits=bits)
        loss, g = P.softmax_xent(logits, y)
        E.network_backward(spec, params, tapes, g, x, mode=mode)
        tb = []
        for t in tapes:
            if t is None or t.mode == "plain":
                continue
            tb.append(host(t.sigma2))
            if t.is_quantized:
                tb += [host(t.stored.codes), np.array([t.stored.clip_count])]
            else:
                tb.append(host(t.stored))
        rm = [host(p.running_mean) for p in params if p.preact]
        res.append((host(logits), host(params.grads).copy(), tb, rm))
    (l0, g0, t0, r0), (l1, g1, t1, r1) = res
    # the fused kernel sums the moments with 512 threads (float64, another
    # order): mean / var agree to MOMENT_TOL, so mean32 / inv32 and with them
    # the codes are equal except where a last-ulp difference moves an A2
    # across a boundary
    assert norm_err(l1, l0) < 1e-6
    for a, b in zip(t0, t1):
        if a.dtype == np.float64:
            assert norm_err(b, a) < MOMENT_TOL
        elif a.dtype == np.uint8:
            assert np.mean(a == b) > 0.9999
    assert all(norm_err(b, a) < MOMENT_TOL for a, b in zip(r0, r1))
    assert norm_err(g1, g0) < 5e-2
