"""Whole-network parity: one training step of the reference's tiny residual
net and of the C1 network against the golden vectors, plus the engine
invariants of reference tests/test_engine.py on the device."""

import json

import numpy as np
import pytest
import torch

import oracle as O
from gpu_util import FLIP_TOL, STEP_TOL, code_flips, dev, host, norm_err

pytestmark = pytest.mark.gpu

import paper_1901_07988_b200 as P  # noqa: E402
from paper_1901_07988_b200 import engine as E  # noqa: E402
from paper_1901_07988_b200.errors import StateError  # noqa: E402


def test_golden_network_steps(golden_nets):
    g = golden_nets
    for i in range(int(g["n_net"])):
        k = f"n{i}"
        spec = E.NetworkSpec.from_json(json.loads(str(g[k + "_spec"])))
        mode, bits = str(g[k + "_mode"]), int(g[k + "_bits"])
        params = P.init_params(spec, 0)
        x = dev(g[k + "_x"])
        logits, tapes = E.network_forward(spec, params, x, mode=mode, bits=bits)
        assert norm_err(host(logits), g[k + "_logits"]) < STEP_TOL, k
        loss, lg = P.softmax_xent(logits, g[k + "_labels"])
        assert abs(loss - float(g[k + "_loss"])) <= STEP_TOL * abs(float(g[k + "_loss"])), k
        # the oracle's forward (pinned: its codes == the golden codes) gives
        # the A2 behind every code; each device code that differs must be a
        # neighbouring code within FLIP_TAU of its boundary (gpu_util.code_flips)
        _, rtapes = O.net_fwd(spec.to_json(), O.init_params(spec.to_json(), 0), g[k + "_x"],
                              mode, bits, keep_a2=True)
        flips = 0
        for j, t in enumerate(tapes):
            if t is not None and t.is_quantized:
                assert np.array_equal(rtapes[j]["q"]["codes"], g[f"{k}_codes{j}"]), (k, j)
                f = code_flips(host(t.stored.codes), rtapes[j], bits)
                assert f["bad"] == 0 and f["flips"] <= f["near"], (k, j, f)
                flips += f["flips"]
        # Forward activations agree to fp32 level (split-precision tensor-core
        # convs vs the reference's float64-accumulated loops); a value within
        # an ulp of a quantization boundary can land in the neighbouring code,
        # which moves that activation by a whole step in the backward pass.
        # Gradients get STEP_TOL when every code matches, FLIP_TOL otherwise.
        gtol = STEP_TOL if flips == 0 else FLIP_TOL
        E.network_backward(spec, params, tapes, lg, x, mode=mode)
        for j, p in enumerate(params):
            assert norm_err(host(p.grad_weight), g[f"{k}_gw{j}"]) < gtol, (k, j, flips)
            if p.preact:
                assert norm_err(host(p.grad_gamma), g[f"{k}_gg{j}"]) < gtol, (k, j, flips)
                assert norm_err(host(p.grad_beta), g[f"{k}_gb{j}"]) < gtol, (k, j, flips)
        P.sgd_step(params, 0.1, 0.9, 2e-4)
        for j, p in enumerate(params):
            assert norm_err(host(p.weight), g[f"{k}_w{j}"]) < gtol, (k, j)


def _tiny(blocks=2, channels=4, hw=8, in_ch=2):
    layers = [E.LayerSpec("conv", channels, 3, 1, 1, preact=False)]
    bl = []
    for _ in range(blocks):
        bl.append((len(layers), len(layers) + 1))
        layers += [E.LayerSpec("conv", channels, 3, 1, 1), E.LayerSpec("conv", channels, 3, 1, 1)]
    layers.append(E.LayerSpec("gap_dense", 10))
    return E.NetworkSpec((in_ch, hw, hw), 10, layers, bl)


def test_exact_equals_approx_logits_and_head_exact():
    spec = _tiny()
    x = dev(np.random.default_rng(0).standard_normal((4, 2, 8, 8)).astype(np.float32))
    le, _ = E.network_forward(spec, P.init_params(spec, 0), x, mode="exact")
    la, tapes = E.network_forward(spec, P.init_params(spec, 0), x, mode="approx", bits=4)
    assert torch.equal(le, la)
    assert tapes[1].is_quantized and not tapes[-1].is_quantized


def test_identity_bypass_gradients_bitwise():
    spec = _tiny()
    x = dev(np.random.default_rng(4).standard_normal((3, 2, 8, 8)).astype(np.float32))
    gl = dev(np.random.default_rng(5).standard_normal((3, 10)).astype(np.float32))
    grads = {}
    for mode, bits in (("exact", 8), ("approx", None)):
        params = P.init_params(spec, 11)
        logits, tapes = E.network_forward(spec, params, x, mode=mode, bits=bits)
        E.network_backward(spec, params, tapes, gl, x, mode=mode)
        grads[mode] = host(params.grads).copy()
    assert np.array_equal(grads["exact"], grads["approx"])


def test_determinism_bitwise():
    spec = E.resnet164_spec()
    rng = np.random.default_rng(8)
    x = dev(rng.standard_normal((16, 3, 32, 32)).astype(np.float32))
    g = torch.ones((16, 10), device="cuda")
    outs = []
    for _ in range(2):
        params = P.init_params(spec, 5)
        logits, tapes = E.network_forward(spec, params, x, mode="approx", bits=4)
        E.network_backward(spec, params, tapes, g, x, mode="approx")
        outs.append((host(logits), host(params.grads).copy(),
                     [host(t.stored.codes) for t in tapes if t is not None and t.is_quantized]))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])
    assert all(np.array_equal(a, b) for a, b in zip(outs[0][2], outs[1][2]))


def test_memory_report_matches_instrumented_pool():
    for spec, shape in ((_tiny(), (4, 2, 8, 8)), (E.resnet164_spec(), (8, 3, 32, 32))):
        params = P.init_params(spec, 0)
        x = dev(np.random.default_rng(9).standard_normal(shape).astype(np.float32))
        pool = E.BufferPool(spec.width() + 1)
        logits, tapes = E.network_forward(spec, params, x, mode="approx", bits=4, pool=pool)
        E.network_backward(spec, params, tapes, torch.ones_like(logits), x, mode="approx",
                           pool=pool)
        rep = E.memory_report(spec, shape, mode="approx", bits=4)
        dev_rep = E.memory_report(spec, shape, mode="approx", bits=4, schedule="device")
        # the default report reproduces the reference's W+1 schedule
        # (engine.py:419-482); the device engine holds the block input as the
        # shortcut operand instead of copying it -- its own schedule
        # (schedule="device") equals the instrumented pool byte for byte
        # (reference test_engine.py:246-260), and never exceeds the reference's
        assert pool.peak_live_bytes == dev_rep.transient_buffer_bytes
        assert pool.peak_live_count == dev_rep.peak_live_tensors
        assert dev_rep.transient_buffer_bytes <= rep.transient_buffer_bytes
        assert pool.peak_live_count <= rep.peak_live_tensors <= spec.width() + 1
        assert rep.persistent_tape_bytes == E.measured_tape_bytes(tapes)
        assert rep.channel_overhead_bytes == E.measured_overhead_bytes(tapes)


def test_tape_arena_matches_report():
    spec = E.resnet164_spec()
    arena = E.TapeArena(spec, 128, "approx", 4, torch.device("cuda"))
    rep = E.memory_report(spec, (128, 3, 32, 32), mode="approx", bits=4)
    quant_bytes = sum(pl["persistent_bytes"] for pl in rep.per_layer[:-1])
    assert quant_bytes <= arena.code_arena_bytes <= quant_bytes + 16 * len(spec.layers)


def test_zero_loss_grad_and_errors():
    spec = _tiny()
    params = P.init_params(spec, 0)
    x = dev(np.random.default_rng(3).standard_normal((3, 2, 8, 8)).astype(np.float32))
    logits, tapes = E.network_forward(spec, params, x, mode="approx", bits=8)
    E.network_backward(spec, params, tapes, torch.zeros_like(logits), x, mode="approx")
    assert not bool(params.grads.any())
    with pytest.raises(StateError):
        E.network_backward(spec, params, [None], torch.zeros((3, 10), device="cuda"), x)
    with pytest.raises(Exception):
        E.network_forward(spec, params, torch.zeros((2, 3, 8, 8), device="cuda"))


def test_full_size_c2_step_properties():
    """C2 (ResNet-164, batch 128, K=4) at full size: size-independent
    properties -- tape bytes == memory_report, logits finite, codes in
    range (K=4 nibbles), approx forward == exact forward."""
    spec = E.resnet164_spec()
    x = torch.randn((128, 3, 32, 32), device="cuda", generator=torch.Generator("cuda").manual_seed(0))
    pa = P.init_params(spec, 0)
    la, tapes = E.network_forward(spec, pa, x, mode="approx", bits=4)
    le, _ = E.network_forward(spec, P.init_params(spec, 0), x, mode="exact")
    assert torch.equal(la, le) and bool(torch.isfinite(la).all())
    rep = E.memory_report(spec, (128, 3, 32, 32), mode="approx", bits=4)
    assert E.measured_tape_bytes(tapes) == rep.persistent_tape_bytes
    loss, g = P.softmax_xent(la, np.arange(128) % 10)
    E.network_backward(spec, pa, tapes, g, x, mode="approx")
    assert bool(torch.isfinite(pa.grads).all()) and bool(pa.grads.any())


def test_imagenet_plane_widths_network_step():
    """One approx step of a small bottleneck net whose stages sit on the
    ImageNet plane widths 56 / 28 / 14 / 7 (segmented 3x3 convs with and
    without a halo, flat zero-padded 1x1 / 2x2-s2 convs, 4-pixel BN-backward
    groups, the lower-resolution shortcut adjoint on 28-wide rows) against
    the oracle."""
    spec = E.make_bottleneck_spec([1, 1, 1, 1], [16, 16, 16, 16], input_shape=(3, 112, 112),
                                  stem=(2, 2, 0, 16))
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 3, 112, 112)).astype(np.float32)
    y = rng.integers(0, 10, 2)
    params = P.init_params(spec, 0)
    xd = dev(x)
    logits, tapes = E.network_forward(spec, params, xd, mode="approx", bits=4)
    loss, lg = P.softmax_xent(logits, y)
    E.network_backward(spec, params, tapes, lg, xd, mode="approx")
    sj = spec.to_json()
    ref = O.init_params(sj, 0)
    rlog, rtapes = O.net_fwd(sj, ref, x, "approx", 4, keep_a2=True)
    rloss, rg = O.softmax_xent(rlog, y)
    O.net_bwd(sj, ref, rtapes, rg)
    assert norm_err(host(logits), rlog) < STEP_TOL
    flips = 0
    for t, r in zip(tapes, rtapes):
        if t is not None and t.is_quantized:
            f = code_flips(host(t.stored.codes), r, 4)
            assert f["bad"] == 0 and f["flips"] <= f["near"], f
            flips += f["flips"]
    gtol = STEP_TOL if flips == 0 else FLIP_TOL
    for j, (p, rp) in enumerate(zip(params, ref)):
        assert norm_err(host(p.grad_weight), rp["grad_weight"]) < gtol, (j, flips)
        if p.preact:
            assert norm_err(host(p.grad_gamma), rp["grad_gamma"]) < gtol, (j, flips)
            assert norm_err(host(p.grad_beta), rp["grad_beta"]) < gtol, (j, flips)
