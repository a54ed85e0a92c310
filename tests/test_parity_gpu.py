"""Oracle parity of one full training step at the headline network shapes.

The measured configurations (BASELINE.json configs[1..3]) are ResNet-164
(C2), ResNet-1001 (C3, K=4 and K=2) and ResNet-152 at 224^2 (C4).  Each is
run here at a batch the CPU oracle finishes in seconds, through the same
engine entry points the captured Trainer step uses, and compared with the
oracle (the numpy restatement of /root/reference/pkg/src/qtape/engine.py:282-376
and training.py:192-199):

  forward    per layer, on the input the engine actually passed it: the
             output equals the reference layer's within local_tol(K) and the
             packed codes are the reference's codes of that input (bit-exact
             up to last-ulp moment differences, each within FLIP_TAU of its
             boundary); end to end the logits drift by at most
             drift_tol(depth) (fp32-level differences compounding);
  backward   with identical tapes (the oracle's codes, sigma^2 and head A2
             written into the device tapes) and the oracle's loss gradient:
             per layer, on the output gradient the engine passed it, the
             input gradient and every parameter gradient within local_tol(K)
             of the reference layer's; end to end every grad_* and the
             SGD-updated parameters within drift_tol(depth);
  free run   the step on the device's own tapes is logged (flips, gradient
             differences), gpurun_out/parity_<case>.json.
"""

import json
import os

import numpy as np
import pytest
import torch

import oracle as O
from oracle import qtape_oracle as OQ
from gpu_util import (STEP_TOL, drift_tol, code_flips, dev, host, local_tol,
                      norm_err)

pytestmark = pytest.mark.gpu

import paper_1901_07988_b200 as P  # noqa: E402
from paper_1901_07988_b200 import engine as E  # noqa: E402


def _c4_width():
    # every ResNet-152 layer class (widths 64..512, planes 56^2 -> 7^2, the
    # 4x4/s4 stem, 2x2/s2 transitions, 2048-channel head) with 1-2 blocks per stage
    return E.make_bottleneck_spec([1, 1, 2, 1], [64, 128, 256, 512], (3, 224, 224), 1000,
                                  stem=(4, 4, 0, 64))


CASES = {
    "C2-resnet164-b4-k4": (E.resnet164_spec, 4, 4, 2e-4),
    # 1- and 8-bit tapes (FAST 1-bit / 8-bit decodes); "-bn": gamma, beta drawn
    # off their init so 8-bit offsets take both signs (FAST and FAST2 CTAs)
    "C2-resnet164-b4-k1": (E.resnet164_spec, 4, 1, 2e-4),
    "C2-resnet164-b4-k8-bn": (E.resnet164_spec, 4, 8, 2e-4),
    "C3-resnet1001-b2-k2": (E.resnet1001_spec, 2, 2, 2e-4),
    "C3-resnet1001-b2-k4": (E.resnet1001_spec, 2, 4, 2e-4),
    "C4w-bottleneck1121-224-b2-k4": (_c4_width, 2, 4, 1e-4),
    "C4-resnet152-224-b1-k4": (E.resnet152_spec, 1, 4, 1e-4),
}


def _log(name, rows):
    """Per-layer flip table -> gpurun_out/ (merged back from the GPU box)."""
    root = os.environ.get("GRAFT_REPO_ROOT") or os.path.dirname(os.path.dirname(__file__))
    out = os.path.join(root, "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, f"parity_{name}.json"), "w") as f:
            json.dump(rows, f, indent=1)


def _grad_errs(params, ref):
    errs = []
    for j, (p, rp) in enumerate(zip(params, ref)):
        e = {"layer": j, "w": norm_err(host(p.grad_weight), rp["grad_weight"])}
        if p.preact:
            e["g"] = norm_err(host(p.grad_gamma), rp["grad_gamma"])
            e["b"] = norm_err(host(p.grad_beta), rp["grad_beta"])
        errs.append(e)
    return errs


def _worst(errs):
    return max(max(v for k, v in e.items() if k != "layer") for e in errs)


def _spy_forward(spec, params, xd, bits, check):
    """network_forward with ``check(j, x, y, res)`` called on every layer's
    input, output and fused shortcut operand (host copies) as the engine
    passes them."""
    index = {id(p): j for j, p in enumerate(params)}
    real_fwd = E.layer_forward

    def spy(a_in, p, *a, **k):
        x = host(a_in).copy()
        res = k.get("residual")
        res = None if res is None else host(res).copy()
        out, tape = real_fwd(a_in, p, *a, **k)
        check(index[id(p)], x, host(out), res, tape)
        return out, tape

    E.layer_forward = spy
    try:
        return E.network_forward(spec, params, xd, mode="approx", bits=bits)
    finally:
        E.layer_forward = real_fwd


def _spy_backward(spec, params, tapes, lg, xd, check):
    """network_backward with ``check(j, g_out, g_in, res_g, grads)`` called
    after every layer (host copies; the side-stream weight gradient is
    synchronised first)."""
    index = {id(p): j for j, p in enumerate(params)}
    real_bwd = E.layer_backward

    def spy(g_out, tape, p, *a, **k):
        g = host(g_out).copy()
        res = k.get("residual_grad")
        res = None if res is None else host(res).copy()
        g_in = real_bwd(g_out, tape, p, *a, **k)
        torch.cuda.synchronize()
        grads = {"grad_weight": host(p.grad_weight).copy()}
        if p.preact:
            grads["grad_gamma"] = host(p.grad_gamma).copy()
            grads["grad_beta"] = host(p.grad_beta).copy()
        check(index[id(p)], g, None if g_in is None else host(g_in).copy(), res, grads)
        return g_in

    E.layer_backward = spy
    try:
        E.network_backward(spec, params, tapes, lg, xd, mode="approx")
    finally:
        E.layer_backward = real_bwd


def _force_oracle_tapes(tapes, rtapes):
    """Write the oracle's tapes into the device tapes: packed codes and
    sigma^2 of every quantized layer, the head's exact A2 (gamma/beta copies
    are already identical: same parameters)."""
    for t, r in zip(tapes, rtapes):
        if t is None or t.mode == "plain":
            continue
        if t.is_quantized:
            t.stored.codes.copy_(torch.from_numpy(np.ascontiguousarray(r["q"]["codes"])))
        else:
            t.stored.copy_(torch.from_numpy(np.ascontiguousarray(r["a2"])))
        t.sigma2.copy_(torch.from_numpy(np.ascontiguousarray(r["sigma2"], dtype=np.float64)))


def _bn_draws(ref, name):
    """(gamma, beta) per BN layer for the "-bn" cases: gamma ~ U(0.7, 1.3),
    beta ~ U(-0.2, 0.2) (8-bit offsets floor(beta * 2^8 / (6 gamma)) of
    either sign, up to ~12); None elsewhere."""
    if not name.endswith("-bn"):
        return None
    rng = np.random.default_rng(11)
    out = []
    for p in ref:
        if p["gamma"] is None:
            out.append(None)
            continue
        c = len(p["gamma"])
        out.append((rng.uniform(0.7, 1.3, c).astype(p["gamma"].dtype),
                    rng.uniform(-0.2, 0.2, c).astype(p["beta"].dtype)))
    return out


def _set_bn(draws, oracle_params=None, device_params=None):
    if draws is None:
        return
    for j, d in enumerate(draws):
        if d is None:
            continue
        if oracle_params is not None:
            oracle_params[j]["gamma"][...] = d[0]
            oracle_params[j]["beta"][...] = d[1]
        if device_params is not None:
            device_params[j].gamma.copy_(torch.from_numpy(d[0]))
            device_params[j].beta.copy_(torch.from_numpy(d[1]))


@pytest.mark.parametrize("name", list(CASES))
def test_headline_network_step(name):
    build, n, bits, wd = CASES[name]
    spec = build()
    sj = spec.to_json()
    L = len(spec.layers)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((n,) + tuple(sj["input_shape"])).astype(np.float32)
    y = rng.integers(0, sj["num_classes"], n)

    # ---- oracle: one step (forward keeps A2 / layer inputs for the analysis)
    ref = O.init_params(sj, 0)
    draws = _bn_draws(ref, name)
    _set_bn(draws, oracle_params=ref)
    rlog, rtapes = O.net_fwd(sj, ref, x, "approx", bits, keep_a2=True)
    rloss, rg = O.softmax_xent(rlog, y)
    O.net_bwd(sj, ref, rtapes, rg)

    # ---- forward, layer by layer on the device's own inputs: each layer's
    # output equals the reference layer (O.layer_fwd) applied to the input the
    # engine actually passed it, within local_tol(K); its codes are the
    # reference's codes of that input (differences only from last-ulp moment
    # differences, each within FLIP_TAU of its boundary)
    xd = dev(x)
    params = P.init_params(spec, 0)
    fresh = O.init_params(sj, 0)
    _set_bn(draws, oracle_params=fresh, device_params=params)
    rows, stat = [], {"flips": 0, "local_max": 0.0}

    def check(j, xin, yout, res, t):
        r = rtapes[j]
        want, own = O.layer_fwd(xin, fresh[j], "exact" if j == L - 1 else "approx", bits,
                                keep_a2=True)
        if res is not None:
            want = OQ._shortcut_add(want, res)
        local = norm_err(yout, want)
        stat["local_max"] = max(stat["local_max"], local)
        lspec = spec.layers[j]
        k = xin.shape[1] * (lspec.kernel ** 2 if lspec.kind == "conv" else 1)
        assert local < local_tol(k), (name, j, k, local)
        row = {"layer": j, "local_err": local, "k": k,
               "input_drift": norm_err(xin, r["a_in"]) if "a_in" in r else None}
        if t is not None and t.is_quantized:
            mine = host(t.stored.codes)
            f = code_flips(mine, own, bits)
            assert f["bad"] == 0 and f["flips"] <= f["near"], (name, j, f)
            free = code_flips(mine, r, bits)
            row.update(flips_vs_own_input=f["flips"], flips_vs_oracle=free["flips"],
                       elements=free["elements"])
            stat["flips"] += free["flips"]
        rows.append(row)

    logits, tapes = _spy_forward(spec, params, xd, bits, check)
    flips, local_max = stat["flips"], stat["local_max"]
    # end to end the per-layer fp32-level differences compound over depth
    logits_err = norm_err(host(logits), rlog)
    assert logits_err < drift_tol(L), (name, logits_err)
    loss, lg = P.softmax_xent(logits, y)
    assert abs(loss - rloss) <= drift_tol(L) * abs(rloss), (name, loss, rloss)

    # ---- free-running step (the device's own tapes): reported, not a parity
    # criterion -- a flipped code moves its activation by a whole step, so at a
    # batch of 1-4 images two valid quantizations give visibly different
    # gradients (the reference's own acceptance tests are statistical)
    E.network_backward(spec, params, tapes, lg, xd, mode="approx")
    free = _grad_errs(params, ref)
    assert all(np.isfinite(list(e.values())).all() for e in free)

    # ---- backward parity: identical tapes (the oracle's codes, sigma^2 and
    # head A2 in the device tapes) and the oracle's loss gradient.  Per layer,
    # on the output gradient the engine actually passed it, the input
    # gradient and grad_weight / grad_gamma / grad_beta equal the reference
    # layer's (O.layer_bwd on the same tape) within local_tol(K); end to end
    # every parameter gradient is within drift_tol(depth) of the
    # oracle's backward pass
    params = P.init_params(spec, 0)
    _set_bn(draws, device_params=params)
    _, tapes = E.network_forward(spec, params, xd, mode="approx", bits=bits)
    _force_oracle_tapes(tapes, rtapes)
    fresh_b = O.init_params(sj, 0)
    _set_bn(draws, oracle_params=fresh_b)
    shapes = spec.layer_shapes(n)
    bstat = {"local_max": 0.0}

    def bcheck(j, g_out, g_in, res_g, grads):
        want_in = O.layer_bwd(g_out, rtapes[j], fresh_b[j], need_input_grad=(j != 0))
        if res_g is not None:
            want_in = OQ._shortcut_adj(want_in, res_g)
        ls = spec.layers[j]
        ins, outs = shapes[j]
        k = max(int(np.prod(outs)) // outs[1] if len(outs) == 4 else outs[0],
                outs[1] * (ls.kernel ** 2 if ls.kind == "conv" else 1))
        errs = {name_: norm_err(v, fresh_b[j][name_]) for name_, v in grads.items()}
        if g_in is not None:
            errs["g_in"] = norm_err(g_in, want_in)
        worst = max(errs.values())
        bstat["local_max"] = max(bstat["local_max"], worst)
        rows[j]["bwd_local_err"] = worst
        assert worst < local_tol(k), (name, j, k, errs)

    _spy_backward(spec, params, tapes, dev(rg), xd, bcheck)
    forced = _grad_errs(params, ref)
    assert _worst(forced) < drift_tol(L), (name, max(forced, key=lambda e: max(
        v for k, v in e.items() if k != "layer")))
    P.sgd_step(params, 0.1, 0.9, wd)
    O.sgd(ref, 0.1, 0.9, wd)
    w_err = max(norm_err(host(p.weight), rp["weight"]) for p, rp in zip(params, ref))
    assert w_err < drift_tol(L), (name, w_err)
    _log(name, {"case": name, "bits": bits, "batch": n, "layers": L,
                "local_tol": "max(1e-5, 5e-7 sqrt(K))", "max_local_err": local_max,
                "logits_err": logits_err, "logits_tol": drift_tol(L),
                "loss": loss, "oracle_loss": rloss,
                "total_flips_vs_oracle": flips, "flip_tau": 1e-4,
                "worst_grad_err_free_running": _worst(free),
                "max_bwd_local_err": bstat["local_max"],
                "worst_grad_err_identical_tapes": _worst(forced), "grad_tol": drift_tol(L),
                "sgd_weight_err": w_err, "per_layer": rows})


def test_dp_shard_gradients_match_oracle():
    """SURVEY.md 8(e) parity at G=2 with local BN: each rank's pre-all-reduce
    gradients equal the oracle on its shard, and their mean (what the
    all-reduce produces) equals the mean of the oracle's shard gradients.
    The shards run one after the other on this GPU, exactly as two ranks'
    engines would (each rank's engine sees only its N/G samples)."""
    spec = E.resnet164_spec()
    sj = spec.to_json()
    rng = np.random.default_rng(5)
    x = rng.standard_normal((4, 3, 32, 32)).astype(np.float32)
    y = rng.integers(0, 10, 4)
    mine, theirs = [], []
    for r in range(2):
        xs, ys = x[2 * r:2 * r + 2], y[2 * r:2 * r + 2]
        ref = O.init_params(sj, 0)
        rlog, rtapes = O.net_fwd(sj, ref, xs, "approx", 4)
        _, rg = O.softmax_xent(rlog, ys)
        O.net_bwd(sj, ref, rtapes, rg)
        params = P.init_params(spec, 0)
        xd = dev(xs)
        _, tapes = E.network_forward(spec, params, xd, mode="approx", bits=4)
        _force_oracle_tapes(tapes, rtapes)
        E.network_backward(spec, params, tapes, dev(rg), xd, mode="approx")
        assert _worst(_grad_errs(params, ref)) < STEP_TOL, r
        mine.append(host(params.grads).copy())
        flat = []
        for p, rp in zip(params, ref):
            flat.append(rp["grad_weight"].ravel())
        for p, rp in zip(params, ref):
            if p.preact:
                flat += [rp["grad_gamma"].ravel(), rp["grad_beta"].ravel()]
        theirs.append(np.concatenate(flat))
    assert norm_err((mine[0] + mine[1]) / 2, (theirs[0] + theirs[1]) / 2) < STEP_TOL
