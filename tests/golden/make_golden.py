"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run here (the reference only exists in the build container):

    PYTHONPATH=/root/reference/pkg/src XDG_CACHE_HOME=/tmp/qtape_cache \
        python tests/golden/make_golden.py

It imports ``qtape`` from /root/reference/pkg/src and records inputs and
outputs of the hot-path functions on small seeded cases:

* codec.npz   -- quantize/dequantize/pack on random + edge-case tensors
                 (codec.py:59-156), incl. NaN/inf/subnormal/huge inputs.
* layers.npz  -- layer_forward / layer_backward for every kind x mode
                 (layer.py:208-381).
* nets.npz    -- one full training step (forward, xent, backward, SGD) of
                 the tiny residual net of test_engine.py:12-22 and of the C1
                 network make_residual_spec(8,3,3) (engine.py:557-585).
* memory.json -- memory_report (engine.py:485-534) for C1..C4 specs.

The fixtures pin the oracle (tests/test_oracle_golden.py) and are the
golden vectors of the GPU parity tests.
"""

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("XDG_CACHE_HOME", "/tmp/qtape_cache")

from qtape import codec as Q  # noqa: E402
from qtape import engine as E  # noqa: E402
from qtape import layer as L  # noqa: E402
from qtape import training as T  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def bottleneck_spec_json(blocks, widths, input_shape, classes, stem):
    """SURVEY.md Appendix C recipe (pre-activation bottleneck)."""
    k, s, p, c0 = stem
    layers = [{"kind": "conv", "out_channels": c0, "kernel": k, "stride": s,
               "pad": p, "preact": False}]
    blist = []
    for si, (nb, c) in enumerate(zip(blocks, widths)):
        for b in range(nb):
            first = len(layers)
            mid = ({"kind": "conv", "out_channels": c, "kernel": 2, "stride": 2, "pad": 0}
                   if (si > 0 and b == 0) else
                   {"kind": "conv", "out_channels": c, "kernel": 3, "stride": 1, "pad": 1})
            layers += [{"kind": "conv", "out_channels": c, "kernel": 1, "stride": 1, "pad": 0},
                       mid,
                       {"kind": "conv", "out_channels": 4 * c, "kernel": 1, "stride": 1, "pad": 0}]
            blist.append([first, first + 2])
    layers.append({"kind": "gap_dense", "out_channels": classes})
    for l in layers:
        l.setdefault("preact", True)
    return {"input_shape": list(input_shape), "num_classes": classes,
            "layers": layers, "blocks": blist}


def specs():
    return {
        "C1": E.make_residual_spec(base_channels=8, blocks_per_stage=3, stages=3).to_json(),
        "C2": bottleneck_spec_json([18, 18, 18], [16, 32, 64], (3, 32, 32), 10, (3, 1, 1, 16)),
        "C3": bottleneck_spec_json([111, 111, 111], [16, 32, 64], (3, 32, 32), 100, (3, 1, 1, 16)),
        "C4": bottleneck_spec_json([3, 8, 36, 3], [64, 128, 256, 512], (3, 224, 224), 1000,
                                   (4, 4, 0, 64)),
    }


def codec_cases(out):
    rng = np.random.default_rng(1234)
    idx = 0
    for bits in (1, 2, 4, 8):
        for shape in [(2, 3, 5, 7), (3, 5, 7, 7), (4, 17), (1, 2, 3, 3)]:
            c = shape[1]
            a = (rng.standard_normal(shape) * 3 + 1).astype(np.float32)
            gamma = rng.uniform(0.5, 2.0, c).astype(np.float32)
            beta = rng.uniform(-1, 1, c).astype(np.float32)
            if idx % 3 == 1:
                gamma[0] = -gamma[0]          # negative gamma: |gamma| coding range
            if idx % 5 == 2:
                gamma[-1] = 0.0               # floored gamma
            flat = a.reshape(-1)
            if flat.size > 12 and idx % 2 == 0:
                flat[:8] = [np.nan, np.inf, -np.inf, 1e30, -1e30,
                            np.float32(1.4e-45), np.float32(-1.4e-45), 0.0]
            t = Q.quantize(a, gamma, beta, bits, sigma2=rng.uniform(0.1, 2, c))
            key = f"c{idx}"
            out[key + "_a"] = a
            out[key + "_gamma"] = gamma
            out[key + "_beta"] = beta
            out[key + "_bits"] = np.int64(bits)
            out[key + "_codes"] = t.codes
            out[key + "_step"] = t.step
            out[key + "_offset"] = t.offset
            out[key + "_clip"] = np.int64(t.clip_count)
            out[key + "_deq"] = Q.dequantize(t)
            idx += 1
    out["n_codec"] = np.int64(idx)


def conv_params(ci, co, rng, k, stride, pad, dtype, preact=True):
    w = (rng.standard_normal((co, ci, k, k)) * 0.3).astype(dtype)
    if not preact:
        return L.LayerParams(kind="conv", weight=w, stride=stride, pad=pad)
    return L.LayerParams(kind="conv", weight=w, stride=stride, pad=pad,
                         gamma=rng.uniform(0.5, 1.5, ci).astype(dtype),
                         beta=rng.uniform(-0.3, 0.3, ci).astype(dtype))


def layer_cases(out):
    rng = np.random.default_rng(99)
    cases = []
    for kind, geo in [("conv", (3, 1, 1)), ("conv", (2, 2, 0)), ("conv", (1, 1, 0)),
                      ("conv", (4, 4, 0)), ("dense", None), ("gap_dense", None),
                      ("plain_conv", (3, 1, 1))]:
        for mode, bits in [("exact", 8), ("approx", 4), ("approx", 8), ("approx", 2),
                           ("naive", 4), ("approx", None)]:
            if kind == "plain_conv" and mode != "exact":
                continue
            cases.append((kind, geo, mode, bits))
    for i, (kind, geo, mode, bits) in enumerate(cases):
        key = f"l{i}"
        if kind in ("conv", "plain_conv"):
            k, s, p = geo
            ci, co, hw = 5, 6, 8
            prm = conv_params(ci, co, rng, k, s, p, np.float32, preact=(kind == "conv"))
            x = (rng.standard_normal((4, ci, hw, hw)) * 2 + 0.5).astype(np.float32)
        elif kind == "dense":
            prm = L.LayerParams(kind="dense",
                                weight=(rng.standard_normal((7, 5)) * 0.5).astype(np.float32),
                                gamma=rng.uniform(0.5, 1.5, 7).astype(np.float32),
                                beta=rng.uniform(-0.3, 0.3, 7).astype(np.float32))
            x = rng.standard_normal((6, 7)).astype(np.float32)
        else:
            prm = L.LayerParams(kind="gap_dense",
                                weight=(rng.standard_normal((5, 10)) * 0.5).astype(np.float32),
                                gamma=rng.uniform(0.5, 1.5, 5).astype(np.float32),
                                beta=rng.uniform(-0.3, 0.3, 5).astype(np.float32))
            x = rng.standard_normal((4, 5, 4, 4)).astype(np.float32)
        out[key + "_kind"] = np.array(kind)
        out[key + "_mode"] = np.array(mode)
        out[key + "_bits"] = np.int64(-1 if bits is None else bits)
        out[key + "_x"] = x
        out[key + "_w"] = prm.weight.copy()
        out[key + "_stride"] = np.int64(prm.stride)
        out[key + "_pad"] = np.int64(prm.pad)
        if prm.preact:
            out[key + "_gamma"] = prm.gamma.copy()
            out[key + "_beta"] = prm.beta.copy()
        y, tape = L.layer_forward(x, prm, mode=mode, bits=bits)
        g = rng.standard_normal(y.shape).astype(np.float32)
        internals = {}
        gin = L.layer_backward(g, tape, prm, internals=internals)
        out[key + "_y"] = y
        out[key + "_g"] = g
        out[key + "_gin"] = gin
        out[key + "_gw"] = prm.grad_weight
        if prm.preact:
            out[key + "_ggamma"] = prm.grad_gamma
            out[key + "_gbeta"] = prm.grad_beta
            out[key + "_sigma2"] = tape.sigma2
            out[key + "_rmean"] = prm.running_mean
            out[key + "_rvar"] = prm.running_var
            if tape.is_quantized:
                out[key + "_codes"] = tape.stored.codes
                out[key + "_step"] = tape.stored.step
                out[key + "_offset"] = tape.stored.offset
                out[key + "_clip"] = np.int64(tape.stored.clip_count)
            else:
                out[key + "_a2"] = tape.stored
    out["n_layer"] = np.int64(len(cases))


def tiny_residual_json():
    layers = [{"kind": "conv", "out_channels": 4, "kernel": 3, "stride": 1, "pad": 1,
               "preact": False}]
    blocks = []
    for _ in range(2):
        first = len(layers)
        layers += [{"kind": "conv", "out_channels": 4, "kernel": 3, "stride": 1, "pad": 1,
                    "preact": True}] * 2
        blocks.append([first, first + 1])
    # a downsampling block exercises the stride-2 / channel-pad shortcut
    first = len(layers)
    layers += [{"kind": "conv", "out_channels": 8, "kernel": 2, "stride": 2, "pad": 0,
                "preact": True},
               {"kind": "conv", "out_channels": 8, "kernel": 3, "stride": 1, "pad": 1,
                "preact": True}]
    blocks.append([first, first + 1])
    layers.append({"kind": "gap_dense", "out_channels": 10, "kernel": 3, "stride": 1,
                   "pad": 1, "preact": True})
    return {"input_shape": [2, 8, 8], "num_classes": 10, "layers": layers, "blocks": blocks}


def net_cases(out):
    nets = [("tiny", tiny_residual_json(), 3), ("c1", specs()["C1"], 8)]
    idx = 0
    for name, sj, batch in nets:
        spec = E.NetworkSpec.from_json(sj)
        for mode, bits in [("approx", 4), ("approx", 8), ("exact", 8), ("naive", 4),
                           ("approx", 2)]:
            if name == "c1" and mode in ("naive",):
                continue
            rng = np.random.default_rng(idx)
            x = rng.standard_normal((batch,) + tuple(sj["input_shape"])).astype(np.float32)
            labels = rng.integers(0, sj["num_classes"], batch)
            params = T.init_params(spec, 0)
            logits, tapes = E.network_forward(spec, params, x, mode=mode, bits=bits)
            loss, g = T.softmax_xent(logits, labels)
            E.network_backward(spec, params, tapes, g, x, mode=mode)
            key = f"n{idx}"
            out[key + "_spec"] = np.array(json.dumps(sj))
            out[key + "_mode"] = np.array(mode)
            out[key + "_bits"] = np.int64(bits)
            out[key + "_x"] = x
            out[key + "_labels"] = labels
            out[key + "_logits"] = logits
            out[key + "_loss"] = np.float64(loss)
            for i, (p, t) in enumerate(zip(params, tapes)):
                out[f"{key}_gw{i}"] = p.grad_weight.copy()
                if p.preact:
                    out[f"{key}_gg{i}"] = p.grad_gamma.copy()
                    out[f"{key}_gb{i}"] = p.grad_beta.copy()
                    out[f"{key}_sigma2_{i}"] = t.sigma2
                    if t.is_quantized:
                        out[f"{key}_codes{i}"] = t.stored.codes
            T.sgd_step(params, 0.1, 0.9, 2e-4)
            for i, p in enumerate(params):
                out[f"{key}_w{i}"] = p.weight.copy()
                if p.preact:
                    out[f"{key}_gamma{i}"] = p.gamma.copy()
                    out[f"{key}_beta{i}"] = p.beta.copy()
            idx += 1
    out["n_net"] = np.int64(idx)


def memory_cases():
    res = {}
    batches = {"C1": 32, "C2": 128, "C3": 128, "C4": 32}
    for name, sj in specs().items():
        spec = E.NetworkSpec.from_json(sj)
        res[name] = {"spec": sj, "batch": batches[name], "reports": []}
        shape = (batches[name],) + tuple(sj["input_shape"])
        for mode, bits in [("exact", None), ("approx", 8), ("approx", 4), ("approx", 2),
                           ("approx", 1), ("naive", 4)]:
            r = E.memory_report(spec, shape, mode=mode, bits=bits)
            res[name]["reports"].append({
                "mode": mode, "bits": bits, "width": r.width,
                "persistent_tape_bytes": r.persistent_tape_bytes,
                "channel_overhead_bytes": r.channel_overhead_bytes,
                "transient_buffer_bytes": r.transient_buffer_bytes,
                "peak_live_tensors": r.peak_live_tensors,
                "parameter_bytes": r.parameter_bytes,
                "exact_persistent_bytes": r.exact_persistent_bytes,
            })
    return res


def main():
    out = {}
    codec_cases(out)
    np.savez_compressed(os.path.join(HERE, "codec.npz"), **out)
    out = {}
    layer_cases(out)
    np.savez_compressed(os.path.join(HERE, "layers.npz"), **out)
    out = {}
    net_cases(out)
    np.savez_compressed(os.path.join(HERE, "nets.npz"), **out)
    with open(os.path.join(HERE, "memory.json"), "w") as f:
        json.dump(memory_cases(), f, indent=1)
    for fn in ("codec.npz", "layers.npz", "nets.npz", "memory.json"):
        print(fn, os.path.getsize(os.path.join(HERE, fn)))


if __name__ == "__main__":
    main()
