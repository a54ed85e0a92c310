"""Pin the CPU oracle (oracle/qtape_oracle.py) against fixtures produced by
the unmodified reference (tests/golden/make_golden.py).  CPU only."""

import json

import numpy as np
import pytest

import oracle as O
from conftest import rel_err


def _bits(v):
    v = int(v)
    return None if v < 0 else v


def test_kats():
    # reference tests/test_quantize.py:20-87 known answers
    def one(values, gamma=1.0, beta=0.0, bits=4):
        a = np.asarray(values, np.float64).reshape(1, 1, -1, 1)
        return O.quantize(a, np.array([gamma]), np.array([beta]), bits)

    t = one([0.1]); assert O.unpack(t["codes"], 4, 1)[0] == 8 and t["clip_count"] == 0
    t = one([10.0]); assert O.unpack(t["codes"], 4, 1)[0] == 15 and t["clip_count"] == 1
    t = one([-0.01], bits=8); assert O.unpack(t["codes"], 8, 1)[0] == 127
    assert O.dequantize(one([0.1]))[0, 0, 0, 0] == 0.1875
    assert O.dequantize(one([10.0]))[0, 0, 0, 0] == 2.8125
    assert O.dequantize(one([-0.01], bits=8))[0, 0, 0, 0] == -0.01171875
    assert one([0.5], gamma=0.0)["step"][0] == pytest.approx(6e-8 / 16)
    assert O.pack(np.array([3, 7, 0, 15]), 4).tolist() == [0x73, 0xF0]
    assert O.pack(np.array([1, 0, 1, 1, 0, 0, 0, 0]), 1).tolist() == [0x0D]
    assert O.pack(np.array([1, 2, 3, 0, 3]), 2).tolist() == [0x39, 0x03]
    with pytest.raises(ValueError):
        O.unpack(np.zeros(3, np.uint8), 4, 4)


def test_codec_bit_exact(golden_codec):
    g = golden_codec
    for i in range(int(g["n_codec"])):
        k = f"c{i}"
        t = O.quantize(g[k + "_a"], g[k + "_gamma"], g[k + "_beta"], int(g[k + "_bits"]))
        assert np.array_equal(t["codes"], g[k + "_codes"]), k
        assert np.array_equal(t["step"], g[k + "_step"]), k
        assert np.array_equal(t["offset"], g[k + "_offset"]), k
        assert t["clip_count"] == int(g[k + "_clip"]), k
        assert np.array_equal(O.dequantize(t), g[k + "_deq"]), k


def _params_from(g, k):
    kind = str(g[k + "_kind"])
    gamma = g.get(k + "_gamma")
    beta = g.get(k + "_beta")
    kind = "conv" if kind == "plain_conv" else kind
    return O.new_params(kind, g[k + "_w"].copy(), int(g[k + "_stride"]),
                        int(g[k + "_pad"]),
                        None if gamma is None else gamma.copy(),
                        None if beta is None else beta.copy())


def test_layers(golden_layers):
    g = golden_layers
    for i in range(int(g["n_layer"])):
        k = f"l{i}"
        p = _params_from(g, k)
        y, tape = O.layer_fwd(g[k + "_x"], p, str(g[k + "_mode"]), _bits(g[k + "_bits"]))
        # forward is fixed-order: bit exact
        assert np.array_equal(y, g[k + "_y"]), k
        if p["gamma"] is not None:
            assert np.array_equal(tape["sigma2"], g[k + "_sigma2"]), k
            assert np.array_equal(p["running_mean"], g[k + "_rmean"]), k
            if "q" in tape:
                assert np.array_equal(tape["q"]["codes"], g[k + "_codes"]), k
                assert tape["q"]["clip_count"] == int(g[k + "_clip"]), k
            else:
                assert np.array_equal(tape["a2"], g[k + "_a2"]), k
        gin = O.layer_bwd(g[k + "_g"], tape, p)
        # backward contractions are BLAS-ordered: tolerance
        assert rel_err(gin, g[k + "_gin"], 1e-3) < 1e-5, k
        assert rel_err(p["grad_weight"], g[k + "_gw"], 1e-3) < 1e-5, k
        if p["gamma"] is not None:
            assert rel_err(p["grad_gamma"], g[k + "_ggamma"], 1e-3) < 1e-5, k
            assert rel_err(p["grad_beta"], g[k + "_gbeta"], 1e-3) < 1e-5, k


def test_nets(golden_nets):
    g = golden_nets
    for i in range(int(g["n_net"])):
        k = f"n{i}"
        spec = json.loads(str(g[k + "_spec"]))
        params = O.init_params(spec, 0)
        logits, tapes = O.net_fwd(spec, params, g[k + "_x"], str(g[k + "_mode"]),
                                  int(g[k + "_bits"]))
        assert np.array_equal(logits, g[k + "_logits"]), k
        loss, lg = O.softmax_xent(logits, g[k + "_labels"])
        assert loss == float(g[k + "_loss"]), k
        for j, t in enumerate(tapes):
            if t is not None and "q" in t:
                assert np.array_equal(t["q"]["codes"], g[f"{k}_codes{j}"]), (k, j)
        O.net_bwd(spec, params, tapes, lg)
        for j, p in enumerate(params):
            assert rel_err(p["grad_weight"], g[f"{k}_gw{j}"], 1e-3) < 1e-4, (k, j)
        O.sgd(params, 0.1, 0.9, 2e-4)
        for j, p in enumerate(params):
            assert rel_err(p["weight"], g[f"{k}_w{j}"], 1e-3) < 1e-5, (k, j)


def test_ref_kernels_agree_with_numpy_loop():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 3, 7, 7)).astype(np.float32)
    k = rng.standard_normal((4, 3, 3, 3)).astype(np.float32)
    a = O.conv_fwd(x, k, 2, 1)
    import os
    os.environ["QTAPE_ORACLE_NO_REF"] = "1"
    O.qtape_oracle._REF_TRIED = False
    O.qtape_oracle._REF_LIB = None
    try:
        b = O.conv_fwd(x, k, 2, 1)
    finally:
        del os.environ["QTAPE_ORACLE_NO_REF"]
        O.qtape_oracle._REF_TRIED = False
    assert np.array_equal(a, b)
