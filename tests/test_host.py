"""Host-side logic on CPU: specs, memory accounting, pool bookkeeping."""

import json

import pytest
import torch

import paper_1901_07988_b200 as P
from paper_1901_07988_b200 import engine as E
from paper_1901_07988_b200.errors import ConfigError, ShapeError, StateError


def tiny_residual_spec(blocks=2, channels=4, hw=8, in_ch=2):
    layers = [E.LayerSpec("conv", channels, 3, 1, 1, preact=False)]
    bl = []
    for _ in range(blocks):
        bl.append((len(layers), len(layers) + 1))
        layers += [E.LayerSpec("conv", channels, 3, 1, 1), E.LayerSpec("conv", channels, 3, 1, 1)]
    layers.append(E.LayerSpec("gap_dense", 10))
    return E.NetworkSpec((in_ch, hw, hw), 10, layers, bl)


def test_width():
    ff = E.NetworkSpec((4,), 3, [E.LayerSpec("dense", 8), E.LayerSpec("dense", 3)])
    assert ff.width() == 1
    assert tiny_residual_spec().width() == 2
    assert E.make_uniform_spec(8).width() == 2
    assert E.make_uniform_spec(8, residual=False).width() == 1


@pytest.mark.parametrize("kwargs", [
    dict(input_shape=(2, 8, 8), num_classes=10,
         layers=[E.LayerSpec("conv", 4), E.LayerSpec("gap_dense", 10)], blocks=[(0, 0)]),
    dict(input_shape=(4, 16, 16), num_classes=10,
         layers=[E.LayerSpec("conv", 4, 2, 2, 0), E.LayerSpec("conv", 4, 2, 2, 0),
                 E.LayerSpec("gap_dense", 10)], blocks=[(0, 1)]),
    dict(input_shape=(2, 8, 8), num_classes=10, layers=[E.LayerSpec("conv", 4)]),
    dict(input_shape=(2, 8, 8), num_classes=10,
         layers=[E.LayerSpec("conv", 4), E.LayerSpec("conv", 4, preact=False),
                 E.LayerSpec("gap_dense", 10)]),
])
def test_rejects_bad_specs(kwargs):
    with pytest.raises(ConfigError):
        E.NetworkSpec(**kwargs)


def test_rejects_non_integral_extent():
    with pytest.raises(ShapeError):
        E.NetworkSpec((3, 32, 32), 10, [E.LayerSpec("conv", 8, 3, 2, 1),
                                        E.LayerSpec("gap_dense", 10)])


def test_json_roundtrip(tmp_path):
    spec = E.make_residual_spec()
    path = tmp_path / "spec.json"
    spec.save(str(path))
    assert E.NetworkSpec.load(str(path)).to_json() == spec.to_json()


@pytest.mark.parametrize("name,builder", [
    ("C1", lambda: E.make_residual_spec()), ("C2", E.resnet164_spec),
    ("C3", E.resnet1001_spec), ("C4", E.resnet152_spec)])
def test_memory_report_matches_reference(golden_memory, name, builder):
    """Byte-exact with the reference memory_report (engine.py:485-534)."""
    g = golden_memory[name]
    spec = builder()
    assert spec.to_json() == E.NetworkSpec.from_json(g["spec"]).to_json()
    shape = (g["batch"],) + tuple(g["spec"]["input_shape"])
    for r in g["reports"]:
        rep = E.memory_report(spec, shape, mode=r["mode"], bits=r["bits"])
        for k, v in r.items():
            if k not in ("mode", "bits"):
                assert getattr(rep, k) == v, (name, r["mode"], r["bits"], k)


def test_headline_reduction():
    spec = E.resnet164_spec()
    a = E.memory_report(spec, (128, 3, 32, 32), mode="approx", bits=4)
    assert a.persistent_tape_bytes // 128 == 1632256
    assert a.exact_persistent_bytes // 128 == 12599296
    assert 1 / a.persistent_ratio_vs_exact >= 6.0


def test_ratios_like_reference():
    rep = E.memory_report(E.make_uniform_spec(40), (2, 8, 16, 16), mode="approx", bits=8)
    assert abs(rep.persistent_ratio_vs_exact - 0.25) < 0.02
    rep = E.memory_report(E.make_uniform_spec(164), (2, 8, 16, 16), mode="approx", bits=4)
    assert abs(rep.ratio_vs_exact - (3 / 164 + 1 / 8)) < 0.01
    rep = E.memory_report(E.make_residual_spec(), (8, 3, 32, 32), mode="approx", bits=4)
    assert rep.total_bytes == (rep.persistent_tape_bytes + rep.channel_overhead_bytes
                               + rep.transient_buffer_bytes + rep.parameter_bytes)


def test_pool_bookkeeping_cpu():
    pool = E.BufferPool(3, device="cpu")
    a = pool.acquire((2, 3))
    b = pool.acquire((4,))
    c = pool.replace(a, (5,))
    assert pool.live_count == 2 and pool.peak_live_bytes == (6 + 4) * 4
    pool.acquire((1,))
    with pytest.raises(StateError):
        pool.acquire((1,))
    pool.release(b)
    pool.release(c)
    pool.release_all()
    assert pool.live_count == 0 and pool.peak_live_count == 3


def test_train_config():
    cfg = P.TrainConfig(total_iters=64000)
    assert P.lr_at(cfg, 200) == pytest.approx(1e-2)
    assert P.lr_at(cfg, 1000) == pytest.approx(1e-1)
    assert P.lr_at(cfg, 50000) == pytest.approx(1e-3)
    with pytest.raises(ConfigError):
        P.TrainConfig(lr_schedule=[(5, 0.1)])
    again = P.TrainConfig.from_json(P.TrainConfig(mode="approx", bits=4, seed=3).to_json())
    assert again.to_json()["bits"] == 4 and again.seed == 3


def test_conv_out_shape_rule():
    from paper_1901_07988_b200.ops import conv2d_out_shape
    assert conv2d_out_shape((2, 3, 32, 32), (8, 3, 2, 2), 2, 0) == (2, 8, 16, 16)
    with pytest.raises(ShapeError):
        conv2d_out_shape((2, 3, 32, 32), (8, 3, 3, 3), 2, 1)


def test_synth_styles_match_reference():
    """The block-style corpora (sparse / natural / smooth) draw the reference
    generator's random numbers in its order: byte-identical to
    qtape.data.synth_cifar_like (digests from tests/golden/make_golden_synth.py)."""
    import hashlib
    import json
    import os

    from paper_1901_07988_b200 import data as D
    path = os.path.join(os.path.dirname(__file__), "golden", "synth_styles.json")
    for case in json.load(open(path)):
        images, labels = D.synth_cifar_images(case["seed"], case["n"], noise=case["noise"],
                                              style=case["style"])
        h = hashlib.sha256(images.tobytes() + labels.astype("int64").tobytes()).hexdigest()
        assert h == case["sha256"], case["style"]
