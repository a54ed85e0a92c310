"""Device input pipeline and diagnostics against
golden vectors of the unmodified reference (tests/golden/make_golden_data.py):
CIFAR record decode + standardization (data.py:60-87), flip / crop
augmentation (data.py:182-206), the augmented training loop
(training.py:169-203), grad_error_report / sign_agreement / quantizer_check /
the depth sweep (diag.py), and the command line (cli.py)."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from gpu_util import MOMENT_TOL, STEP_TOL, dev, host, norm_err

pytestmark = pytest.mark.gpu

import paper_1901_07988_b200 as P  # noqa: E402
from paper_1901_07988_b200 import data as D  # noqa: E402
from paper_1901_07988_b200 import diag as G  # noqa: E402
from paper_1901_07988_b200 import engine as E  # noqa: E402
from paper_1901_07988_b200.errors import DataError  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def golden():
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "data.npz")))


@pytest.fixture(scope="module")
def cifar_dir(golden, tmp_path_factory):
    d = tmp_path_factory.mktemp("cifar")
    golden["rec_train"].tofile(str(d / "data_batch_1.bin"))
    golden["rec_test"].tofile(str(d / "test_batch.bin"))
    return str(d)


def test_load_cifar10_on_device(golden, cifar_dir):
    tr = D.load_cifar10(cifar_dir)
    assert tr.on_device and tuple(tr.images.shape) == golden["images"].shape
    assert np.array_equal(tr.labels, golden["labels"])
    assert norm_err(tr.norm_mean, golden["mean"]) < MOMENT_TOL
    assert norm_err(tr.norm_std, golden["std"]) < MOMENT_TOL
    assert norm_err(host(tr.images), golden["images"]) < 1e-6
    # given the same constants the decode + standardization is bit-identical
    te = D.load_cifar10(cifar_dir, "test", norm_stats=(golden["mean"], golden["std"]))
    assert np.array_equal(host(te.images).view(np.uint32), golden["images_test"].view(np.uint32))
    assert np.array_equal(te.labels, golden["labels_test"])
    with pytest.raises(DataError):
        D.load_cifar10(cifar_dir, "test")


def test_augment_bit_identical(golden):
    imgs = dev(golden["images"][:8])
    rng = np.random.default_rng(np.random.SeedSequence((5, 0, 3)))
    out = D.augment_batch(imgs, rng)
    assert np.array_equal(host(out).view(np.uint32), golden["aug"].view(np.uint32))
    rng = np.random.default_rng(np.random.SeedSequence((5, 1, 2)))
    out = D.augment_batch(dev(golden["images"][8:16]), rng, hflip=True, translate=False)
    assert np.array_equal(host(out).view(np.uint32), golden["aug_flip_only"].view(np.uint32))


def test_train_with_device_augmentation(golden):
    spec = E.NetworkSpec.from_json(json.loads(str(golden["train_spec"])))
    ds = D.Dataset(images=dev(golden["images"]), labels=golden["labels"], num_classes=10)
    cfg = P.TrainConfig(mode="approx", bits=4, batch_size=16, total_iters=4, seed=7,
                        lr_schedule=[[0, 0.05]])
    res = P.train(spec, cfg, ds)
    losses = res.losses()
    # one step from identical parameters matches to STEP_TOL; the trajectory
    # tolerance widens per step (K-bit codes near an interval edge can flip)
    for it, (a, b) in enumerate(zip(losses, golden["train_losses"])):
        assert abs(a - b) <= STEP_TOL * 10 ** it * abs(b), (it, a, b)


def test_diagnostics_match_reference(golden):
    spec = E.NetworkSpec.from_json(json.loads(str(golden["train_spec"])))
    ds = D.Dataset(images=dev(golden["images"]), labels=golden["labels"], num_classes=10)
    rep = G.grad_error_report(spec, P.init_params(spec, 0), ds, bits=4, batches=3,
                              batch_size=8, seed=1)
    noise = np.array([r["sgd_noise"] for r in rep.rows])
    err = np.array([r["approx_error"] for r in rep.rows])
    assert np.allclose(noise, golden["ger_sgd_noise"], rtol=1e-4, atol=0)
    assert np.allclose(err, golden["ger_approx_error"], rtol=5e-2, atol=0)
    rows = G.sign_agreement(spec, P.init_params(spec, 0), ds, bits=4, batch_size=8, seed=2)
    assert [r["layer"] for r in rows] == list(golden["sign_layers"])
    tab = np.array([[r["clipped_fraction"], r["unclipped_match"], r["clipped_match"],
                     r["overall_match"]] for r in rows])
    assert np.allclose(tab, golden["sign_table"], atol=2e-3)
    q = G.quantizer_check(4, n=4096, seed=3)
    assert q["ok"] and abs(q["clipped_fraction"] - golden["qc"][0]) < 2e-3
    sw = G.naive_vs_proposed_depth_sweep([4, 6], 4, ds, seed=0, batches=2, batch_size=8)
    got = np.array([[r["depth"], r["proposed_error"], r["naive_error"]] for r in sw])
    assert np.allclose(got, golden["sweep"], rtol=5e-2)
    assert all(r["naive_error"] > r["proposed_error"] for r in sw)


def test_cli_subcommands(tmp_path):
    spec = E.make_residual_spec()
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps({"network": spec.to_json(),
                               "train": {"mode": "approx", "bits": 4, "batch_size": 32,
                                         "total_iters": 6, "lr_schedule": [[0, 0.05]]}}))
    env = dict(os.environ, TMPDIR=str(tmp_path))

    def run(*args):
        r = subprocess.run([sys.executable, "-m", "paper_1901_07988_b200", *args], cwd=ROOT,
                           env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        return r.stdout

    out = run("train", "--config", str(cfg), "--synth", "256", "--eval",
              "--out", str(tmp_path / "log.csv"))
    assert "trained 6 iterations" in out and "top-1 error" in out
    assert (tmp_path / "log.csv").read_text().startswith("iter,loss,lr,elapsed_ms")
    assert "PASS" in run("quantcheck", "--bits", "4", "--values", "20000")
    assert "persistent tape bytes" in run("memreport", "--config", str(cfg))
    assert "worst ratio" in run("gradcheck", "--config", str(cfg), "--synth", "256",
                                "--batches", "2", "--bits", "4")
    assert "depth   4" in run("sweep", "--depths", "4,6", "--batches", "2", "--synth", "256")
