"""Golden fixtures of the input pipeline and the diagnostics from the
UNMODIFIED reference.  Run here:

    PYTHONPATH=/root/reference/pkg/src XDG_CACHE_HOME=/tmp/qtape_cache \
        python tests/golden/make_golden_data.py

data.npz:
* rec_train / rec_test -- the raw CIFAR binary records of a small synthetic
  corpus (reference make_synthetic_cifar_dir, data.py:168-179);
* the reference load_cifar10 of them (data.py:60-87): images, labels,
  norm mean / std, and the test split standardized with the train stats;
* augment_batch (data.py:182-206) of 8 images with a seeded generator keyed
  like training.py:193-196;
* training.train's augmentation-on run (training.py:169-203): losses of 4
  iterations of a tiny net (approx, K=4, hflip + translate);
* diag (diag.py): grad_error_report, sign_agreement, quantizer_check and
  naive_vs_proposed_depth_sweep on the same data.
"""

import json
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("XDG_CACHE_HOME", "/tmp/qtape_cache")

from qtape import data as D  # noqa: E402
from qtape import diag as G  # noqa: E402
from qtape import engine as E  # noqa: E402
from qtape import training as T  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    out = {}
    d = tempfile.mkdtemp(prefix="qtape-golden-data-")
    D.make_synthetic_cifar_dir(d, seed=3, train_n=64, test_n=16)
    out["rec_train"] = np.fromfile(os.path.join(d, "data_batch_1.bin"), dtype=np.uint8)
    out["rec_test"] = np.fromfile(os.path.join(d, "test_batch.bin"), dtype=np.uint8)
    tr = D.load_cifar10(d)
    te = D.load_cifar10(d, "test", norm_stats=(tr.norm_mean, tr.norm_std))
    out.update(images=tr.images, labels=tr.labels, mean=tr.norm_mean, std=tr.norm_std,
               images_test=te.images, labels_test=te.labels)
    rng = np.random.default_rng(np.random.SeedSequence((5, 0, 3)))
    out["aug"] = D.augment_batch(tr.images[:8], rng)
    rng = np.random.default_rng(np.random.SeedSequence((5, 1, 2)))
    out["aug_flip_only"] = D.augment_batch(tr.images[8:16], rng, hflip=True, translate=False)
    # training with augmentation (the engine's default config path)
    spec = G.make_sweep_spec(6, (3, 32, 32))
    out["train_spec"] = json.dumps(spec.to_json())
    cfg = T.TrainConfig(mode="approx", bits=4, batch_size=16, total_iters=4, seed=7,
                        lr_schedule=[[0, 0.05]])
    res = T.train(spec, cfg, tr)
    out["train_losses"] = np.array([r[1] for r in res.records])
    # diagnostics
    params = T.init_params(spec, 0)
    rep = G.grad_error_report(spec, params, tr, bits=4, batches=3, batch_size=8, seed=1)
    out["ger_approx_error"] = np.array([r["approx_error"] for r in rep.rows])
    out["ger_sgd_noise"] = np.array([r["sgd_noise"] for r in rep.rows])
    rows = G.sign_agreement(spec, T.init_params(spec, 0), tr, bits=4, batch_size=8, seed=2)
    out["sign_layers"] = np.array([r["layer"] for r in rows])
    out["sign_table"] = np.array([[r["clipped_fraction"], r["unclipped_match"], r["clipped_match"],
                                   r["overall_match"]] for r in rows])
    q = G.quantizer_check(4, n=4096, seed=3)
    out["qc"] = np.array([q["clipped_fraction"], q["ok"]], dtype=np.float64)
    rows = G.naive_vs_proposed_depth_sweep([4, 6], 4, tr, seed=0, batches=2, batch_size=8)
    out["sweep"] = np.array([[r["depth"], r["proposed_error"], r["naive_error"]] for r in rows])
    np.savez_compressed(os.path.join(HERE, "data.npz"), **out)
    print("wrote", os.path.join(HERE, "data.npz"), sorted(out))


if __name__ == "__main__":
    main()
