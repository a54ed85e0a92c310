"""One eager C2 training step for ncu (launch list / per-kernel capture).

    python scripts/profile_step.py [--config C2] [--warmup 1] [--steps 1]

Runs the same Trainer as bench.py but without the CUDA graph so every
kernel is a separate, attributable launch."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1901_07988_b200 as P
from paper_1901_07988_b200 import engine as E

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--bits", type=int, default=4)
a = ap.parse_args()
builders = {"C1": (E.make_residual_spec, 32), "C2": (E.resnet164_spec, 128),
            "C3": (E.resnet1001_spec, 128), "C4": (E.resnet152_spec, 64)}
b, n = builders[a.config]
spec = b()
tr = P.Trainer(spec, n, mode="approx", bits=a.bits, use_graph=False)
rng = np.random.default_rng(0)
tr.load_batch(rng.standard_normal((n,) + spec.input_shape).astype(np.float32),
              rng.integers(0, spec.num_classes, n))
for _ in range(a.warmup + a.steps):
    tr.step_device()
torch.cuda.synchronize()
print("ok", float(tr.loss_buf[0]))
