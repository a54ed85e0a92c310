"""Timing-only ablation of the captured C2 step: skip the launches of the
named qt_* entry points (results are wrong; only the step time matters)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1901_07988_b200 as P
from paper_1901_07988_b200 import _native as N, engine as E

skip = set(sys.argv[1].split(",")) if len(sys.argv) > 1 and sys.argv[1] else set()
cfg = sys.argv[2] if len(sys.argv) > 2 else "C2"
real = N.call
def call(name, *args):
    if name in skip:
        return
    return real(name, *args)
N.call = call
spec = {"C2": E.resnet164_spec, "C3": E.resnet1001_spec, "C4": E.resnet152_spec}[cfg]()
nb = 64 if cfg == "C4" else 128
tr = P.Trainer(spec, nb, mode="approx", bits=4)
rng = np.random.default_rng(0)
tr.load_batch(rng.standard_normal((nb,) + tuple(spec.input_shape)).astype(np.float32),
              rng.integers(0, spec.num_classes, nb))
tr.capture()
for _ in range(5):
    tr.step_device()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    tr.step_device()
e1.record()
torch.cuda.synchronize()
print(f"skip={sorted(skip)} ms/step={e0.elapsed_time(e1)/20:.3f}")
