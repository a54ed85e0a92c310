"""Debug: which Python call sites launch torch fill kernels inside one step."""
import os
import sys
import traceback
from collections import Counter

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1901_07988_b200 as P
from paper_1901_07988_b200 import engine as E

spec = E.resnet164_spec()
tr = P.Trainer(spec, 128, mode="approx", bits=4, use_graph=False)
rng = np.random.default_rng(0)
tr.load_batch(rng.standard_normal((128,) + spec.input_shape).astype(np.float32),
              rng.integers(0, 10, 128))
tr.step_device()
torch.cuda.synchronize()
sites = Counter()
orig_zero, orig_fill, orig_zeros = torch.Tensor.zero_, torch.Tensor.fill_, torch.zeros


def site():
    st = traceback.extract_stack()[-3]
    return f"{os.path.basename(st.filename)}:{st.lineno}"


def z(self):
    sites["zero_ " + site()] += 1
    return orig_zero(self)


def f(self, v):
    sites["fill_ " + site()] += 1
    return orig_fill(self, v)


def zs(*a, **k):
    sites["zeros " + site()] += 1
    return orig_zeros(*a, **k)


torch.Tensor.zero_, torch.Tensor.fill_, torch.zeros = z, f, zs
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    tr.step_device()
    torch.cuda.synchronize()
print(sites.most_common(20))
rows = [(e.key, e.count, e.device_time_total) for e in prof.key_averages() if e.device_time_total > 0]
tot = sum(r[2] for r in rows)
print(f"total device time {tot / 1000:.3f} ms")
fam = Counter()
for k, c, t in rows:
    name = k.split("(")[0].replace("void ", "")
    fam[name.split("<")[0]] += t
for k, t in fam.most_common(25):
    print(f"{t / 1000:8.3f} ms  {k}")
print()
for k, c, t in sorted(rows, key=lambda r: -r[2])[:30]:
    print(f"{t / 1000:8.3f} ms {c:5d}x {t / c:8.2f} us  {k[:90]}")
