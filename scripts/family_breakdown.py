"""Per-call device times of one entry point's calls in a C2 step (graph with
event nodes between calls).  python scripts/family_breakdown.py qt_bn_backward_reduce"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1901_07988_b200 as P
from paper_1901_07988_b200 import _native as N, engine as E

fam = sys.argv[1] if len(sys.argv) > 1 else "qt_bn_backward_reduce"
spec = E.resnet164_spec()
tr = P.Trainer(spec, 128, mode="approx", bits=4)
rng = np.random.default_rng(0)
tr.load_batch(rng.standard_normal((128,) + spec.input_shape).astype(np.float32),
              rng.integers(0, 10, 128))
tr.capture()
tr.step_device()
rec = bench.CallRecorder()
hold = torch.cuda.CUDAGraph()
cs = torch.cuda.Stream()
cs.wait_stream(torch.cuda.current_stream())
N.hook = rec
with torch.cuda.stream(cs):
    with torch.cuda.graph(hold, stream=cs):
        tr._body()
N.hook = None
torch.cuda.synchronize()
calls = [a for n, a in rec.calls if n == fam]
fn = getattr(N.lib(), fam)
ts = []
for a in calls:   # one small graph per call, replayed between events
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(cs):
        with torch.cuda.graph(g, stream=cs):
            for _ in range(5):
                fn(*a, N.stream())
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(cs):
        e0.record(cs)
        g.replay()
        e1.record(cs)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3 / 5)
print(f"{fam}: {len(calls)} calls, total {sum(ts):.1f} us")
from collections import defaultdict
by = defaultdict(list)
for a, t in zip(calls, ts):
    key = tuple(x for x in a if isinstance(x, int) and not isinstance(x, bool) and x < 1 << 32)[:6]
    by[key].append(t)
for k, v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
    print(f"  {str(k):40s} n={len(v):3d} avg {sum(v)/len(v):7.2f} us  total {sum(v):8.1f}")
