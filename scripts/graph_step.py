"""One captured C2 step replay (for ncu --graph-profiling node launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1901_07988_b200 as P
from paper_1901_07988_b200 import engine as E
spec = E.resnet164_spec()
tr = P.Trainer(spec, 128, mode="approx", bits=4)
rng = np.random.default_rng(0)
tr.load_batch(rng.standard_normal((128,) + spec.input_shape).astype(np.float32), rng.integers(0, 10, 128))
tr.capture()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
tr.step_device()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
