"""Time plain-input / transition wgrad calls (stem, 2x2/s2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_07988_b200 import ops, codec
dev = torch.device("cuda:0")
def timeit(fn, it=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(it): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / it
x = torch.randn(128, 3, 32, 32, device=dev)
go = torch.randn(128, 16, 32, 32, device=dev)
gw = torch.zeros(16, 3, 3, 3, device=dev)
print("stem plain", timeit(lambda: ops.conv2d_wgrad(go, (16, 3, 3, 3), 1, 1, gw, x_plain=x)))
for (n, ci, h, co) in [(128, 32, 32, 32), (128, 64, 16, 64)]:
    xa = torch.randn(n, ci, h, h, device=dev)
    tape = codec.quantize(xa, torch.ones(ci, device=dev), torch.zeros(ci, device=dev), 4).as_native()
    go = torch.randn(n, co, h // 2, h // 2, device=dev)
    gw = torch.zeros(co, ci, 2, 2, device=dev)
    print("s2 tape", ci, h, timeit(lambda: ops.conv2d_wgrad(go, (co, ci, 2, 2), 2, 0, gw, tape=tape, in_shape=(n, ci, h, h))))
