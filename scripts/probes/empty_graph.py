"""Per-node overhead of a CUDA graph of tiny kernels on this box (PDL on/off)."""
import ctypes, sys, torch
sys.path.insert(0, ".")
from paper_1901_07988_b200 import _native as N
x = torch.zeros(1024, device="cuda"); y = torch.zeros(1024, device="cuda")
for n in (100, 1000):
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        N.call("qt_copy", N.ptr(x), N.ptr(y), 1024)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                N.call("qt_copy", N.ptr(x), N.ptr(y), 1024)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(5): g.replay()
    e1.record(); torch.cuda.synchronize()
    print(n, "kernels: us per node", e0.elapsed_time(e1) * 1e3 / (5 * n))
