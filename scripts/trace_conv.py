"""Per-stage timeline of one conv-forward CTA (debug hook qt_debug_conv_trace)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1901_07988_b200 import _native as N, ops

shape = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "128,16,32,16,3,1").split(",")]
n, ci, h, co, k, pad = shape
dev = torch.device("cuda:0")
x = torch.randn(n, ci, h, h, device=dev)
w = torch.randn(co, ci, k, k, device=dev) * 0.1
run = lambda: ops.conv2d_forward(x, w, 1, pad)
run()
torch.cuda.synchronize()
fn = N.lib().qt_debug_conv_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = torch.zeros(1002, dtype=torch.int64, device=dev)
fn(buf.data_ptr(), 0)
run()
torch.cuda.synchronize()
fn(None, 0)
b = buf.cpu().tolist()
t0 = b[1000]
rel = lambda v: (v - t0) if v else -1
print(f"CTA 0: total {b[1001] - t0} cycles  R={b[990]} G={b[991]} OPS={b[992]}")
print("  gi  prod  s_raw  s_empty  s_done(q2)  mma_go  mma_issued  mma_pre_wait  s_done(q0)")
for gi in range(64):
    r = b[8 * gi: 8 * gi + 8]
    if not any(r):
        break
    print(f"{gi:4d} " + " ".join(f"{rel(v):7d}" for v in r))
print("  tile  epi_go  epi_stored  ldtm_done  compute_done")
for lt in range(32):
    r = b[600 + 4 * lt: 600 + 4 * lt + 4]
    if not any(r):
        break
    print(f"{lt:4d} " + " ".join(f"{rel(v):7d}" for v in r))
