import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_07988_b200 import ops, _native as N
dev = torch.device("cuda:0")
lib = N.lib(); fn = lib.qt_debug_wgrad_trace; fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
x = torch.randn(128, 3, 32, 32, device=dev)
go = torch.randn(128, 16, 32, 32, device=dev)
gw = torch.zeros(16, 3, 3, 3, device=dev)
buf = torch.zeros(4000, dtype=torch.int64, device=dev)
fn(buf.data_ptr(), 0)
ops.conv2d_wgrad(go, (16, 3, 3, 3), 1, 1, gw, x_plain=x)
torch.cuda.synchronize(); fn(None, 0)
print("trace nonzero:", int((buf != 0).sum()))
ref = torch.nn.grad.conv2d_weight(x.double(), (16, 3, 3, 3), go.double(), padding=1)
print("err", float((gw.double() - ref).abs().max() / ref.abs().max()))
