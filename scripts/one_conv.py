"""Run one conv forward (for ncu): python scripts/one_conv.py n,ci,h,co,k,pad"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1901_07988_b200 import ops

n, ci, h, co, k, pad = [int(v) for v in sys.argv[1].split(",")]
x = torch.randn(n, ci, h, h, device="cuda")
w = torch.randn(co, ci, k, k, device="cuda") * 0.1
for _ in range(2):
    ops.conv2d_forward(x, w, 1, pad)
torch.cuda.synchronize()
print("ok")
