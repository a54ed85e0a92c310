"""One large quantize + dequantize (ncu target): python scripts/one_codec.py N C HW K"""
import sys
import torch
sys.path.insert(0, ".")
from paper_1901_07988_b200 import codec

n, c, hw, k = (int(v) for v in sys.argv[1:5])
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(n, c, hw, 1, device="cuda", generator=g).mul_(3).add_(1)
gamma = torch.rand(c, device="cuda", generator=g) * 1.5 + 0.5
beta = torch.rand(c, device="cuda", generator=g) * 2 - 1
codes = torch.empty(codec.packed_nbytes(x.numel(), k), dtype=torch.uint8, device="cuda")
t = codec.quantize(x, gamma, beta, k, codes_out=codes)
out = torch.empty_like(x)
codec.dequantize(t, out=out)
torch.cuda.synchronize()
print("ok")
