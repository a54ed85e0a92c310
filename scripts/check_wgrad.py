"""Debug: TC wgrad from a tape vs a float64 torch reference, error by row/col."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1901_07988_b200 import codec, ops

cases = [
    (2, 16, 32, 16, 3, 1, 4, "narrow"), (2, 16, 32, 16, 3, 1, 4, "wide"), (2, 16, 32, 16, 1, 0, 4, "wide"),
    (2, 32, 16, 32, 3, 1, 2, "narrow"), (2, 16, 32, 16, 3, 1, 8, "narrow"), (2, 16, 32, 16, 3, 1, 0, "plain"),
]
torch.manual_seed(0)
dev = torch.device("cuda:0")
for n, ci, hw, co, k, pad, bits, regime in cases:
    x = torch.randn(n, ci, hw, hw, device=dev)
    gamma = torch.rand(ci, device=dev) + 0.5
    beta = torch.randn(ci, device=dev) * 0.1
    if regime == "wide":
        gamma = torch.rand(ci, device=dev) * 0.05 + 0.05
        beta = torch.rand(ci, device=dev) * 1.5 + 1.5
    gout = torch.randn(n, co, hw, hw, device=dev)
    gw = torch.zeros(co, ci, k, k, device=dev)
    if bits:
        t = codec.quantize(x, gamma, beta, bits)
        act = codec.dequantize(t, relu=True)
        ops.conv2d_wgrad(gout, (co, ci, k, k), 1, pad, gw, tape=t.as_native(), in_shape=(n, ci, hw, hw))
    else:
        act = x
        ops.conv2d_wgrad(gout, (co, ci, k, k), 1, pad, gw, x_plain=x)
    ref = torch.nn.grad.conv2d_weight(act.double(), (co, ci, k, k), gout.double(), padding=pad)
    err = (gw.double() - ref).abs()
    rel = (err.norm() / ref.norm()).item()
    print(f"{(n, ci, hw, co, k, pad, bits, regime)}: rel {rel:.3e}")
    if rel > 1e-5:
        e = err.reshape(co, -1)
        print("  worst rows (ci,u,v flat):", e.amax(0).topk(8).indices.tolist())
        print("  worst co:", e.amax(1).topk(8).indices.tolist())
        print("  row err profile:", [f"{v:.1e}" for v in e.amax(0)[:20].tolist()])
        print("  ref row scale:", [f"{v:.1e}" for v in ref.reshape(co, -1).abs().amax(0)[:20].tolist()])
