import torch, sys
sys.path.insert(0, '.')
from paper_1901_07988_b200 import codec, ops
n, ci, hw, co, sd, reps = [int(v) for v in sys.argv[1:7]]
x = torch.randn(n, ci, hw, hw, device="cuda")
gamma, beta = torch.rand(ci, device="cuda") + 0.5, torch.randn(ci, device="cuda") * 0.1
t = codec.quantize(x, gamma, beta, 4)
act = codec.dequantize(t, relu=True)
tn = t.as_native()
g = torch.randn(n, co, hw // sd, hw // sd, device="cuda")
gw = torch.zeros((co, ci, sd, sd), device="cuda")
for r in range(reps):
    ops.conv2d_wgrad(g, (co, ci, sd, sd), sd, 0, gw, tape=tn, in_shape=(n, ci, hw, hw))
    torch.cuda.synchronize()
    print("rep", r, flush=True)
ref = reps * torch.nn.grad.conv2d_weight(act.double(), (co, ci, sd, sd), g.double(), stride=sd)
print("err", ((gw.double() - ref).norm() / ref.norm()).item())
