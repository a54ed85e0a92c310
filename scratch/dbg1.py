import numpy as np, torch, sys
sys.path.insert(0, '.')
import oracle as O
import paper_1901_07988_b200 as P
from paper_1901_07988_b200 import ops, _native as N
x = torch.full((4, 3, 5, 5), 2.5, device="cuda")
m, v = ops.channel_moments(x)
print("const mean", m.cpu().numpy(), "var", v.cpu().numpy())
ws = ops._WS
for k, b in ws.items(): print(k, b.numel(), b[:16].cpu().numpy())
rng = np.random.default_rng(0)
x = (rng.standard_normal((8, 4, 12, 12)) * 3 + 1).astype(np.float32)
m, v = ops.channel_moments(torch.from_numpy(x).cuda())
print(m.cpu().numpy(), O.moments(x)[0])
print(v.cpu().numpy(), O.moments(x)[1])
# K1 check
shape=(4,5,8,8); bits=4; c=5
x = (rng.standard_normal(shape) * 2 + 0.5).astype(np.float32)
gamma = rng.uniform(0.5, 1.5, c).astype(np.float32); beta = rng.uniform(-0.3, 0.3, c).astype(np.float32)
mean, var = O.moments(x)
b = lambda t: t.reshape(1,-1,1,1)
a2w = ((((x - b(mean.astype(np.float32))) * b((1.0/np.sqrt(var+1e-5)).astype(np.float32))) * b(gamma)) + b(beta))
want = O.quantize(a2w, gamma, beta, bits)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
a3 = torch.empty(shape, device="cuda"); codes = torch.empty((bits*x.size+7)//8, dtype=torch.uint8, device="cuda")
step = torch.empty(c, dtype=torch.float64, device="cuda"); off = torch.empty(c, dtype=torch.int64, device="cuda"); clip = torch.zeros(1, dtype=torch.int64, device="cuda")
N.call("qt_bn_relu_forward", N.ptr(d(x)), 4, 5, 64, N.ptr(d(mean)), N.ptr(d(var)), 1e-5, N.ptr(d(gamma)), N.ptr(d(beta)), 1, bits, N.ptr(a3), None, N.ptr(codes), N.ptr(step), N.ptr(off), N.ptr(clip))
got = O.unpack(codes.cpu().numpy(), bits, x.size); ref = O.unpack(want["codes"], bits, x.size)
bad = np.nonzero(got != ref)[0]
print("mismatch", len(bad), bad[:10], got[bad[:10]], ref[bad[:10]])
print("a3 match", np.array_equal(a3.cpu().numpy(), np.maximum(a2w, 0)), np.abs(a3.cpu().numpy()-np.maximum(a2w,0)).max())
print("step", step.cpu().numpy(), want["step"]); print("off", off.cpu().numpy(), want["offset"])
