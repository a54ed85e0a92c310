import numpy as np, torch, sys
sys.path.insert(0, '.')
import oracle as O
from paper_1901_07988_b200 import ops, _native as N
geo = tuple(int(v) for v in sys.argv[1].split(","))
n, ci, h, co, k, s, p = geo
rng = np.random.default_rng(0)
x = rng.standard_normal((n, ci, h, h)).astype(np.float32)
w = rng.standard_normal((co, ci, k, k)).astype(np.float32)
want = O.conv_fwd(x, w, s, p)
xd = torch.from_numpy(x).cuda(); wd = torch.from_numpy(w).cuda()
out = torch.full(want.shape, 7.0, device="cuda")
ws = torch.zeros(1 << 22, dtype=torch.uint8, device="cuda")
try:
    N.call("qt_conv_forward", N.ptr(xd), N.ptr(wd), N.ptr(out), n, ci, h, h, co, k, k, s, p, None, 0, 1, N.ptr(ws))
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    print(geo, "tc", N.query("qt_conv_uses_tc", n, ci, h, h, co, k, k, s, p, 0), "rel err", np.linalg.norm(got-want)/np.linalg.norm(want))
except Exception as e:
    print(geo, "ERR", str(e).splitlines()[0])
