import numpy as np, torch, sys
sys.path.insert(0, '.')
import oracle as O
from paper_1901_07988_b200 import ops, _native as N
for geo in [(2, 16, 8, 16, 1, 1, 0), (2,32,32,64,1,1,0), (4,16,32,16,3,1,1)]:
    n, ci, h, co, k, s, p = geo
    rng = np.random.default_rng(0)
    x = rng.standard_normal((n, ci, h, h)).astype(np.float32)
    w = rng.standard_normal((co, ci, k, k)).astype(np.float32)
    want = O.conv_fwd(x, w, s, p)
    xd = torch.from_numpy(x).cuda(); wd = torch.from_numpy(w).cuda()
    out = torch.full(want.shape, 7.0, device="cuda")
    ws = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    try:
        N.call("qt_conv_forward", N.ptr(xd), N.ptr(wd), N.ptr(out), n, ci, h, h, co, k, k, s, p, None, 0, 1, N.ptr(ws))
        torch.cuda.synchronize()
    except Exception as e:
        print("ERR", e); raise
    got = out.cpu().numpy()
    print(geo, "uses_tc", N.query("qt_conv_uses_tc", n, ci, h, h, co, k, k, s, p, 0))
    print(" got[0,0,0,:8]", got[0,0,0,:8]); print(" want", want[0,0,0,:8])
    bh = ws[: co*ci*k*k*4].view(torch.float32).cpu().numpy()
    print(" bhi[:4]", bh[:4], "w", w.reshape(co,ci,k*k).transpose(0,2,1).reshape(co,-1)[0,:4])
    print(" rel err", np.linalg.norm(got-want)/np.linalg.norm(want))
