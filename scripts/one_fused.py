"""Run one fused-forward configuration eagerly (ncu target):
python scripts/one_fused.py N CI H CO K MODE   (MODE: plain | pro | epi | both)"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1901_07988_b200 import _native as N, ops
from paper_1901_07988_b200.layer import TapeSlot

n, ci, h, co, k = (int(v) for v in sys.argv[1:6])
mode = sys.argv[6]
pad = 1 if k == 3 else 0
rng = np.random.default_rng(0)
x = torch.tensor(rng.standard_normal((n, ci, h, h)).astype(np.float32), device="cuda")
w = torch.tensor((rng.standard_normal((co, ci, k, k)) * 0.2).astype(np.float32), device="cuda")
out = torch.empty((n, co, h + 2 * pad - k + 1, h + 2 * pad - k + 1), device="cuda")
g = torch.ones(ci, device="cuda"); b = torch.zeros(ci, device="cuda")
slot = TapeSlot((n, ci, h, h), ci, 4, False, x.device)
rm = torch.zeros(ci, dtype=torch.float64, device="cuda"); rv = torch.ones_like(rm)
sws = ops.workspace(N.query("qt_bn_stats_workspace", n, ci, h * h), x.device, "stats")
N.call("qt_bn_stats_prep", N.ptr(x), n, ci, h * h, 1e-5, N.ptr(g), N.ptr(b), 4, N.ptr(slot.mean),
       N.ptr(slot.var), N.ptr(rm), N.ptr(rv), N.ptr(slot.gamma), N.ptr(slot.beta),
       N.ptr(slot.step), N.ptr(slot.offset), N.ptr(slot.clip), N.ptr(slot.consts), N.ptr(sws))
g2 = torch.ones(co, device="cuda"); b2 = torch.zeros(co, device="cuda")
s2 = TapeSlot(tuple(out.shape), co, 4, False, x.device)
rm2 = torch.zeros(co, dtype=torch.float64, device="cuda"); rv2 = torch.ones_like(rm2)
fws = torch.zeros(N.query("qt_conv_stats_workspace", co), dtype=torch.uint8, device="cuda")
epi = N.BnStatsEpilogue(1e-5, N.ptr(g2), N.ptr(b2), 4, N.ptr(s2.mean), N.ptr(s2.var), N.ptr(rm2),
                        N.ptr(rv2), N.ptr(s2.gamma), N.ptr(s2.beta), N.ptr(s2.step),
                        N.ptr(s2.offset), N.ptr(s2.clip), N.ptr(s2.consts), N.ptr(fws))
pro = N.BnPrologue(N.ptr(slot.consts), N.ptr(slot.codes), N.ptr(slot.clip), 4)
ws = ops._conv_ws(w, None, tuple(x.shape), 1, pad)
pp = pro if mode in ("pro", "both") else None
ee = epi if mode in ("epi", "both") else None
for _ in range(3):
    ops.conv2d_forward_fused(x, w, 1, pad, out, ws=ws, prologue=pp, epilogue=ee)
torch.cuda.synchronize()
