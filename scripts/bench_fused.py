"""Microbenchmark of qt_conv_forward_fused on C2 layer shapes: plain conv,
prologue only, epilogue only, both (device time per call, CUDA graph of
20 calls)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1901_07988_b200 import _native as N, ops
from paper_1901_07988_b200.layer import TapeSlot

SHAPES = [(128, 16, 32, 64, 1, 0), (128, 64, 32, 16, 1, 0), (128, 16, 32, 16, 3, 1),
          (128, 32, 16, 32, 3, 1), (128, 64, 8, 64, 3, 1), (128, 64, 8, 256, 1, 0),
          (128, 256, 8, 64, 1, 0)]


def timeit(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    rng = np.random.default_rng(0)
    for (n, ci, h, co, k, pad) in SHAPES:
        x = torch.tensor(rng.standard_normal((n, ci, h, h)).astype(np.float32), device="cuda")
        w = torch.tensor((rng.standard_normal((co, ci, k, k)) * 0.2).astype(np.float32), device="cuda")
        out = torch.empty((n, co, h + 2 * pad - k + 1, h + 2 * pad - k + 1), device="cuda")
        g = torch.ones(ci, device="cuda"); b = torch.zeros(ci, device="cuda")
        slot = TapeSlot((n, ci, h, h), ci, 4, False, x.device)
        rm = torch.zeros(ci, dtype=torch.float64, device="cuda"); rv = torch.ones_like(rm)
        sws = ops.workspace(N.query("qt_bn_stats_workspace", n, ci, h * h), x.device, "stats")
        N.call("qt_bn_stats_prep", N.ptr(x), n, ci, h * h, 1e-5, N.ptr(g), N.ptr(b), 4,
               N.ptr(slot.mean), N.ptr(slot.var), N.ptr(rm), N.ptr(rv), N.ptr(slot.gamma),
               N.ptr(slot.beta), N.ptr(slot.step), N.ptr(slot.offset), N.ptr(slot.clip),
               N.ptr(slot.consts), N.ptr(sws))
        g2 = torch.ones(co, device="cuda"); b2 = torch.zeros(co, device="cuda")
        s2 = TapeSlot(tuple(out.shape), co, 4, False, x.device)
        rm2 = torch.zeros(co, dtype=torch.float64, device="cuda"); rv2 = torch.ones_like(rm2)
        fws = torch.zeros(N.query("qt_conv_stats_workspace", co), dtype=torch.uint8, device="cuda")
        epi = N.BnStatsEpilogue(1e-5, N.ptr(g2), N.ptr(b2), 4, N.ptr(s2.mean), N.ptr(s2.var),
                                N.ptr(rm2), N.ptr(rv2), N.ptr(s2.gamma), N.ptr(s2.beta),
                                N.ptr(s2.step), N.ptr(s2.offset), N.ptr(s2.clip), N.ptr(s2.consts),
                                N.ptr(fws))
        pro = N.BnPrologue(N.ptr(slot.consts), N.ptr(slot.codes), N.ptr(slot.clip), 4)
        ws = ops._conv_ws(w, None, tuple(x.shape), 1, pad)
        res = {}
        for name, pp, ee in (("plain", None, None), ("pro", pro, None), ("epi", None, epi),
                             ("both", pro, epi)):
            res[name] = timeit(lambda: ops.conv2d_forward_fused(x, w, 1, pad, out, ws=ws,
                                                                 prologue=pp, epilogue=ee))
        print((n, ci, h, co, k), " ".join(f"{k_}={v:.1f}us" for k_, v in res.items()), flush=True)


if __name__ == "__main__":
    main()
