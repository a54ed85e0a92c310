"""Per-chunk timeline of one wgrad CTA (debug hook qt_debug_wgrad_trace)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1901_07988_b200 import _native as N, codec, ops

shape = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "128,16,32,32,16,3,1").split(",")]
n, ci, h, w, co, k, pad = shape
dev = torch.device("cuda:0")
x = torch.randn(n, ci, h, w, device=dev)
if os.environ.get("WIDE"):   # offsets beyond the FAST range: GENERIC CTAs
    tape = codec.quantize(x, torch.rand(ci, device=dev) * 0.05 + 0.05, torch.rand(ci, device=dev) + 1.5,
                          4).as_native()
else:
    tape = codec.quantize(x, torch.rand(ci, device=dev) + 0.5, torch.randn(ci, device=dev) * 0.1,
                          4).as_native()
gout = torch.randn(n, co, h, w, device=dev)
gw = torch.zeros(co, ci, k, k, device=dev)
lib = N.lib()
fn = lib.qt_debug_wgrad_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
if os.environ.get("PLAIN"):
    run = lambda: ops.conv2d_wgrad(gout, (co, ci, k, k), 1, pad, gw, x_plain=x)
else:
    run = lambda: ops.conv2d_wgrad(gout, (co, ci, k, k), 1, pad, gw, tape=tape, in_shape=(n, ci, h, w))
run()
torch.cuda.synchronize()
for cta in (0,):
    buf = torch.zeros(4000, dtype=torch.int64, device=dev)
    fn(buf.data_ptr(), cta)
    run()
    torch.cuda.synchronize()
    fn(None, 0)
    b = buf.cpu().tolist()
    t0 = b[0]
    print(f"CTA {cta}: globaltimer start {b[332]} end {b[333]} dur {(b[333]-b[332])/1e3:.2f} us;"
          f" fast {b[525]} setup {b[1]-t0} cyc, epi start {b[330]-t0}, end {b[331]-t0}")
    print("  i  prod  opraw  opempty  split0  dec0  split1  dec1  opdone  mma  lastwarp_done  mma_committed")
    for i in range(64):
        r = b[2 + 5 * i: 7 + 5 * i]
        if not any(r):
            break
        r = r[:3] + b[3700 + 4 * i: 3704 + 4 * i] + r[3:] + b[400 + 2 * i: 402 + 2 * i]
        print(f"{i:3d} " + " ".join(f"{(v - t0) if v else -1:7d}" for v in r))

    import collections
    st = [(b[600 + 3 * j], b[601 + 3 * j], b[602 + 3 * j]) for j in range(1024) if b[600 + 3 * j]]
    t0g = min(x[0] for x in st)
    print(f"CTAs {len(st)}: span {(max(x[1] for x in st) - t0g) / 1e3:.2f} us")
    d = sorted((x[1] - x[0]) / 1e3 for x in st)
    print("  duration us: min %.2f med %.2f max %.2f" % (d[0], d[len(d) // 2], d[-1]))
    starts = sorted((x[0] - t0g) / 1e3 for x in st)
    print("  start us quantiles:", [round(starts[int(q * (len(starts) - 1))], 2) for q in (0, .25, .5, .75, .9, 1)])
    per_sm = collections.Counter(x[2] for x in st)
    print("  SMs used", len(per_sm), "max CTAs/SM", max(per_sm.values()))
