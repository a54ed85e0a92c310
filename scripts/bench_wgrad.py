"""Micro-benchmark of the conv weight-gradient from a K-bit tape (C2 shapes).

    python scripts/bench_wgrad.py [--iters 20] [--only IDX] [--bits 4]

Times qt_conv_wgrad (kernel + fixed-order split reduction) per layer shape
with CUDA events on the launching stream; --only runs one shape once (for
ncu)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_1901_07988_b200 import codec, ops

# (n, ci, h, w, co, k, pad): the ResNet-164 bottleneck shapes at batch 128
SHAPES = [
    (128, 64, 32, 32, 16, 1, 0), (128, 16, 32, 32, 16, 3, 1), (128, 16, 32, 32, 64, 1, 0),
    (128, 128, 16, 16, 32, 1, 0), (128, 32, 16, 16, 32, 3, 1), (128, 32, 16, 16, 128, 1, 0),
    (128, 256, 8, 8, 64, 1, 0), (128, 64, 8, 8, 64, 3, 1), (128, 64, 8, 8, 256, 1, 0),
]

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2", choices=["C2", "C4"])
ap.add_argument("--op", default="wgrad", choices=["wgrad", "fwd", "dgrad"])
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--only", type=int, default=-1)
ap.add_argument("--bits", type=int, default=4)
a = ap.parse_args()
MULT = [1] * len(SHAPES)
STRIDE = [1] * len(SHAPES)
if a.config == "C4":   # distinct conv layers of ResNet-152 224^2 at batch 64, with multiplicity
    from collections import Counter
    import paper_1901_07988_b200 as P
    spec = P.resnet152_spec()
    cnt = Counter()
    for l, (ins, _) in zip(spec.layers, spec.layer_shapes(64)):
        if l.kind == "conv":
            cnt[(ins[0], ins[1], ins[2], ins[3], l.out_channels, l.kernel, l.pad, l.stride)] += 1
    SHAPES = [k[:7] for k in cnt]
    STRIDE = [k[7] for k in cnt]
    MULT = list(cnt.values())
total_us = 0.0
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
_w = torch.randn(1 << 26, device=dev)      # ~0.3 s of work: clocks up before the first shape
for _ in range(200):
    _w.mul_(1.0)
torch.cuda.synchronize()
for i, (n, ci, h, w, co, k, pad) in enumerate(SHAPES):
    if a.only >= 0 and i != a.only:
        continue
    x = torch.randn(n, ci, h, w, device=dev, generator=g)
    gamma = torch.rand(ci, device=dev, generator=g) + 0.5
    beta = torch.randn(ci, device=dev, generator=g) * 0.1
    qtape = codec.quantize(x, gamma, beta, a.bits)   # keeps the codes alive
    tape = qtape.as_native()
    sd = STRIDE[i]
    oh, ow = (h + 2 * pad - k) // sd + 1, (w + 2 * pad - k) // sd + 1
    gout = torch.randn(n, co, oh, ow, device=dev, generator=g)
    gw = torch.zeros(co, ci, k, k, device=dev)
    if a.op == "wgrad":
        run = lambda: ops.conv2d_wgrad(gout, (co, ci, k, k), sd, pad, gw, tape=tape,
                                       in_shape=(n, ci, h, w))
    elif a.op == "fwd":
        yb = torch.empty(n, co, oh, ow, device=dev)
        run = lambda: ops.conv2d_forward(x, gw, sd, pad, out=yb)
    else:
        gxb = torch.empty(n, ci, h, w, device=dev)
        run = lambda: ops.conv2d_dgrad(gout, gw, (n, ci, h, w), sd, pad, gxb)
    if a.only >= 0:
        run()
        torch.cuda.synchronize()
        print("ok", i)
        continue
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    # capture the launches so host overhead does not pace the GPU
    graph = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        with torch.cuda.graph(graph, stream=cs):
            for _ in range(a.iters):
                run()
    graph.replay()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    graph.replay()
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / a.iters
    R = ci * k * k
    mt = (R + 127) // 128
    floor_us = (n * h * w / 32) * mt * 8 * 46 / 148 / 1.965e3   # 2 tf32 passes, 46 clk/MMA
    total_us += us * MULT[i]
    tflops = 2.0 * n * oh * ow * co * ci * k * k / us / 1e6
    print(f"{i}: n={n} ci={ci} {h}x{w} co={co} k={k}/s{sd} x{MULT[i]}: {us:8.2f} us "
          f"{tflops:6.1f} TF/s (MMA floor {floor_us:6.2f} us)")
print(f"total {a.op}: {total_us / 1e3:.2f} ms per step")
