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
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--only", type=int, default=-1)
ap.add_argument("--bits", type=int, default=4)
a = ap.parse_args()
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
    tape = codec.quantize(x, gamma, beta, a.bits).as_native()
    gout = torch.randn(n, co, h, w, device=dev, generator=g)
    gw = torch.zeros(co, ci, k, k, device=dev)
    ws = None
    run = lambda: ops.conv2d_wgrad(gout, (co, ci, k, k), 1, pad, gw, tape=tape,
                                   in_shape=(n, ci, h, w))
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
    print(f"{i}: n={n} ci={ci} {h}x{w} co={co} k={k}: {us:8.2f} us  (MMA floor {floor_us:6.2f} us)")
