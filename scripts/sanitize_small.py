"""Small workload for compute-sanitizer (tests/test_sanitizer_gpu.py): one
tensor-core forward / data-gradient / weight-gradient conv each (3x3 row
tiles, 1x1, kernel == stride), the fused forward (BN prologue + statistics
epilogue), and one approx training step of a 2-block network with the
side-stream weight gradients on.  Exits 0; the sanitizer reports errors."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1901_07988_b200 as P  # noqa: E402
from paper_1901_07988_b200 import engine as E, ops  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    dev = torch.device("cuda", 0)
    for (n, ci, h, co, k, s, p) in [(2, 16, 16, 32, 3, 1, 1), (2, 32, 8, 64, 1, 1, 0),
                                    (2, 16, 16, 16, 2, 2, 0)]:
        x = torch.tensor(rng.standard_normal((n, ci, h, h)).astype(np.float32), device=dev)
        w = torch.tensor(rng.standard_normal((co, ci, k, k)).astype(np.float32), device=dev)
        y = ops.conv2d_forward(x, w, s, p)
        g = torch.randn_like(y)
        ops.conv2d_backward(x, w, g, s, p)
    layers = [E.LayerSpec("conv", 16, 3, 1, 1, preact=False)]
    blocks = []
    for _ in range(2):
        blocks.append((len(layers), len(layers) + 2))
        layers += [E.LayerSpec("conv", 16, 1, 1, 0), E.LayerSpec("conv", 16, 3, 1, 1),
                   E.LayerSpec("conv", 32 if not blocks[:-1] else 32, 1, 1, 0)]
    layers.append(E.LayerSpec("gap_dense", 10))
    spec = E.NetworkSpec((3, 16, 16), 10, layers, blocks)
    x = torch.tensor(rng.standard_normal((4, 3, 16, 16)).astype(np.float32), device=dev)
    for fuse in ("0", "1"):
        import os
        os.environ["QTAPE_FUSE"] = fuse
        params = P.init_params(spec, 0)
        logits, tapes = E.network_forward(spec, params, x, mode="approx", bits=4)
        loss, gl = P.softmax_xent(logits, np.arange(4) % 10)
        E.network_backward(spec, params, tapes, gl, x, mode="approx")
        P.sgd_step(params, 0.1, 0.9, 2e-4)
    torch.cuda.synchronize()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
