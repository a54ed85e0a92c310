"""Helpers shared by the GPU parity tests (tolerances are stated here)."""

import numpy as np
import torch

# Tolerances of the parity contract:
#   codes / offsets / steps / dequantized values / SGD / matmul: bit-exact
#   conv forward & data/weight gradients (fp32-faithful GEMMs vs the
#   reference's float64 accumulation): normwise relative error <= CONV_TOL
#   one full training step (logits, loss, every gradient): normwise <= STEP_TOL
#   ... when some K-bit code landed in the neighbouring interval (a forward
#   value within an ulp of a boundary): gradients normwise <= FLIP_TOL
CONV_TOL = 1e-5
LAYER_TOL = 1e-5
STEP_TOL = 1e-4
FLIP_TOL = 2e-3
MOMENT_TOL = 1e-12


def dev(x, dtype=None):
    t = torch.as_tensor(np.ascontiguousarray(x))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def host(t):
    return t.detach().cpu().numpy()


def norm_err(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    d = np.linalg.norm(want.ravel())
    e = np.linalg.norm((got - want).ravel())
    return float(e / d) if d > 0 else float(e)
