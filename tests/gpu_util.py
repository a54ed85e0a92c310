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
#   a layer of a deep network, given the input the engine passed it:
#   output normwise <= local_tol(K) (the conv's split-precision products
#   accumulate in fp32 on the tensor cores, the reference in float64, so the
#   difference grows like sqrt(K) for a contraction of K = ci*kh*kw terms:
#   LOCAL_TOL up to K = 400, 5e-7 * sqrt(K) beyond -- 1.6e-5 at the
#   ImageNet 1x1 512x4 -> 512 transition, K = 2048)
LOCAL_TOL = 1e-5


def local_tol(k_contract: int) -> float:
    return max(LOCAL_TOL, 5e-7 * float(np.sqrt(k_contract)))
#   a whole forward pass of L layers against the free-running oracle: the
#   per-layer differences compound through the residual stream, so logits
#   and loss are held to DRIFT_PER_LAYER * L (2e-6 / layer: ResNet-164
#   measures ~0.6e-6 / layer, ResNet-1001 ~0.5e-6 / layer)
DRIFT_PER_LAYER = 2e-6


def drift_tol(depth: int) -> float:
    """End-to-end tolerance of an L-layer network: STEP_TOL for shallow
    nets, DRIFT_PER_LAYER * L once depth dominates."""
    return max(STEP_TOL, DRIFT_PER_LAYER * depth)


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


# Network-level code agreement.  With identical A2 the codes are bit-exact
# (test_layer_gpu.py); through a whole network the layer inputs carry the
# fp32-level error of the split-precision convolutions upstream, so an A2
# lying within that error of a quantization boundary can take the
# neighbouring code.  Every such flip must be explained: the two codes are
# neighbours and the oracle's A2 * scale lies within FLIP_TAU code intervals
# of the boundary between them.  FLIP_TAU = 1e-4 intervals: A2 moves by
# (relative input error) * 2^K/6 intervals, i.e. 2.7e-6 at K=4 for a 1e-6
# relative conv error, so the bound leaves a 30x margin while a genuine codec
# or BN bug (flips at arbitrary distance from the boundaries) fails it.
FLIP_TAU = 1e-4


def code_flips(mine_packed, ref_tape, bits):
    """Compare one layer's codes with the oracle's (tape from
    ``O.net_fwd(..., keep_a2=True)``).  Returns a dict: flips, elements,
    near (oracle elements within FLIP_TAU of any boundary -- the expected
    upper bound on flips), max_dist (largest boundary distance of a flip,
    code intervals), bad (flips that are not neighbouring codes or lie
    farther than FLIP_TAU from their boundary)."""
    import oracle as O
    a2 = ref_tape["a2_pre"]
    shape = a2.shape
    numel = a2.size
    mine = O.unpack(mine_packed, bits, numel).astype(np.int64)
    ref = O.unpack(ref_tape["q"]["codes"], bits, numel).astype(np.int64)
    scale, _, off = O.code_constants(ref_tape["gamma"], ref_tape["beta"], bits)
    c = shape[1]
    hw = numel // (shape[0] * c)
    ch_all = (np.arange(numel) // hw) % c
    t = a2.reshape(-1).astype(np.float64) * scale[ch_all]
    frac = np.abs(t - np.round(t))
    near = int(np.count_nonzero(frac <= FLIP_TAU))
    idx = np.nonzero(mine != ref)[0]
    out = {"flips": int(idx.size), "elements": int(numel), "near": near, "max_dist": 0.0,
           "bad": 0}
    if idx.size:
        ch = ch_all[idx]
        hi = np.maximum(mine[idx], ref[idx])
        boundary = hi - (1 << (bits - 1)) + off[ch]
        dist = np.abs(t[idx] - boundary)
        neighbour = np.abs(mine[idx] - ref[idx]) == 1
        out["max_dist"] = float(dist.max())
        out["bad"] = int(np.count_nonzero(~neighbour | (dist > FLIP_TAU)))
    return out
