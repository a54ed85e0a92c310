"""The reference's own property tests, restated on the device path.

Each class mirrors a test class of /root/reference/pkg/tests (test_ops.py,
test_layer.py, test_quantize.py) test by test, on float32 CUDA tensors
through this package's operator API.  Where the reference asserts exact
equality of float64 arithmetic, the device contract is stated instead:
exact where the computation is exact in fp32 (identity kernels, zero
gradients, all-ones sums, the fixed-order fp64 matmul, constant moments),
CONV_TOL / 1e-12 otherwise (tests/gpu_util.py)."""

import numpy as np
import pytest
import torch

from gpu_util import CONV_TOL, dev, host, norm_err

pytestmark = pytest.mark.gpu

import paper_1901_07988_b200 as P  # noqa: E402
from paper_1901_07988_b200 import codec, layer as L, ops  # noqa: E402
from paper_1901_07988_b200.errors import CodecError, ConfigError, ShapeError, StateError  # noqa: E402


def f32(a):
    return dev(np.asarray(a, dtype=np.float32))


class TestMatmul:   # test_ops.py:10-37
    def test_identity(self):
        b = f32([[2.0, -1.0], [0.5, 3.0]])
        assert torch.equal(ops.matmul(f32(np.eye(2)), b), b)

    def test_hand_sum(self):
        got = host(ops.matmul(f32([[1.0, 2.0], [3.0, 4.0]]), f32([[1.0], [1.0]])))
        assert np.array_equal(got, [[3.0], [7.0]])

    def test_matches_fixed_order_loop_exactly(self):
        rng = np.random.default_rng(0)
        a = rng.standard_normal((5, 7)).astype(np.float32)
        b = rng.standard_normal((7, 3)).astype(np.float32)
        want = np.zeros((5, 3), np.float32)
        for i in range(5):          # float64 accumulation in index order, one fp32 rounding
            for j in range(3):
                s = 0.0
                for k in range(7):
                    s += float(a[i, k]) * float(b[k, j])
                want[i, j] = np.float32(s)
        assert np.array_equal(host(ops.matmul(f32(a), f32(b))), want)

    def test_shape_errors(self):
        with pytest.raises(ShapeError):
            ops.matmul(f32(np.zeros((2, 3))), f32(np.zeros((4, 2))))

    def test_repeat_determinism(self):
        rng = np.random.default_rng(1)
        a, b = f32(rng.standard_normal((8, 13))), f32(rng.standard_normal((13, 4)))
        first = ops.matmul(a, b)
        for _ in range(3):
            assert torch.equal(ops.matmul(a, b), first)


class TestConvForward:   # test_ops.py:42-80
    @pytest.mark.parametrize("c", [3, 16, 64])   # SIMT (3) and tensor-core (16, 64) paths
    def test_identity_kernel(self, c):
        # exact on the SIMT path; on the tensor cores 3xTF32 carries ~22
        # bits (the lo term of the split is itself read at TF32 precision),
        # so identity holds to 2^-21 relative -- inside CONV_TOL
        rng = np.random.default_rng(2)
        x = f32(rng.standard_normal((2, c, 8, 8)))
        k = torch.zeros(c, c, 1, 1, device="cuda")
        k[torch.arange(c), torch.arange(c)] = 1.0
        y = ops.conv2d_forward(x, k)
        if c % 16:
            assert torch.equal(y, x)
        else:
            assert bool(((y - x).abs() <= x.abs() * 2.0 ** -21).all())

    def test_all_ones(self):
        out = ops.conv2d_forward(torch.ones(1, 1, 3, 3, device="cuda"),
                                 torch.ones(1, 1, 3, 3, device="cuda"))
        assert tuple(out.shape) == (1, 1, 1, 1) and float(out) == 9.0

    @pytest.mark.parametrize("stride,pad", [(1, 0), (1, 1), (2, 1)])
    @pytest.mark.parametrize("ci,co", [(3, 4), (16, 32)])
    def test_matches_brute_force(self, stride, pad, ci, co):
        rng = np.random.default_rng(3)
        x = rng.standard_normal((2, ci, 7, 9)).astype(np.float32)
        k = rng.standard_normal((co, ci, 3, 3)).astype(np.float32)
        got = host(ops.conv2d_forward(f32(x), f32(k), stride=stride, pad=pad))
        want = torch.nn.functional.conv2d(torch.from_numpy(x).double(), torch.from_numpy(k).double(),
                                          stride=stride, padding=pad).numpy()
        assert norm_err(got, want) < CONV_TOL

    def test_non_integral_extent(self):
        with pytest.raises(ShapeError):
            ops.conv2d_forward(torch.zeros(1, 1, 5, 5, device="cuda"),
                               torch.zeros(1, 1, 2, 2, device="cuda"), stride=2, pad=0)


class TestConvBackward:   # test_ops.py:83-132
    def test_zero_gradient(self):
        rng = np.random.default_rng(5)
        x, k = f32(rng.standard_normal((2, 16, 4, 4))), f32(rng.standard_normal((16, 16, 3, 3)))
        g_x, g_k = ops.conv2d_backward(x, k, torch.zeros(2, 16, 4, 4, device="cuda"), 1, 1)
        assert not bool(g_x.any()) and not bool(g_k.any())

    def test_identity_kernel_adjoint(self):
        rng = np.random.default_rng(6)
        x, g = f32(rng.standard_normal((2, 1, 4, 4))), f32(rng.standard_normal((2, 1, 4, 4)))
        g_x, _ = ops.conv2d_backward(x, torch.ones(1, 1, 1, 1, device="cuda"), g)
        assert torch.equal(g_x, g)

    @pytest.mark.parametrize("stride,pad", [(1, 1), (2, 1)])
    @pytest.mark.parametrize("ci,co", [(2, 3), (16, 16)])
    def test_adjoint_dot_product_identity(self, stride, pad, ci, co):
        # <g, conv(dx, k)> == <g_x, dx>  and  <g, conv(x, dk)> == <g_k, dk>
        rng = np.random.default_rng(8)
        x, k = f32(rng.standard_normal((2, ci, 9, 9))), f32(rng.standard_normal((co, ci, 3, 3)))
        shape = ops.conv2d_out_shape(tuple(x.shape), tuple(k.shape), stride, pad)
        g = f32(rng.standard_normal(shape))
        dx, dk = f32(rng.standard_normal(tuple(x.shape))), f32(rng.standard_normal(tuple(k.shape)))
        g_x, g_k = ops.conv2d_backward(x, k, g, stride, pad)
        lhs = float((g.double() * ops.conv2d_forward(dx, k, stride, pad).double()).sum())
        rhs = float((g_x.double() * dx.double()).sum())
        assert abs(lhs - rhs) / max(abs(lhs), 1e-12) < 1e-5
        lhs = float((g.double() * ops.conv2d_forward(x, dk, stride, pad).double()).sum())
        rhs = float((g_k.double() * dk.double()).sum())
        assert abs(lhs - rhs) / max(abs(lhs), 1e-12) < 1e-5

    def test_gradient_shape_mismatch(self):
        with pytest.raises(ShapeError):
            ops.conv2d_backward(torch.zeros(1, 1, 4, 4, device="cuda"),
                                torch.zeros(1, 1, 3, 3, device="cuda"),
                                torch.zeros(1, 1, 9, 9, device="cuda"), stride=1, pad=1)


class TestChannelReductions:   # test_ops.py:134-170
    def test_constant_tensor(self):
        mean, var = ops.channel_moments(torch.full((3, 2, 4, 4), 2.5, device="cuda"))
        assert np.all(host(mean) == 2.5) and np.all(host(var) == 0.0)

    def test_two_point_moments(self):
        mean, var = ops.channel_moments(f32([[1.0], [3.0]]))
        assert float(mean[0]) == 2.0 and float(var[0]) == 1.0

    def test_moments_match_two_pass_oracle(self):
        rng = np.random.default_rng(9)
        x = rng.standard_normal((4, 3, 5, 6)).astype(np.float32)
        mean, var = (host(t) for t in ops.channel_moments(f32(x)))
        for c in range(3):
            vals = x[:, c].reshape(-1).astype(np.float64)
            m = sum(float(v) for v in vals) / vals.size
            v = sum((float(u) - m) ** 2 for u in vals) / vals.size
            assert abs(mean[c] - m) / max(abs(m), 1e-12) < 1e-12
            assert abs(var[c] - v) / v < 1e-12

    def test_variance_nonnegative(self):
        rng = np.random.default_rng(10)
        x = (rng.standard_normal((8, 4, 3, 3)) * 1e-4 + 7.0).astype(np.float32)
        _, var = ops.channel_moments(f32(x))
        assert bool((var >= 0).all())

    def test_sum_zeros_and_count(self):
        assert not bool(ops.channel_sum(torch.zeros(2, 3, 2, 2, device="cuda")).any())
        assert float(ops.channel_sum(torch.ones(2, 1, 2, 2, device="cuda"))[0]) == 8.0

    def test_sum_matches_loop(self):
        rng = np.random.default_rng(11)
        x = rng.standard_normal((3, 2, 4, 5)).astype(np.float32)
        got = host(ops.channel_sum(f32(x)))
        for c in range(2):
            want = sum(float(v) for v in x[:, c].reshape(-1))
            assert abs(got[c] - want) / max(abs(want), 1e-12) < 1e-12


def _conv_params(ci, co, rng, gamma=None, beta=None):
    w = f32(rng.standard_normal((co, ci, 3, 3)) * 0.3)
    g = torch.ones(ci, device="cuda") if gamma is None else f32(gamma)
    b = torch.zeros(ci, device="cuda") if beta is None else f32(beta)
    return L.LayerParams(kind="conv", weight=w, stride=1, pad=1, gamma=g, beta=b)


class TestLayer:   # test_layer.py:32-260
    def test_approx_forward_equals_exact_forward(self):
        rng = np.random.default_rng(2)
        p = _conv_params(16, 16, rng)
        x = f32(rng.standard_normal((4, 16, 8, 8)))
        out_e, _ = L.layer_forward(x, p, mode="exact")
        out_a, tape_a = L.layer_forward(x, p, mode="approx", bits=4)
        assert torch.equal(out_e, out_a) and tape_a.is_quantized

    def test_normalization_self_check(self):
        rng = np.random.default_rng(4)
        p = _conv_params(16, 16, rng, gamma=rng.uniform(0.5, 2, 16), beta=rng.uniform(-1, 1, 16))
        x = f32(rng.standard_normal((8, 16, 12, 12)) * 3 + 1)
        _, tape = L.layer_forward(x, p, mode="exact")
        a1, _, _ = L.reconstruct_from_tape(tape)
        a1 = host(a1).astype(np.float64)
        assert np.all(np.abs(a1.mean(axis=(0, 2, 3))) < 1e-6)
        assert np.all(np.abs(a1.var(axis=(0, 2, 3)) - 1.0) < 1e-4)

    def test_eval_mode_uses_running_stats(self):
        rng = np.random.default_rng(5)
        p = _conv_params(16, 16, rng)
        x = f32(rng.standard_normal((4, 16, 6, 6)))
        for _ in range(20):
            L.layer_forward(x, p, mode="exact")
        out_eval, tape = L.layer_forward(x, p, training=False)
        assert tape is None
        mean = p.running_mean.clone()
        out_eval2, _ = L.layer_forward(x, p, training=False)
        assert torch.equal(out_eval, out_eval2) and torch.equal(p.running_mean, mean)

    @pytest.mark.parametrize("mode", ["exact", "approx"])
    def test_zero_gradient(self, mode):
        rng = np.random.default_rng(6)
        p = _conv_params(16, 16, rng)
        x = f32(rng.standard_normal((2, 16, 8, 8)))
        out, tape = L.layer_forward(x, p, mode=mode, bits=4)
        g_in = L.layer_backward(torch.zeros_like(out), tape, p)
        assert not bool(g_in.any()) and not bool(p.grad_weight.any())
        assert not bool(p.grad_gamma.any()) and not bool(p.grad_beta.any())

    def test_backward_without_tape_raises(self):
        rng = np.random.default_rng(7)
        p = _conv_params(16, 16, rng)
        out, tape = L.layer_forward(f32(rng.standard_normal((2, 16, 4, 4))), p, training=False)
        with pytest.raises(StateError):
            L.layer_backward(out, tape, p)

    def test_gout_shape_mismatch_raises(self):
        rng = np.random.default_rng(8)
        p = _conv_params(16, 16, rng)
        _, tape = L.layer_forward(f32(rng.standard_normal((2, 16, 4, 4))), p, mode="exact")
        with pytest.raises(StateError):   # as the reference (test_layer.py:210-216)
            L.layer_backward(torch.zeros(2, 16, 5, 5, device="cuda"), tape, p)

    @pytest.mark.parametrize("bits", [2, 4, 8])
    def test_approx_normalized_error_bound(self, bits):
        # every unclipped stored value is within half an interval of the exact one
        rng = np.random.default_rng(9)
        p = _conv_params(16, 16, rng, gamma=rng.uniform(0.5, 2, 16), beta=rng.uniform(-1, 1, 16))
        x = f32(rng.standard_normal((4, 16, 8, 8)))
        _, tape_e = L.layer_forward(x, p, mode="exact")
        _, tape_a = L.layer_forward(x, p, mode="approx", bits=bits)
        a2 = tape_e.stored
        recon = codec.dequantize(tape_a.stored)
        raw = codec.raw_codes(a2, tape_a.gamma, tape_a.beta, bits)
        ok = (raw >= 0) & (raw <= (1 << bits) - 1)
        bound = codec.error_bound(tape_a.gamma, bits).reshape(1, -1, 1, 1).expand_as(a2)
        assert bool(((recon.double() - a2.double()).abs()[ok] <= bound[ok]).all())

    def test_nonpositive_entries_rectify_to_zero(self):
        rng = np.random.default_rng(10)
        p = _conv_params(16, 16, rng)
        out, tape = L.layer_forward(f32(rng.standard_normal((2, 16, 6, 6))), p, mode="approx", bits=4)
        _, a2, a3 = L.reconstruct_from_tape(tape)
        assert bool((a3[a2 <= 0] == 0).all())


class TestQuantize:   # test_quantize.py:80-112
    def test_all_zero(self):
        codes = torch.zeros(64, dtype=torch.uint8, device="cuda")
        packed = codec.pack_codes(codes, 4)
        assert not bool(packed.any()) and torch.equal(codec.unpack_codes(packed, 4, 64), codes)

    def test_out_of_range_code(self):
        with pytest.raises(CodecError):
            codec.pack_codes(torch.full((8,), 16, dtype=torch.uint8, device="cuda"), 4)

    def test_wrong_byte_count(self):
        with pytest.raises(CodecError):
            codec.unpack_codes(torch.zeros(3, dtype=torch.uint8, device="cuda"), 4, 64)

    def test_bad_bits(self):
        with pytest.raises((CodecError, ConfigError)):
            codec.quantize(torch.zeros(2, 16, 4, 4, device="cuda"), torch.ones(16, device="cuda"),
                           torch.zeros(16, device="cuda"), 3)
