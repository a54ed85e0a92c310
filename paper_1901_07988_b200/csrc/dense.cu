// Dense/head kernels (fixed-order float64 matmul, softmax cross-entropy),
// momentum SGD and library metadata.
#include <cstdio>

#include "common.cuh"

namespace qt {

// C[m,n] (=|+=) fp32(sum_k A[m,k]*B[k,n]); float64, ascending k, separately
// rounded multiply and add: bit-identical to ops.matmul (ops.py:54-77).
__global__ void matmul_f64_kernel(const float *a, const float *b, float *c, int64_t M, int64_t K,
                                  int64_t N, int ta, int tb, int accumulate) {
    pdl_enter();
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= M * N) return;
    const int64_t m = idx / N, n = idx - m * N;
    double acc = 0.0;
    for (int64_t k = 0; k < K; ++k) {
        const double av = (double)(ta ? a[k * M + m] : a[m * K + k]);
        const double bv = (double)(tb ? b[n * K + k] : b[k * N + n]);
        acc = __dadd_rn(acc, __dmul_rn(av, bv));
    }
    const float r = __double2float_rn(acc);
    c[idx] = accumulate ? __fadd_rn(c[idx], r) : r;
}

// One warp per row; loss written by the last warp pass (deterministic
// sequential sum of the per-row nll in row order).  training.py:120-134.
__global__ void xent_kernel(const float *logits, const int64_t *labels, int64_t n, int64_t c,
                            double *loss, float *grad, double *nll_scratch, int32_t *bad) {
    pdl_enter();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    for (int64_t r = warp; r < n; r += nw) {
        const float *z = logits + r * c;
        double mx = -INFINITY;
        for (int64_t j = lane; j < c; j += 32) mx = fmax(mx, (double)z[j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        double s = 0.0;
        for (int64_t j = lane; j < c; j += 32) s += exp((double)z[j] - mx);
        s = warp_sum(s);
        const int64_t lab = labels[r];
        const bool ok = lab >= 0 && lab < c;
        if (!ok && lane == 0 && bad) *bad = 1;
        for (int64_t j = lane; j < c; j += 32) {
            double zj = (double)z[j] - mx;
            double g = exp(zj) / s;
            if (j == lab) g -= 1.0;
            grad[r * c + j] = __double2float_rn(g / (double)n);
        }
        if (lane == 0) nll_scratch[r] = ok ? -(((double)z[lab] - mx) - log(s)) : 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int64_t r = 0; r < n; ++r) t += nll_scratch[r];
        *loss = t / (double)n;
    }
}

__global__ void sgd_kernel(float *w, float *g, float *v, int64_t count, float lr,
                           const float *lr_dev, float mom, float wd) {
    pdl_enter();
    const float l = lr_dev ? *lr_dev : lr;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        float vel = __fmul_rn(v[i], mom);                                // vel *= m
        const float gr = g[i];
        vel = wd != 0.f ? __fadd_rn(vel, __fadd_rn(gr, __fmul_rn(wd, w[i])))  // vel += g + wd*w
                        : __fadd_rn(vel, gr);
        v[i] = vel;
        w[i] = __fsub_rn(w[i], __fmul_rn(l, vel));                       // w -= lr*vel
        g[i] = 0.f;                                                      // zero_grads
    }
}

}  // namespace qt

using namespace qt;

extern "C" int qt_version(void) { return 10000; }

extern "C" const char *qt_error_string(int status) {
    if (status == QT_OK) return "ok";
    if (status == QT_EINVAL) return "invalid argument";
    if (status == QT_EUNSUPPORTED) return "unsupported shape";
    if (status > 0) return cudaGetErrorString((cudaError_t)status);
    return "unknown error";
}

namespace qt {
int g_concurrent_bwd = 0;
}

extern "C" int qt_set_concurrent_backward(int on) {
    const int prev = qt::g_concurrent_bwd;
    qt::g_concurrent_bwd = on ? 1 : 0;
    return prev;
}

extern "C" int qt_num_sms(void) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    return n;
}

extern "C" int qt_matmul(const float *a, const float *b, float *c, int64_t m, int64_t k, int64_t nn,
                         int ta, int tb, int accumulate, qt_stream_t stream) {
    QT_REQUIRE(a && b && c && m >= 0 && k >= 0 && nn >= 0);
    if (m * nn == 0) return QT_OK;
    launch_pdl(matmul_f64_kernel, (unsigned)qt_cdiv(m * nn, 128), 128, 0, qt_s(stream), a, b, c, m, k, nn, ta,
                                                                              tb, accumulate);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

extern "C" int qt_softmax_xent(const float *logits, const int64_t *labels, int64_t n, int64_t c,
                               double *loss, float *grad, int32_t *bad_label, qt_stream_t stream) {
    QT_REQUIRE(logits && labels && loss && grad && n > 0 && c > 0);
    // nll scratch lives past the loss slot: caller passes loss with room for 1 + n doubles
    launch_pdl(xent_kernel, 1, 1024, 0, qt_s(stream), logits, labels, n, c, loss, grad, loss + 1, bad_label);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

extern "C" int qt_sgd(float *value, float *grad, float *vel, int64_t count, float lr,
                      const float *lr_dev, float momentum, float weight_decay, qt_stream_t stream) {
    QT_REQUIRE(count >= 0 && (count == 0 || (value && grad && vel)));
    if (count == 0) return QT_OK;
    int64_t blocks = qt_cdiv(count, 256);
    if (blocks > qt_sm_count() * 16) blocks = qt_sm_count() * 16;
    launch_pdl(sgd_kernel, (unsigned)blocks, 256, 0, qt_s(stream), value, grad, vel, count, lr, lr_dev, momentum,
                                                        weight_decay);
    QT_CHECK_LAUNCH();
    return QT_OK;
}
