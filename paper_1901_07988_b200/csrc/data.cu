// Device-side input pipeline (reference data.py:45-87 and :182-206):
// CIFAR-10 binary records -> labels + fp32 pixels, per-channel
// standardization, and the batch gather fused with horizontal-flip and
// pad-4 random-crop augmentation.  All three are bit-identical to the
// reference's numpy arithmetic (one IEEE fp32 divide; a subtract and a
// divide; pure data movement with zero fill).
#include <algorithm>

#include "common.cuh"

namespace qt {

constexpr int kDThreads = 256;
constexpr int64_t kRecordBytes = 3073;     // data.py:20
constexpr int64_t kPixels = 3 * 32 * 32;

// records (n x 3073 B: label byte, then 3072 channel-major pixels) ->
// labels int64, images fp32 = u8 / 255 (data.py:52-57, :76)
__global__ void cifar_decode_kernel(const uint8_t *rec, int64_t n, float *images, int64_t *labels,
                                    int32_t *bad) {
    pdl_enter();
    const int64_t total = n * kPixels;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / kPixels, p = i - r * kPixels;
        images[i] = __fdiv_rn((float)rec[r * kRecordBytes + 1 + p], 255.0f);
        if (p == 0) {
            const uint8_t lab = rec[r * kRecordBytes];
            labels[r] = lab;
            if (lab > 9 && bad) *bad = 1;      // data.py:73-74
        }
    }
}

// images[n][c][hw] = (images - mean32[c]) / std32[c]  (data.py:84-85)
__global__ void standardize_kernel(float *images, int64_t n, int64_t c, int64_t hw,
                                   const float *mean, const float *stdv) {
    pdl_enter();
    const int64_t total = n * c * hw;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ch = (i / hw) % c;
        images[i] = __fdiv_rn(__fsub_rn(images[i], mean[ch]), stdv[ch]);
    }
}

// dst[i] = augment(src[idx[i]]): optional horizontal flip, then the image
// shifted inside a zero border of `pad` pixels by (dy, dx) - pad
// (data.py:182-206: out[i] = padded[:, dy:dy+h, dx:dx+w]).
__global__ void gather_augment_kernel(const float *src, const int64_t *idx, int64_t n, int64_t c,
                                      int64_t h, int64_t w, const uint8_t *flip,
                                      const int32_t *offs, int pad, float *dst) {
    pdl_enter();
    const int64_t per = c * h * w, total = n * per;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / per, r = i - b * per;
        const int64_t ch = r / (h * w), yx = r - ch * h * w;
        const int64_t y = yx / w, x = yx - y * w;
        const int64_t sy = offs ? y + offs[2 * b] - pad : y;
        const int64_t sxf = offs ? x + offs[2 * b + 1] - pad : x;     // column of the flipped image
        float v = 0.f;
        if (sy >= 0 && sy < h && sxf >= 0 && sxf < w) {
            const int64_t sx = (flip && flip[b]) ? w - 1 - sxf : sxf;
            v = src[((idx ? idx[b] : b) * c + ch) * h * w + sy * w + sx];
        }
        dst[i] = v;
    }
}

static unsigned dgrid(int64_t total) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(qt_cdiv(total, kDThreads),
                                                            (int64_t)qt_sm_count() * 16));
}

}  // namespace qt

using namespace qt;

extern "C" int qt_cifar_decode(const uint8_t *records, int64_t n, float *images, int64_t *labels,
                               int32_t *bad_label, qt_stream_t stream) {
    QT_REQUIRE(records && images && labels && n >= 0);
    if (n == 0) return QT_OK;
    launch_pdl(cifar_decode_kernel, dgrid(n * kPixels), kDThreads, 0, qt_s(stream), records, n,
               images, labels, bad_label);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

extern "C" int qt_standardize(float *images, int64_t n, int64_t c, int64_t hw, const float *mean,
                              const float *std_, qt_stream_t stream) {
    QT_REQUIRE(images && mean && std_ && n >= 0 && c > 0 && hw > 0);
    if (n == 0) return QT_OK;
    launch_pdl(standardize_kernel, dgrid(n * c * hw), kDThreads, 0, qt_s(stream), images, n, c, hw,
               mean, std_);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

extern "C" int qt_gather_augment(const float *src, const int64_t *idx, int64_t n, int64_t c,
                                 int64_t h, int64_t w, const uint8_t *flip, const int32_t *offsets,
                                 int pad, float *dst, qt_stream_t stream) {
    QT_REQUIRE(src && dst && n >= 0 && c > 0 && h > 0 && w > 0 && pad >= 0);
    if (n == 0) return QT_OK;
    launch_pdl(gather_augment_kernel, dgrid(n * c * h * w), kDThreads, 0, qt_s(stream), src, idx,
               n, c, h, w, flip, offsets, pad, dst);
    QT_CHECK_LAUNCH();
    return QT_OK;
}
