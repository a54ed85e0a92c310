// Implicit-GEMM convolutions on the CUDA cores (fp32 FFMA, fp32 accumulate).
//
// This is the generic path: any kernel size / stride / padding the reference
// accepts (ops.py:80-183), including the 3-channel stem.  The tensor-core
// path (conv_tc.cu) takes the shapes it supports; both sit behind the same
// qt_conv_* entry points.
//
//   forward : M = N*OH*OW pixels, N = Co, K = Ci*KH*KW      (x gathered)
//   dgrad   : M = N*H*W pixels,   N = Ci, K = Co*KH*KW      (g gathered)
//   wgrad   : M = Co, N = Ci*KH*KW, K = N*OH*OW (split-K, deterministic)
//
// Tile BMxBN per 256-thread block, BK = 16, register double buffering,
// each thread owns TMxTN outputs strided so that a warp's epilogue stores
// are contiguous along the NCHW pixel axis.
#include <algorithm>

#include "common.cuh"

namespace qt {

constexpr int kBK = 16;
constexpr int kCT = 256;

// ---------------------------------------------------------------- loaders

// A operand of the forward pass: im2col of x, m = (n, oh, ow), k = (ci, u, v).
struct FwdA {
    const float *x;
    ConvGeo g;
    __device__ __forceinline__ float operator()(int64_t m, int64_t k) const {
        const int64_t ohw = g.oh * g.ow;
        int64_t nn = m / ohw, p = m - nn * ohw;
        int64_t oy = p / g.ow, ox = p - oy * g.ow;
        int64_t kk = g.kh * g.kw;
        int64_t ci = k / kk, r = k - ci * kk;
        int64_t u = r / g.kw, v = r - u * g.kw;
        int64_t iy = oy * g.s + u - g.pad, ix = ox * g.s + v - g.pad;
        if (iy < 0 || iy >= g.h || ix < 0 || ix >= g.w) return 0.f;
        return __ldg(g_ptr(nn, ci, iy, ix));
    }
    __device__ __forceinline__ const float *g_ptr(int64_t nn, int64_t ci, int64_t iy, int64_t ix) const {
        return x + ((nn * g.ci + ci) * g.h + iy) * g.w + ix;
    }
};

// B operand of the forward pass: w[co][k] (k contiguous).
struct FwdB {
    const float *w;
    int64_t K;
    __device__ __forceinline__ float operator()(int64_t k, int64_t nn) const { return __ldg(w + nn * K + k); }
};

// A operand of dgrad: m = (n, iy, ix) input pixel, k = (co, u, v);
// value g[n, co, (iy+pad-u)/s, (ix+pad-v)/s] when integral and in range.
struct DgradA {
    const float *gr;
    ConvGeo g;
    __device__ __forceinline__ float operator()(int64_t m, int64_t k) const {
        const int64_t hw = g.h * g.w;
        int64_t nn = m / hw, p = m - nn * hw;
        int64_t iy = p / g.w, ix = p - iy * g.w;
        int64_t kk = g.kh * g.kw;
        int64_t co = k / kk, r = k - co * kk;
        int64_t u = r / g.kw, v = r - u * g.kw;
        int64_t ty = iy + g.pad - u, tx = ix + g.pad - v;
        if (ty < 0 || tx < 0) return 0.f;
        int64_t oy = ty / g.s, ox = tx / g.s;
        if (oy * g.s != ty || ox * g.s != tx || oy >= g.oh || ox >= g.ow) return 0.f;
        return __ldg(gr + ((nn * g.co + co) * g.oh + oy) * g.ow + ox);
    }
};

// B operand of dgrad: B[k = (co,u,v)][n = ci] = w[co][ci][u][v].
struct DgradB {
    const float *w;
    ConvGeo g;
    __device__ __forceinline__ float operator()(int64_t k, int64_t ci) const {
        int64_t kk = g.kh * g.kw;
        int64_t co = k / kk, r = k - co * kk;
        return __ldg(w + (co * g.ci + ci) * kk + r);
    }
};

// A operand of wgrad: A[m = co][k = (n, oy, ox)] = g_out.
struct WgradA {
    const float *gr;
    ConvGeo g;
    __device__ __forceinline__ float operator()(int64_t co, int64_t k) const {
        const int64_t ohw = g.oh * g.ow;
        int64_t nn = k / ohw, p = k - nn * ohw;
        return __ldg(gr + (nn * g.co + co) * ohw + p);
    }
};

// B operand of wgrad: B[k = (n, oy, ox)][j = (ci, u, v)] = act(n, ci, iy, ix)
// where act is the plain input, relu(a2 tape) or relu(decode(codes)).
struct WgradB {
    qt_tape_t t;
    const float *plain;
    ConvGeo g;
    __device__ __forceinline__ float operator()(int64_t k, int64_t j) const {
        const int64_t ohw = g.oh * g.ow;
        int64_t nn = k / ohw, p = k - nn * ohw;
        int64_t oy = p / g.ow, ox = p - oy * g.ow;
        int64_t kk = g.kh * g.kw;
        int64_t ci = j / kk, r = j - ci * kk;
        int64_t u = r / g.kw, v = r - u * g.kw;
        int64_t iy = oy * g.s + u - g.pad, ix = ox * g.s + v - g.pad;
        if (iy < 0 || iy >= g.h || ix < 0 || ix >= g.w) return 0.f;
        int64_t i = ((nn * g.ci + ci) * g.h + iy) * g.w + ix;
        if (plain) return __ldg(plain + i);
        float a = tape_value(t, i, (int)ci);
        return (a >= 0.f || isnan(a)) ? a : 0.f;  // relu as np.maximum (layer.py:356)
    }
};

// ------------------------------------------------------------ epilogues

// Store into NCHW rows: m -> (n, pixel), column -> channel; optional
// shortcut add (engine.py:262-269): res (N, CR, OH*sr, OW*sr), cols < CR.
struct StoreNCHW {
    float *out;
    int64_t npix, ncols, ow;   // pixels per image, channels, output width
    const float *res;
    int64_t cr, sr;
    __device__ __forceinline__ void operator()(int64_t m, int64_t col, float v, int) const {
        int64_t nn = m / npix, p = m - nn * npix;
        if (res && col < cr) {
            float r;
            if (sr == 1) {
                r = res[(nn * cr + col) * npix + p];
            } else {
                int64_t oy = p / ow, ox = p - oy * ow;
                r = res[((nn * cr + col) * (npix / ow * sr) + oy * sr) * (ow * sr) + ox * sr];
            }
            v = __fadd_rn(v, r);
        }
        out[(nn * ncols + col) * npix + p] = v;
    }
};

// Split-K partial tile for wgrad: ws[split][m][n].
struct StorePartial {
    float *ws;
    int64_t M, N;
    __device__ __forceinline__ void operator()(int64_t m, int64_t nn, float v, int split) const {
        ws[((int64_t)split * M + m) * N + nn] = v;
    }
};

// ---------------------------------------------------------------- GEMM

template <int BM, int BN, int TM, int TN, bool A_KFAST, bool B_KFAST, class LA, class LB, class EP>
__global__ void __launch_bounds__(kCT) simt_gemm(LA la, LB lb, EP ep, int64_t M, int64_t N,
                                                 int64_t K, int64_t k_per_split) {
    pdl_enter();
    static_assert((BM / TM) * (BN / TN) == kCT, "thread layout");
    constexpr int RA = BM * kBK / kCT;
    constexpr int RB = BN * kBK / kCT;
    constexpr int PA = A_KFAST ? 1 : 0;
    constexpr int PB = B_KFAST ? 1 : 0;
    __shared__ float As[2][kBK][BM + PA];
    __shared__ float Bs[2][kBK][BN + PB];

    const int tid = threadIdx.x;
    const int tm = tid % (BM / TM), tn = tid / (BM / TM);
    const int64_t m0 = (int64_t)blockIdx.x * BM;
    const int64_t n0 = (int64_t)blockIdx.y * BN;
    const int split = blockIdx.z;
    const int64_t kb = (int64_t)split * k_per_split;
    const int64_t ke = min(K, kb + k_per_split);

    float ra[RA], rb[RB];
    auto fetch = [&](int64_t k0) {
#pragma unroll
        for (int r = 0; r < RA; ++r) {
            int e = tid + r * kCT;
            int ml, kl;
            if (A_KFAST) { kl = e % kBK; ml = e / kBK; } else { ml = e % BM; kl = e / BM; }
            int64_t m = m0 + ml, k = k0 + kl;
            ra[r] = (m < M && k < ke) ? la(m, k) : 0.f;
        }
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            int e = tid + r * kCT;
            int nl, kl;
            if (B_KFAST) { kl = e % kBK; nl = e / kBK; } else { nl = e % BN; kl = e / BN; }
            int64_t nn = n0 + nl, k = k0 + kl;
            rb[r] = (nn < N && k < ke) ? lb(k, nn) : 0.f;
        }
    };
    auto stash = [&](int buf) {
#pragma unroll
        for (int r = 0; r < RA; ++r) {
            int e = tid + r * kCT;
            int ml, kl;
            if (A_KFAST) { kl = e % kBK; ml = e / kBK; } else { ml = e % BM; kl = e / BM; }
            As[buf][kl][ml] = ra[r];
        }
#pragma unroll
        for (int r = 0; r < RB; ++r) {
            int e = tid + r * kCT;
            int nl, kl;
            if (B_KFAST) { kl = e % kBK; nl = e / kBK; } else { nl = e % BN; kl = e / BN; }
            Bs[buf][kl][nl] = rb[r];
        }
    };

    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

    int buf = 0;
    if (kb < ke) {
        fetch(kb);
        stash(0);
    }
    __syncthreads();
    for (int64_t k0 = kb; k0 < ke; k0 += kBK) {
        const bool more = k0 + kBK < ke;
        if (more) fetch(k0 + kBK);
#pragma unroll
        for (int kk = 0; kk < kBK; ++kk) {
            float av[TM], bv[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) av[i] = As[buf][kk][tm + i * (BM / TM)];
#pragma unroll
            for (int j = 0; j < TN; ++j) bv[j] = Bs[buf][kk][tn * TN + j];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        if (more) {
            stash(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        int64_t m = m0 + tm + i * (BM / TM);
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            int64_t nn = n0 + tn * TN + j;
            if (nn < N) ep(m, nn, acc[i][j], split);
        }
    }
}

template <bool A_KFAST, bool B_KFAST, class LA, class LB, class EP>
static int run_gemm(LA la, LB lb, EP ep, int64_t M, int64_t N, int64_t K, int64_t kps,
                    cudaStream_t s) {
    if (M == 0 || N == 0) return QT_OK;
    if (kps <= 0) kps = kBK;
    const int64_t splits = std::max<int64_t>(1, qt_cdiv(K, kps));
    if (N <= 16) {
        dim3 grid((unsigned)qt_cdiv(M, 256), (unsigned)qt_cdiv(N, 16), (unsigned)splits);
        launch_pdl(simt_gemm<256, 16, 4, 4, A_KFAST, B_KFAST, LA, LB, EP>, grid, kCT, 0, s, la, lb, ep, M, N, K, kps);
    } else if (N <= 32) {
        dim3 grid((unsigned)qt_cdiv(M, 128), (unsigned)qt_cdiv(N, 32), (unsigned)splits);
        launch_pdl(simt_gemm<128, 32, 4, 4, A_KFAST, B_KFAST, LA, LB, EP>, grid, kCT, 0, s, la, lb, ep, M, N, K, kps);
    } else {
        dim3 grid((unsigned)qt_cdiv(M, 128), (unsigned)qt_cdiv(N, 64), (unsigned)splits);
        launch_pdl(simt_gemm<128, 64, 8, 4, A_KFAST, B_KFAST, LA, LB, EP>, grid, kCT, 0, s, la, lb, ep, M, N, K, kps);
    }
    QT_CHECK_LAUNCH();
    return QT_OK;
}

static ConvGeo make_geo(int64_t n, int64_t ci, int64_t h, int64_t w, int64_t co, int64_t kh,
                        int64_t kw, int64_t s, int64_t pad) {
    ConvGeo g{n, ci, h, w, co, kh, kw, s, pad, 0, 0};
    g.oh = (h + 2 * pad - kh) / s + 1;
    g.ow = (w + 2 * pad - kw) / s + 1;
    return g;
}

static bool geo_ok(const ConvGeo &g) {
    if (g.n <= 0 || g.ci <= 0 || g.h <= 0 || g.w <= 0 || g.co <= 0 || g.kh <= 0 || g.kw <= 0)
        return false;
    if (g.s <= 0 || g.pad < 0) return false;
    if ((g.h + 2 * g.pad - g.kh) % g.s || (g.w + 2 * g.pad - g.kw) % g.s) return false;
    return g.oh > 0 && g.ow > 0;
}

// Split-K plan for wgrad: (k_per_split, splits), k_per_split a multiple of kBK.
static void wgrad_plan(const ConvGeo &g, int64_t &kps, int64_t &splits) {
    const int64_t M = g.co, N = g.ci * g.kh * g.kw, K = g.n * g.oh * g.ow;
    int64_t tiles = qt_cdiv(M, N <= 16 ? 256 : 128) * qt_cdiv(N, N <= 16 ? 16 : (N <= 32 ? 32 : 64));
    int64_t want = std::max<int64_t>(1, (4 * qt_sm_count()) / std::max<int64_t>(tiles, 1));
    int64_t maxs = std::max<int64_t>(1, K / (4 * kBK));
    int64_t sp = std::min(want, maxs);
    kps = std::max<int64_t>(kBK, qt_cdiv(qt_cdiv(K, sp), kBK) * kBK);
    splits = std::max<int64_t>(1, qt_cdiv(K, kps));
}

}  // namespace qt

using namespace qt;

// Tensor-core paths (conv_tc.cu); return QT_EUNSUPPORTED for shapes they do not take.
int qt_tc_conv_forward(const float *x, const float *w, float *out, const qt::ConvGeo &g,
                       const float *res, int64_t cr, int64_t sr, void *ws, cudaStream_t s);
int qt_tc_conv_dgrad(const float *gr, const float *w, float *gx, const qt::ConvGeo &g, void *ws,
                     cudaStream_t s);
int qt_tc_conv_wgrad(const float *gr, qt_tape_t act, const float *x_plain, float *grad_w,
                     const qt::ConvGeo &g, void *ws, cudaStream_t st);
int64_t qt_tc_wgrad_workspace(const qt::ConvGeo &g);
int qt_tc_conv_wgrad_s2d(const float *gr, qt_tape_t act, float *grad_w, const qt::ConvGeo &g,
                         void *ws, cudaStream_t st);
int64_t qt_tc_s2d_workspace(const qt::ConvGeo &g);
int qt_tc_conv_s2d_forward(const float *x, const float *w, float *out, const qt::ConvGeo &g,
                           const float *res, int64_t cr, int64_t sr, void *ws, cudaStream_t s);
int qt_tc_conv_s2d_dgrad(const float *gr, const float *w, float *gx, const qt::ConvGeo &g,
                         void *ws, cudaStream_t s);
int64_t qt_tc_seg_workspace(const qt::ConvGeo &g);
int qt_tc_conv_seg_forward(const float *x, const float *w, float *out, const qt::ConvGeo &g,
                           const float *res, int64_t cr, int64_t sr, void *ws, cudaStream_t st);
int qt_tc_conv_seg_dgrad(const float *gr, const float *w, float *gx, const qt::ConvGeo &g,
                         void *ws, cudaStream_t st);
int64_t qt_tc_seg_wgrad_workspace(const qt::ConvGeo &g);
int qt_tc_conv_seg_wgrad(const float *gr, qt_tape_t act, const float *x_plain, float *grad_w,
                         const qt::ConvGeo &g, void *ws, cudaStream_t st);
int qt_tc_wgrad_reduce(const float *partial, int64_t splits, int64_t count, float *grad_w,
                       cudaStream_t st);

static inline bool ws_bytes_ok(void *ws) { return ws != nullptr; }

// Full scratch need of qt_conv_forward / qt_conv_dgrad for this shape: the
// prepared weight operand, plus the space-to-depth buffer for kernel == stride
extern "C" int64_t qt_conv_workspace_ex(int64_t n, int64_t ci, int64_t h, int64_t wd, int64_t co,
                                        int64_t kh, int64_t kw, int64_t stride, int64_t pad) {
    ConvGeo g = make_geo(n, ci, h, wd, co, kh, kw, stride, pad);
    int64_t need = qt_conv_workspace(ci, co, kh, kw);
    if (geo_ok(g)) need = std::max({need, qt_tc_s2d_workspace(g), qt_tc_seg_workspace(g)});
    return need;
}

extern "C" int qt_conv_forward(const float *x, const float *w, float *out, int64_t n, int64_t ci,
                               int64_t h, int64_t wd, int64_t co, int64_t kh, int64_t kw,
                               int64_t stride, int64_t pad, const float *res, int64_t cr,
                               int64_t sr, void *ws, qt_stream_t stream) {
    ConvGeo g = make_geo(n, ci, h, wd, co, kh, kw, stride, pad);
    QT_REQUIRE(x && out && geo_ok(g));
    QT_REQUIRE(!res || (cr > 0 && cr <= co && sr >= 1));
    int rc = qt_tc_conv_forward(x, w, out, g, res, cr, sr, ws, qt_s(stream));
    if (rc != QT_EUNSUPPORTED) return rc;
    QT_REQUIRE(w);
    if (ws_bytes_ok(ws)) {   // kernel == stride: space-to-depth + tensor-core 1x1
        rc = qt_tc_conv_s2d_forward(x, w, out, g, res, cr, sr, ws, qt_s(stream));
        if (rc != QT_EUNSUPPORTED) return rc;
        // other plane widths: segmented copy + tensor-core rows
        rc = qt_tc_conv_seg_forward(x, w, out, g, res, cr, sr, ws, qt_s(stream));
        if (rc != QT_EUNSUPPORTED) return rc;
    }   // NULL (prepared operand in ws) is only valid on the tensor-core path
    FwdA la{x, g};
    FwdB lb{w, ci * kh * kw};
    StoreNCHW ep{out, g.oh * g.ow, co, g.ow, res, cr, sr};
    return run_gemm<false, true>(la, lb, ep, n * g.oh * g.ow, co, ci * kh * kw,
                                 qt_cdiv(ci * kh * kw, kBK) * kBK, qt_s(stream));
}

extern "C" int qt_conv_dgrad(const float *gr, const float *w, float *gx, int64_t n, int64_t ci,
                             int64_t h, int64_t wd, int64_t co, int64_t kh, int64_t kw,
                             int64_t stride, int64_t pad, void *ws, qt_stream_t stream) {
    ConvGeo g = make_geo(n, ci, h, wd, co, kh, kw, stride, pad);
    QT_REQUIRE(gr && gx && geo_ok(g));
    int rc = qt_tc_conv_dgrad(gr, w, gx, g, ws, qt_s(stream));
    if (rc != QT_EUNSUPPORTED) return rc;
    QT_REQUIRE(w);
    if (ws_bytes_ok(ws)) {
        rc = qt_tc_conv_s2d_dgrad(gr, w, gx, g, ws, qt_s(stream));
        if (rc != QT_EUNSUPPORTED) return rc;
        rc = qt_tc_conv_seg_dgrad(gr, w, gx, g, ws, qt_s(stream));
        if (rc != QT_EUNSUPPORTED) return rc;
    }
    DgradA la{gr, g};
    DgradB lb{w, g};
    StoreNCHW ep{gx, h * wd, ci, wd, nullptr, 0, 1};
    return run_gemm<false, false>(la, lb, ep, n * h * wd, ci, co * kh * kw,
                                  qt_cdiv(co * kh * kw, kBK) * kBK, qt_s(stream));
}

extern "C" int64_t qt_conv_wgrad_workspace(int64_t n, int64_t ci, int64_t h, int64_t wd, int64_t co,
                                           int64_t kh, int64_t kw, int64_t stride, int64_t pad) {
    ConvGeo g = make_geo(n, ci, h, wd, co, kh, kw, stride, pad);
    if (!geo_ok(g)) return 0;
    int64_t kps, splits;
    wgrad_plan(g, kps, splits);
    return std::max({splits * co * ci * kh * kw * (int64_t)sizeof(float), qt_tc_wgrad_workspace(g),
                     qt_tc_seg_wgrad_workspace(g)}) +
           256;
}

extern "C" int qt_conv_wgrad(const float *gr, qt_tape_t act, const float *x_plain, float *grad_w,
                             int64_t n, int64_t ci, int64_t h, int64_t wd, int64_t co, int64_t kh,
                             int64_t kw, int64_t stride, int64_t pad, void *ws,
                             qt_stream_t stream) {
    ConvGeo g = make_geo(n, ci, h, wd, co, kh, kw, stride, pad);
    QT_REQUIRE(gr && grad_w && ws && geo_ok(g));
    QT_REQUIRE(x_plain || act.a2 || (act.codes && act.step && act.offset && qt_bits_ok(act.bits)));
    int rc0 = qt_tc_conv_wgrad(gr, act, x_plain, grad_w, g, ws, qt_s(stream));
    if (rc0 != QT_EUNSUPPORTED) return rc0;
    if (!x_plain) {   // 2x2/s2 on codes: 1x1 of the rearranged (space-to-depth) tape
        rc0 = qt_tc_conv_wgrad_s2d(gr, act, grad_w, g, ws, qt_s(stream));
        if (rc0 != QT_EUNSUPPORTED) return rc0;
    }
    rc0 = qt_tc_conv_seg_wgrad(gr, act, x_plain, grad_w, g, ws, qt_s(stream));
    if (rc0 != QT_EUNSUPPORTED) return rc0;
    const int64_t M = co, N = ci * kh * kw, K = n * g.oh * g.ow;
    int64_t kps, splits;
    wgrad_plan(g, kps, splits);
    WgradA la{gr, g};
    WgradB lb{act, x_plain, g};
    StorePartial ep{(float *)ws, M, N};
    int rc = run_gemm<true, true>(la, lb, ep, M, N, K, kps, qt_s(stream));
    if (rc) return rc;
    return qt_tc_wgrad_reduce((const float *)ws, splits, M * N, grad_w, qt_s(stream));
}
