// BN / ReLU backward from the tape (layer.py:353-381, bn_input_gradient
// :286-308) -- two HBM passes over g3, both reading the packed codes:
//
//   reduce : per channel  S0 = sum g3m, S1 = sum a1*g3m, S2 = sum g1,
//            S3 = sum a1v*g1   (g3m = g3*mask, g1 = g3m*gamma; float64)
//            -> grad_beta += S0, grad_gamma += S1, t2 = S2/n, t3 = S3/n, inv
//   apply  : g_in = ((g1 - t2) - a1v*t3) * inv  (+ shortcut adjoint)
//
// For a K-bit tape every per-element quantity that depends on the stored
// activation (mask = decoded > 0, a1 = (decoded - beta)/safe_gamma) is a
// function of the code alone, so each channel's 2^K-entry table is built
// once (with exactly the reference's float64 decode and fp32 rounding) and
// the element loops are table lookups: no per-element float64 decode or
// IEEE division, 8 elements per thread with 128-bit g3 loads and one K-byte
// code load.  Reductions stay deterministic (fixed partition, float64
// partials, last-block finalize in block order).
#include <algorithm>

#include "common.cuh"

namespace qt {

constexpr int kBT = 256;
constexpr int64_t kBwdCounterBytes = 65536 * 4;
constexpr int64_t kMaxLut = 256;

struct BwdPart {
    int64_t ppb, nb;
};

// ~4 blocks per SM in total, each reducing a contiguous run of planes of one
// channel (enough work per thread that the block's deterministic
// last-block-finalize tail is amortised)
static BwdPart bwd_partition(int64_t n, int64_t c, int64_t hw) {
    // blocks of ~8192 elements (4 groups of 8 per thread, all loads in
    // flight at once): enough blocks to fill the SMs several times over for
    // the large layers, one block per channel for the small ones
    (void)c;
    BwdPart p;
    p.ppb = std::max<int64_t>(1, qt_env_i64("QTAPE_BWD_TGT", qt_red_target()) / hw);
    p.ppb = std::min<int64_t>(p.ppb, std::max<int64_t>(1, n * c / qt_env_i64("QTAPE_BWD_DIV", qt_red_div())));   // >= ~2 blocks / SM
    if (p.ppb > n) p.ppb = n;
    p.nb = qt_cdiv(n, p.ppb);
    return p;
}

// The reduce launch: at most kBwdCluster blocks per channel (one cluster).
constexpr int64_t kBwdCluster = 8;
static BwdPart reduce_partition(int64_t n, int64_t c, int64_t hw) {
    BwdPart p = bwd_partition(n, c, hw);
    // balanced runs: the launch lasts as long as its longest block
    const int64_t nb = std::min<int64_t>(p.nb, qt_red_cluster());
    p.ppb = qt_cdiv(n, nb);
    p.nb = qt_cdiv(n, p.ppb);
    return p;
}

// ws layout: [counters 256 KiB][lut: C x 2 x 256 floats][partials C x nb x 4 doubles]
static inline float *lut_base(void *ws) { return (float *)((char *)ws + kBwdCounterBytes); }
static inline double *part_base(void *ws, int64_t c) {
    return (double *)((char *)ws + kBwdCounterBytes + c * 2 * kMaxLut * sizeof(float));
}

struct BwdArgs {
    const float *g3;
    qt_tape_t tape;
    int64_t n, c, hw;
    const float *gamma, *beta;
    const double *sigma2;
    double eps;
    const float *va1;
    float *grad_gamma, *grad_beta, *stats;
    int64_t ppb, nb;
    double *part;
    unsigned *counter;
    float *lut;      // [C][2][256]: mask, a1 per code
    FastDiv gppd;    // hw / 8
    FastDiv hwd;     // hw (scalar loop of odd planes)
};

// mask (1/0) and a1 for one code of channel ch (layer.py:354-366)
__device__ __forceinline__ void lut_entry(const qt_tape_t &t, int ch, uint32_t code, float bet,
                                          float sg, float &m, float &a1) {
    const float a2 = decode(code, t.step[ch], t.offset[ch], t.bits);
    m = a2 > 0.f ? 1.f : 0.f;
    a1 = __fdiv_rn(__fsub_rn(a2, bet), sg);
}

__device__ __forceinline__ uint64_t load_code_word(const uint8_t *codes, int64_t i0, int bits) {
    const uint8_t *src = codes + (i0 >> 3) * bits;   // i0 multiple of 8
    switch (bits) {
        case 8: { uint2 u = *reinterpret_cast<const uint2 *>(src); return u.x | ((uint64_t)u.y << 32); }
        case 4: return *reinterpret_cast<const uint32_t *>(src);
        case 2: return *reinterpret_cast<const uint16_t *>(src);
        default: return *src;
    }
}

// G consecutive codes starting at element i0 (a multiple of G)
template <int G>
__device__ __forceinline__ uint64_t load_code_group(const uint8_t *codes, int64_t i0, int bits) {
    if (G == 8) return load_code_word(codes, i0, bits);
    const uint8_t *src = codes + ((i0 * bits) >> 3);
    switch (bits) {
        case 8: return *reinterpret_cast<const uint32_t *>(src);
        case 4: return *reinterpret_cast<const uint16_t *>(src);
        case 2: return *src;
        default: return (uint64_t)(*src >> (i0 & 4)) & 0xFu;   // 1-bit: a nibble
    }
}

// vector group width for a plane of hw pixels (rows of w): 8, 4 or 0 (scalar)
static inline int bn_group(int64_t hw, int64_t w) {
    if (hw % 8 == 0 && w >= 8) return 8;
    if (hw % 4 == 0 && w >= 4) return 4;
    return 0;
}

template <bool CODES, bool VA1, int G>
__global__ void __launch_bounds__(kBT) bn_bwd_reduce_kernel(BwdArgs a) {
    pdl_enter();
    __shared__ float s_m[kMaxLut], s_a1[kMaxLut];
    __shared__ float2 s_ma[kMaxLut];      // (mask, a1) per code: one 8-byte lookup
    __shared__ double s_a1d[kMaxLut];
    __shared__ double red[3][kBT / 32];
    __shared__ double s_part[3];          // this block's sums, read by cluster rank 0
    const int ch = blockIdx.y;
    // the finalizing thread (rank 0, thread 0) loads what the finalize needs now
    const bool fin = blockIdx.x == 0 && threadIdx.x == 0;
    double fin_s2 = 0.0;
    float fin_gb = 0.f, fin_gg = 0.f;
    if (fin) {
        fin_s2 = a.sigma2[ch];
        if (a.grad_beta) fin_gb = a.grad_beta[ch];
        if (a.grad_gamma) fin_gg = a.grad_gamma[ch];
    }
    const float gam = a.gamma[ch], bet = a.beta[ch], sg = safe_gamma(gam);
    const int ncode = CODES ? (1 << a.tape.bits) : 0;
    auto build_lut = [&]() {
        if (CODES) {
            for (int code = threadIdx.x; code < ncode; code += kBT) {
                lut_entry(a.tape, ch, code, bet, sg, s_m[code], s_a1[code]);
                s_a1d[code] = (double)s_a1[code];
                s_ma[code] = make_float2(s_m[code], s_a1[code]);
            }
            __syncthreads();
        }
    };
    const int64_t p0 = (int64_t)blockIdx.x * a.ppb;
    const int64_t p1 = min(p0 + a.ppb, a.n);
    // float64 accumulators: S0 = sum g3m, S1 = sum a1*g3m, S3' = sum a1v*g3m
    // (g3m = g3*mask is exact in fp32; S2 = gamma*S0 and S3 = gamma*S3' are
    // formed once per channel).  One float->double conversion per element.
    double v0 = 0.0, v1 = 0.0, v3 = 0.0;
    const uint32_t cmask = (1u << a.tape.bits) - 1u;
    // The summation order depends only on the shape (never on the tape
    // type), so an exact tape and a K-bit tape with variance_a1 substituted
    // produce bit-identical sums (reference test_layer.py:173-202).
    const int64_t cnt8 = ((p1 - p0) * a.hw) / G;
    if (G > 0 && a.hw % G == 0 && cnt8 < (1ll << 31)) {
        const uint32_t groups = (uint32_t)cnt8;
        const uint32_t gpp = (uint32_t)(a.hw / G);
        constexpr int U = 4;                     // groups in flight per thread
        float4 ga[U], gb[U], xa[U], xb[U];
        uint64_t word[U];
        int64_t i0[U];
        auto load = [&](uint32_t g0) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t gi = g0 + u * kBT;
                if (gi >= groups) break;
                const uint32_t pl = fast_div(gi, a.gppd), off = (gi - pl * gpp) * G;
                i0[u] = ((p0 + pl) * a.c + ch) * a.hw + off;
                ga[u] = __ldg(reinterpret_cast<const float4 *>(a.g3 + i0[u]));
                if (G == 8) gb[u] = __ldg(reinterpret_cast<const float4 *>(a.g3 + i0[u]) + 1);
                if (CODES) {
                    word[u] = load_code_group<G>(a.tape.codes, i0[u], a.tape.bits);
                } else {
                    xa[u] = __ldg(reinterpret_cast<const float4 *>(a.tape.a2 + i0[u]));
                    if (G == 8) xb[u] = __ldg(reinterpret_cast<const float4 *>(a.tape.a2 + i0[u]) + 1);
                }
            }
        };
        // the first round of loads is in flight while the code table is built
        load(threadIdx.x);
        build_lut();
        for (uint32_t g0 = threadIdx.x; g0 < groups; g0 += U * kBT) {
            if (g0 != threadIdx.x) load(g0);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (g0 + u * kBT >= groups) break;
                float gv[8], xv[8];
                gv[0] = ga[u].x; gv[1] = ga[u].y; gv[2] = ga[u].z; gv[3] = ga[u].w;
                if (G == 8) { gv[4] = gb[u].x; gv[5] = gb[u].y; gv[6] = gb[u].z; gv[7] = gb[u].w; }
                if (!CODES) {
                    xv[0] = xa[u].x; xv[1] = xa[u].y; xv[2] = xa[u].z; xv[3] = xa[u].w;
                    if (G == 8) { xv[4] = xb[u].x; xv[5] = xb[u].y; xv[6] = xb[u].z; xv[7] = xb[u].w; }
                }
                // the 8 elements of a group are combined in fp32 (fixed order,
                // fused multiply-add for the a1 products), the group sums in
                // float64: one float->double conversion per sum per group
                float f0 = 0.f, f1 = 0.f, f3 = 0.f;
#pragma unroll
                for (int j = 0; j < (G > 0 ? G : 1); ++j) {
                    float m, a1;
                    if (CODES) {
                        const uint32_t code = (uint32_t)(word[u] >> (j * a.tape.bits)) & cmask;
                        const float2 ma = s_ma[code];
                        m = ma.x;
                        a1 = ma.y;
                    } else {
                        m = xv[j] > 0.f ? 1.f : 0.f;
                        a1 = __fdiv_rn(__fsub_rn(xv[j], bet), sg);
                    }
                    const float gm = __fmul_rn(gv[j], m);
                    f0 = __fadd_rn(f0, gm);
                    f1 = __fmaf_rn(a1, gm, f1);
                    if (VA1) f3 = __fmaf_rn(a.va1[i0[u] + j], gm, f3);
                }
                v0 += (double)f0; v1 += (double)f1; v3 += (double)f3;
            }
        }
    } else {
        build_lut();
        const int64_t cnt = (p1 - p0) * a.hw;
        const bool fd = cnt < (1ll << 31) && a.hw < (1ll << 31);   // FastDiv indexing
        for (int64_t e = threadIdx.x; e < cnt; e += kBT) {
            const int64_t pl = fd ? (int64_t)fast_div((uint32_t)e, a.hwd) : e / a.hw;
            const int64_t off = e - pl * a.hw;
            const int64_t i = ((p0 + pl) * a.c + ch) * a.hw + off;
            float m;
            double a1d;
            if (CODES) {
                const uint32_t code = get_code(a.tape.codes, i, a.tape.bits);
                m = s_m[code];
                a1d = s_a1d[code];
            } else {
                const float a2 = a.tape.a2[i];
                m = a2 > 0.f ? 1.f : 0.f;
                a1d = (double)__fdiv_rn(__fsub_rn(a2, bet), sg);
            }
            const double gm = (double)__fmul_rn(a.g3[i], m);
            v0 += gm;
            v1 = fma(a1d, gm, v1);
            if (VA1) v3 = fma((double)a.va1[i], gm, v3);
        }
    }
    if (!VA1) v3 = v1;
    v0 = warp_sum(v0); v1 = warp_sum(v1); v3 = warp_sum(v3);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[0][w] = v0; red[1][w] = v1; red[2][w] = v3;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int j = 0; j < 3; ++j) {
            double t = 0.0;
            for (int q = 0; q < kBT / 32; ++q) t += red[j][q];
            s_part[j] = t;
        }
    }
    // the nb blocks of channel ch form one cluster: rank 0 adds the block
    // sums in rank order through distributed shared memory
    cluster_sync_all();
    double s[3] = {0.0, 0.0, 0.0};
    if (fin) {
        for (unsigned r = 0; r < (unsigned)a.nb; ++r)
            for (int j = 0; j < 3; ++j) s[j] += ld_dsmem_f64(&s_part[j], r);
    }
    cluster_sync_all();   // remote CTAs keep their shared memory until read
    if (blockIdx.x != 0) return;
    // rank 0 publishes the code table for the apply pass
    if (CODES) {
        float *lut = a.lut + (int64_t)ch * 2 * kMaxLut;
        for (int code = threadIdx.x; code < ncode; code += kBT) {
            lut[code] = s_m[code];
            lut[kMaxLut + code] = s_a1[code];
        }
    }
    if (fin) {
        const double g64 = (double)gam;
        const double cntd = (double)(a.n * a.hw);
        if (a.grad_beta) a.grad_beta[ch] = __double2float_rn((double)fin_gb + s[0]);
        if (a.grad_gamma) a.grad_gamma[ch] = __double2float_rn((double)fin_gg + s[1]);
        a.stats[ch] = __double2float_rn(g64 * s[0] / cntd);                   // t2 = mean g1
        a.stats[a.c + ch] = __double2float_rn(g64 * s[2] / cntd);             // t3 = mean a1v*g1
        a.stats[2 * a.c + ch] =
            __double2float_rn(__ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(fin_s2, a.eps))));  // inv
    }
}

struct ApplyArgs {
    const float *g3;
    qt_tape_t tape;
    int64_t n, c, h, w;
    const float *gamma, *beta, *va1, *stats, *res;
    const float *lut;
    int64_t cr, sc;
    float *g_in;
    FastDiv gppd, cd;   // hw / 8, c
    FastDiv wd;         // w
};

__device__ __forceinline__ float res_value(const ApplyArgs &a, int64_t i, int64_t pl, int ch,
                                           int64_t hw) {
    if (a.sc == 1 && a.cr == a.c) return a.res[i];
    const int64_t p = i - pl * hw;
    const int64_t y = p / a.w, x = p - y * a.w;
    if (y % a.sc || x % a.sc) return 0.f;
    const int64_t nn = pl / a.c;
    const int64_t hr = a.h / a.sc, wr = a.w / a.sc;
    return a.res[((nn * a.cr + ch) * hr + y / a.sc) * wr + x / a.sc];
}

template <bool CODES, bool VA1, int G>
__global__ void __launch_bounds__(kBT) bn_bwd_apply_kernel(ApplyArgs a) {
    pdl_enter();
    const int64_t hw = a.h * a.w;
    const int64_t numel = a.n * a.c * hw;
    const uint32_t cmask = (1u << a.tape.bits) - 1u;
    if (CODES && G > 0 && hw % G == 0 && numel / G < (1ll << 31)) {
        const uint32_t groups = (uint32_t)(numel / G);
        for (uint32_t gi = blockIdx.x * kBT + threadIdx.x; gi < groups; gi += gridDim.x * kBT) {
            const int64_t i0 = (int64_t)gi * G;
            const uint32_t pl = fast_div(gi, a.gppd);
            const int ch = (int)(pl - fast_div(pl, a.cd) * (uint32_t)a.c);
            const float gam = __ldg(a.gamma + ch);
            const float t2 = __ldg(a.stats + ch), t3 = __ldg(a.stats + a.c + ch);
            const float inv = __ldg(a.stats + 2 * a.c + ch);
            const float *lm = a.lut + (int64_t)ch * 2 * kMaxLut;
            const float4 ga = __ldg(reinterpret_cast<const float4 *>(a.g3 + i0));
            float gv[8];
            gv[0] = ga.x; gv[1] = ga.y; gv[2] = ga.z; gv[3] = ga.w;
            if (G == 8) {
                const float4 gb = __ldg(reinterpret_cast<const float4 *>(a.g3 + i0) + 1);
                gv[4] = gb.x; gv[5] = gb.y; gv[6] = gb.z; gv[7] = gb.w;
            }
            const uint64_t word = load_code_group<G>(a.tape.codes, i0, a.tape.bits);
            float o[8];
#pragma unroll
            for (int j = 0; j < (G > 0 ? G : 1); ++j) {
                const uint32_t code = (uint32_t)(word >> (j * a.tape.bits)) & cmask;
                const float m = __ldg(lm + code), a1 = __ldg(lm + kMaxLut + code);
                const float g1 = __fmul_rn(__fmul_rn(gv[j], m), gam);
                const float a1v = VA1 ? a.va1[i0 + j] : a1;
                float r = __fsub_rn(g1, t2);                       // layer.py:305
                r = __fsub_rn(r, __fmul_rn(a1v, t3));              // :306
                o[j] = __fmul_rn(r, inv);                          // :307
            }
            if (a.res) {
                if (a.sc == 1 && a.cr == a.c) {
                    const float4 ra = __ldg(reinterpret_cast<const float4 *>(a.res + i0));
                    o[0] = __fadd_rn(o[0], ra.x); o[1] = __fadd_rn(o[1], ra.y);
                    o[2] = __fadd_rn(o[2], ra.z); o[3] = __fadd_rn(o[3], ra.w);
                    if (G == 8) {
                        const float4 rb = __ldg(reinterpret_cast<const float4 *>(a.res + i0) + 1);
                        o[4] = __fadd_rn(o[4], rb.x); o[5] = __fadd_rn(o[5], rb.y);
                        o[6] = __fadd_rn(o[6], rb.z); o[7] = __fadd_rn(o[7], rb.w);
                    }
                } else if (ch < a.cr) {
                    // shortcut adjoint at a lower resolution (engine.py:270-279):
                    // the group's pixels start in row y and may wrap into row
                    // y + 1 (w >= G, so at most once)
                    const uint32_t off = (uint32_t)(i0 - (int64_t)pl * hw);
                    const uint32_t y = fast_div(off, a.wd), x0 = off - y * (uint32_t)a.w;
                    const uint32_t sc = (uint32_t)a.sc, wv = (uint32_t)a.w;
                    const uint32_t nn = fast_div(pl, a.cd);
                    const int64_t hr = a.h / a.sc, wr = a.w / a.sc;
                    const float *rimg = a.res + ((int64_t)nn * a.cr + ch) * hr * wr;
#pragma unroll
                    for (int j = 0; j < G; ++j) {
                        const uint32_t wrap = x0 + j >= wv ? 1u : 0u;
                        const uint32_t yy = y + wrap, xx = x0 + j - wrap * wv;
                        if (yy % sc == 0 && xx % sc == 0)
                            o[j] = __fadd_rn(o[j], __ldg(rimg + (int64_t)(yy / sc) * wr + xx / sc));
                    }
                }
            }
            float4 *dst = reinterpret_cast<float4 *>(a.g_in + i0);
            dst[0] = make_float4(o[0], o[1], o[2], o[3]);
            if (G == 8) dst[1] = make_float4(o[4], o[5], o[6], o[7]);
        }
        return;
    }
    for (int64_t i = (int64_t)blockIdx.x * kBT + threadIdx.x; i < numel;
         i += (int64_t)gridDim.x * kBT) {
        const int64_t pl = i / hw;
        const int ch = (int)(pl % a.c);
        const float gam = a.gamma[ch];
        float m, a1;
        if (CODES) {
            const uint32_t code = get_code(a.tape.codes, i, a.tape.bits);
            const float *lm = a.lut + (int64_t)ch * 2 * kMaxLut;
            m = lm[code];
            a1 = lm[kMaxLut + code];
        } else {
            const float a2 = a.tape.a2[i];
            m = a2 > 0.f ? 1.f : 0.f;
            a1 = __fdiv_rn(__fsub_rn(a2, a.beta[ch]), safe_gamma(gam));
        }
        const float g1 = __fmul_rn(__fmul_rn(a.g3[i], m), gam);
        const float a1v = VA1 ? a.va1[i] : a1;
        float r = __fsub_rn(g1, a.stats[ch]);
        r = __fsub_rn(r, __fmul_rn(a1v, a.stats[a.c + ch]));
        r = __fmul_rn(r, a.stats[2 * a.c + ch]);
        if (a.res) r = __fadd_rn(r, res_value(a, i, pl, ch, hw));
        a.g_in[i] = r;
    }
}

}  // namespace qt

using namespace qt;

extern "C" int64_t qt_bn_backward_workspace(int64_t n, int64_t c, int64_t hw) {
    BwdPart p = bwd_partition(n, c, hw);
    return kBwdCounterBytes + c * 2 * kMaxLut * (int64_t)sizeof(float) +
           c * p.nb * 4 * (int64_t)sizeof(double);
}

extern "C" int qt_bn_backward_reduce(const float *g3, qt_tape_t tape, int64_t n, int64_t c,
                                     int64_t hw, const float *gamma_tape, const float *beta_tape,
                                     const double *sigma2, double eps, const float *variance_a1,
                                     float *grad_gamma, float *grad_beta, float *stats, void *ws,
                                     qt_stream_t stream) {
    QT_REQUIRE(g3 && gamma_tape && beta_tape && sigma2 && stats && ws);
    QT_REQUIRE(n > 0 && c > 0 && hw > 0 && c <= 65535);
    QT_REQUIRE(tape.a2 || (tape.codes && tape.step && tape.offset && qt_bits_ok(tape.bits)));
    BwdPart p = reduce_partition(n, c, hw);
    const bool codes = tape.a2 == nullptr;
    if (!codes) tape.bits = 1;
    BwdArgs a{g3, tape, n, c, hw, gamma_tape, beta_tape, sigma2, eps, variance_a1, grad_gamma,
              grad_beta, stats, p.ppb, p.nb, part_base(ws, c), (unsigned *)ws, lut_base(ws)};
    // the vector group width (hence the summation order) depends on the shape
    // and code width only, never on the tape type
    const int G = bn_group(hw, hw);
    a.gppd = make_fastdiv((uint32_t)std::max<int64_t>(1, hw / (G > 0 ? G : 8)));
    a.hwd = make_fastdiv((uint32_t)std::max<int64_t>(1, std::min<int64_t>(hw, INT32_MAX)));
    dim3 grid((unsigned)p.nb, (unsigned)c);
    cudaStream_t s = qt_s(stream);
#define QT_RED(GG)                                                                                \
    (codes ? (variance_a1 ? launch_pdl_cluster(bn_bwd_reduce_kernel<true, true, GG>, grid, kBT, 0, s, (unsigned)p.nb, a)   \
                          : launch_pdl_cluster(bn_bwd_reduce_kernel<true, false, GG>, grid, kBT, 0, s, (unsigned)p.nb, a)) \
           : (variance_a1 ? launch_pdl_cluster(bn_bwd_reduce_kernel<false, true, GG>, grid, kBT, 0, s, (unsigned)p.nb, a)  \
                          : launch_pdl_cluster(bn_bwd_reduce_kernel<false, false, GG>, grid, kBT, 0, s, (unsigned)p.nb, a)))
    if (G == 8) QT_RED(8);
    else if (G == 4) QT_RED(4);
    else QT_RED(0);
#undef QT_RED
    QT_CHECK_LAUNCH();
    return QT_OK;
}

extern "C" int qt_bn_backward_apply(const float *g3, qt_tape_t tape, int64_t n, int64_t c,
                                    int64_t h, int64_t w, const float *gamma_tape,
                                    const float *beta_tape, const float *variance_a1,
                                    const float *stats, const float *res_g, int64_t cr, int64_t sc,
                                    const void *ws, float *g_in, qt_stream_t stream) {
    QT_REQUIRE(g3 && gamma_tape && beta_tape && stats && g_in && ws && n > 0 && c > 0 && h > 0 &&
               w > 0);
    QT_REQUIRE(tape.a2 || (tape.codes && tape.step && tape.offset && qt_bits_ok(tape.bits)));
    QT_REQUIRE(!res_g || (sc >= 1 && h % sc == 0 && w % sc == 0 && cr >= c));
    const bool codes = tape.a2 == nullptr;
    if (!codes) tape.bits = 1;
    ApplyArgs a{g3, tape, n, c, h, w, gamma_tape, beta_tape, variance_a1, stats, res_g,
                lut_base((void *)ws), cr, sc, g_in};
    const int G = codes ? bn_group(h * w, w) : 0;
    a.gppd = make_fastdiv((uint32_t)std::max<int64_t>(1, (h * w) / (G > 0 ? G : 8)));
    a.cd = make_fastdiv((uint32_t)c);
    a.wd = make_fastdiv((uint32_t)w);
    const int64_t work = G > 0 ? (n * c * h * w) / G : n * c * h * w;
    static const int64_t maxb = qt_env_i64("QTAPE_APPLY_MAXB", qt_sm_count() * 16);
    static const int64_t gpt = qt_env_i64("QTAPE_APPLY_GPT", 1);
    int64_t blocks = std::min<int64_t>(qt_cdiv(work, gpt * kBT), maxb);
    blocks = std::max<int64_t>(blocks, 1);
    cudaStream_t s = qt_s(stream);
    const unsigned nb = (unsigned)blocks;
#define QT_APP(GG)                                                                                \
    (codes ? (variance_a1 ? launch_pdl(bn_bwd_apply_kernel<true, true, GG>, nb, kBT, 0, s, a)      \
                          : launch_pdl(bn_bwd_apply_kernel<true, false, GG>, nb, kBT, 0, s, a))    \
           : (variance_a1 ? launch_pdl(bn_bwd_apply_kernel<false, true, GG>, nb, kBT, 0, s, a)     \
                          : launch_pdl(bn_bwd_apply_kernel<false, false, GG>, nb, kBT, 0, s, a)))
    if (G == 8) QT_APP(8);
    else if (G == 4) QT_APP(4);
    else QT_APP(0);
#undef QT_APP
    QT_CHECK_LAUNCH();
    return QT_OK;
}
