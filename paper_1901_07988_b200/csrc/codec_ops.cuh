// Shared by codec.cu and bn.cu (both compiled with -fmad=false, IEEE div /
// sqrt, no FTZ): the fp32 fast path of the K-bit quantizer with its exact
// float64 fallback.
#pragma once
#include "common.cuh"

namespace qt {

// Codes of 8 consecutive A2 values of one channel (approx / naive modes).
// Common path: ONE fp32 fma per element, y = fl(a * s1 + c) with s1 =
// fl32(scale) and c = 2^(K-1) - offset (an exact small float).  Against the
// reference raw = floor(fl64(a * scale)) + c (codec.py:118-120), y is off by
// at most ulp(y)/2 + 2^-24 (|y| + |c| + 1)(1 + 2^-29) (the fma rounding, the
// dropped low part of the scale, the float64 product's rounding), so when
// y's fraction is farther than `marg` (twice that bound) from an integer,
// floor(y) is exactly the reference's raw code.  Elements within marg of an
// integer that could change the clamped code or the clip flag (y in
// (-2, 2^K + 2)), non-finite or |y| >= 2^20 values, and channels with
// |offset| >= 2^20 take the exact float64 recipe (rare).
struct QuantK {
    float s1, cf, marg;
    bool ok;          // |offset| < 2^20: the fp32 common path applies
    double scale;
    int64_t off;
};

template <int BITS>
__device__ __forceinline__ QuantK quant_consts(float s1, double scale, int64_t off) {
    QuantK q;
    q.ok = off > -(1ll << 20) && off < (1ll << 20);
    q.s1 = s1;
    q.cf = q.ok ? (float)((1 << (BITS - 1)) - (int)off) : 0.f;
    // 2^-15 + (|c| + 2^K + 8) 2^-23 >= 2 x the bound above for |y| < 2^K + 2
    q.marg = __fmaf_rn(__fadd_rn(fabsf(q.cf), (float)((1 << BITS) + 8)), 1.1920928955078125e-07f,
                       3.0517578125e-05f);
    q.scale = scale;
    q.off = off;
    return q;
}

template <int BITS, bool LAZY = false>
__device__ __forceinline__ void quant8(const float (&v)[8], const QuantK &k, uint32_t (&code)[8],
                                       uint32_t &clipmask, const float *lazy_g = nullptr,
                                       const float *lazy_b = nullptr) {
    constexpr int top = (1 << BITS) - 1;
    constexpr float mid = 0.5f * (float)top, half_span = 0.5f * (float)top + 2.0f;
    uint32_t slow = k.ok ? 0u : 0xFFu;
    clipmask = 0u;
    const float hi_m = __fsub_rn(1.0f, k.marg);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const float y = __fmaf_rn(v[j], k.s1, k.cf);
        const float f = floorf(y);
        const float fr = __fsub_rn(y, f);              // exact
        const bool inrange = fabsf(__fsub_rn(y, mid)) < half_span;   // y in (-2, 2^K + 2)
        const bool near = (fr <= k.marg) | (fr >= hi_m);
        if (!(fabsf(y) < 1048576.f) | (inrange & near)) slow |= 1u << j;
        const int raw = __float_as_int(__fadd_rn(f, 12582912.f)) - 0x4B400000;   // |f| < 2^22
        const int c = min(max(raw, 0), top);
        code[j] = (uint32_t)c;
        clipmask |= (raw != c) ? (1u << j) : 0u;
    }
    if (slow) {
        const double scale = LAZY ? chan_code(*lazy_g, *lazy_b, BITS).scale : k.scale;
#pragma unroll 1
        for (int j = 0; j < 8; ++j) {
            if (!((slow >> j) & 1u)) continue;
            const int64_t raw = raw_code(v[j], scale, k.off, BITS);
            const bool cl = raw < 0 || raw > top;
            code[j] = (uint32_t)(raw < 0 ? 0 : (raw > top ? top : raw));
            clipmask = (clipmask & ~(1u << j)) | (cl ? (1u << j) : 0u);
        }
    }
}


}  // namespace qt
