// Shared device helpers for the qtape_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <utility>

#include "../../include/qtape_b200.h"

#define QT_CHECK_LAUNCH()                              \
    do {                                               \
        cudaError_t e__ = cudaGetLastError();          \
        if (e__ != cudaSuccess) return (int)e__;       \
    } while (0)

#define QT_REQUIRE(cond)                               \
    do {                                               \
        if (!(cond)) return QT_EINVAL;                 \
    } while (0)

static inline cudaStream_t qt_s(qt_stream_t s) { return (cudaStream_t)s; }

static inline bool qt_bits_ok(int b) { return b == 1 || b == 2 || b == 4 || b == 8; }

static inline int64_t qt_cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// SM count of the current device (cached per device ordinal; one process
// drives one GPU, but a process may switch devices between calls).
static inline int qt_sm_count() {
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
    if (!cache[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = n > 0 ? n : 1;
    }
    return cache[dev];
}

// Programmatic dependent launch: every kernel is launched with programmatic
// stream serialization, triggers its dependents as soon as it starts and
// waits (griddepcontrol.wait) for its predecessor before touching global
// memory, so a kernel's launch and prologue (barrier init, TMEM allocation,
// tensor-map prefetch) overlap the previous kernel's tail.  QTAPE_NO_PDL=1
// launches without the attribute (the wait then returns immediately).
static inline bool qt_pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("QTAPE_NO_PDL");
        v = (e && *e && *e != '0') ? 0 : 1;
    }
    return v == 1;
}
// Reduction partition knobs (tuning only): elements per block and the
// divisor that spreads small layers (blocks per channel >= n*c / div).
static inline int64_t qt_env_i64(const char *name, int64_t dflt) {
    const char *e = getenv(name);
    return (e && *e) ? (int64_t)atoll(e) : dflt;
}
// elements per reduction block before the >= 2 blocks / SM cap (n*c / DIV)
// decides: measured 8192 -> 32768 (plateau to 2^20) C2 8.55 -> 8.42 ms/step,
// C3 50.9 -> 50.4, C4 43.5 -> 42.8 (BN statistics and backward reduce)
static inline int64_t qt_red_target() {
    static int64_t v = qt_env_i64("QTAPE_RED_TGT", 32768);
    return v;
}
static inline int64_t qt_red_div() {
    static int64_t v = qt_env_i64("QTAPE_RED_DIV", 2 * qt_sm_count());
    return v;
}
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                     cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = qt_pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Same, with a thread-block cluster of `cx` CTAs along x (the blocks of one
// channel reduce through distributed shared memory instead of a global
// counter).
// Blocks per channel (= cluster size) of the clustered reductions; above 8
// needs the non-portable cluster attribute (set at launch).
static inline int64_t qt_red_cluster() {
    static int64_t v = qt_env_i64("QTAPE_RED_CLUSTER", 8);
    return v;
}
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block,
                                             size_t smem, cudaStream_t st, unsigned cx,
                                             Args &&...args) {
    if (cx > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cx;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = qt_pdl_enabled() ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

namespace qt {

// qt_set_concurrent_backward (dense.cu): split the SMs between the data- and
// weight-gradient GEMMs of small layers
extern int g_concurrent_bwd;
constexpr double kSmallLayerMacs = 1073741824.0;   // 2^30

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// elementwise / reduction kernels: no prologue worth overlapping
__device__ __forceinline__ void pdl_enter() {
    pdl_wait();
    pdl_trigger();
}

// Cluster-wide barrier (release/acquire: shared-memory writes before it are
// visible to every CTA of the cluster after it).
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Load a double from CTA `rank`'s copy of the shared variable at `p`.
__device__ __forceinline__ double ld_dsmem_f64(const double *p, unsigned rank) {
    uint32_t local = (uint32_t)__cvta_generic_to_shared(p), remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank));
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote) : "memory");
    return v;
}

constexpr double kGammaFloor = 1e-8;   // codec.py:24
constexpr float kGammaFloorF = 1e-8f;  // layer.py:134 (dtype.type(GAMMA_FLOOR))

// x86 numpy float64 -> int64 cast: cvttsd2si yields INT64_MIN ("integer
// indefinite") for NaN, +-inf and anything outside [-2^63, 2^63).
__device__ __forceinline__ int64_t x86_f64_to_i64(double d) {
    if (d >= -9223372036854775808.0 && d < 9223372036854775808.0) return (int64_t)d;
    return INT64_MIN;
}

// Codec constants for one channel, bit-exact with codec._scales and the
// offset computation (codec.py:101-104, :117).
struct ChanCode {
    double scale;   // 2^K / (6 g)
    double step;    // 6 g 2^-K
    int64_t off;    // floor(beta * scale) via x86 cast
};

__device__ __forceinline__ ChanCode chan_code(float gamma, float beta, int bits) {
    double g = fabs((double)gamma);
    g = g > kGammaFloor ? g : kGammaFloor;           // np.maximum (NaN-propagating
    if (isnan((double)gamma)) g = (double)gamma;     //  like numpy)
    double g6 = __dmul_rn(6.0, g);
    ChanCode r;
    r.scale = __ddiv_rn(ldexp(1.0, bits), g6);
    r.step = __dmul_rn(g6, ldexp(1.0, -bits));
    r.off = x86_f64_to_i64(floor(__dmul_rn((double)beta, r.scale)));
    return r;
}

// Per-channel constants of the fused BN-apply + quantize (32 bytes).
struct BnConst {
    float m32, inv32, g, b;   // (float)mean, (float)(1/sqrt(var+eps)), gamma, beta
    double scale;             // 2^K / (6 g)       (codec.py:101-104)
    double step;              // 6 g 2^-K
    int64_t off;              // floor(beta * scale) via x86 cast
    float s1, s2;             // scale = s1 + s2 (+ < 2^-48 rel): code_fast
};

// bn_const with the channel's code constants already computed (they depend
// on gamma / beta only, so a finalizer can evaluate them off the critical path)
__device__ __forceinline__ BnConst bn_const_cc(double mean, double var, double eps, float gamma,
                                               float beta, int bits, const ChanCode &cc) {
    BnConst k;
    const double inv = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(var, eps)));   // layer.py:245
    k.m32 = __double2float_rn(mean);
    k.inv32 = __double2float_rn(inv);
    k.g = gamma;
    k.b = beta;
    k.scale = 0.0;
    k.step = 0.0;
    k.off = 0;
    k.s1 = k.s2 = 0.f;
    if (bits) {
        k.scale = cc.scale;
        k.step = cc.step;
        k.off = cc.off;
        k.s1 = __double2float_rn(cc.scale);
        k.s2 = __double2float_rn(cc.scale - (double)k.s1);
    }
    return k;
}

__device__ __forceinline__ BnConst bn_const(double mean, double var, double eps, float gamma,
                                            float beta, int bits) {
    ChanCode cc{};
    if (bits) cc = chan_code(gamma, beta, bits);
    return bn_const_cc(mean, var, eps, gamma, beta, bits, cc);
}

// Unclipped code with wrapping int64 arithmetic (codec.py:118-120).
__device__ __forceinline__ int64_t raw_code(float a, double scale, int64_t off, int bits) {
    int64_t u = x86_f64_to_i64(floor(__dmul_rn((double)a, scale)));
    uint64_t r = (uint64_t)u + (uint64_t)(1ll << (bits - 1)) - (uint64_t)off;
    return (int64_t)r;
}

// Same code (clamped to [0, 2^K-1]) and clip flag as raw_code, without
// float64 arithmetic on the common path: a*scale is evaluated as
// p + e + a*s2 (p = fl32(a*s1), e its exact FMA error, s1 + s2 = scale), and
// floor() is taken from the fp32 value when the fraction is more than 2^-20
// away from an integer (the float64 product's floor is then the same);
// non-finite / large values, huge offsets and near-integer products take the
// exact float64 path.  Returns the clamped code, sets *clipped.
__device__ __forceinline__ uint32_t code_fast(float a, float s1, float s2, double scale, int64_t off,
                                              int bits, bool *clipped) {
    const float p = __fmul_rn(a, s1);
    const float e = __fmaf_rn(a, s1, -p);
    const float corr = __fmaf_rn(a, s2, e);
    const float f = floorf(p);
    const float fr = __fadd_rn(__fsub_rn(p, f), corr);   // p - f exact
    const int64_t top = (1ll << bits) - 1;
    const float margin = 9.5367431640625e-07f;            // 2^-20
    const bool fast = fabsf(p) < 1048576.f && off > -(1ll << 30) && off < (1ll << 30) &&
                      fabsf(fr) > margin && fabsf(fr - 1.f) > margin && fr > -1.f && fr < 2.f;
    int64_t raw;
    if (fast) {
        // integer value of f (|f| < 2^20) without a conversion instruction
        const int u = (__float_as_int(__fadd_rn(f, 12582912.f)) - 0x4B400000) +
                      (fr < 0.f ? -1 : (fr >= 1.f ? 1 : 0));
        raw = (int64_t)u + (1ll << (bits - 1)) - off;
    } else {
        raw = raw_code(a, scale, off, bits);
    }
    *clipped = raw < 0 || raw > top;
    return (uint32_t)(raw < 0 ? 0 : (raw > top ? top : raw));
}

// code_fast split for unrolled callers: the fp32/int32 common path and a
// flag when the element needs the exact float64 recipe (code_slow, kept out
// of line so the rare path costs a call, not if-converted float64 work).
__device__ __forceinline__ uint32_t code_fast_only(float a, float s1, float s2, int64_t off,
                                                   int bits, bool *clipped, bool *slow) {
    const float p = __fmul_rn(a, s1);
    const float e = __fmaf_rn(a, s1, -p);
    const float corr = __fmaf_rn(a, s2, e);
    const float f = floorf(p);
    const float fr = __fadd_rn(__fsub_rn(p, f), corr);   // p - f exact
    const float dist = fabsf(__fsub_rn(fr, rintf(fr)));
    const bool off_ok = off > -(1ll << 30) && off < (1ll << 30);
    *slow = !(fabsf(p) < 1048576.f && dist > 9.5367431640625e-07f && off_ok);
    // floor(a*scale) = f + floor(fr) (|f| < 2^20): its int value from the float bits
    const float u = __fadd_rn(__fadd_rn(f, floorf(fr)), 12582912.f);
    const int raw = __float_as_int(u) - 0x4B400000 + (1 << (bits - 1)) - (int)(off_ok ? off : 0);
    const int top = (1 << bits) - 1;
    const int c = min(max(raw, 0), top);
    *clipped = raw != c;
    return (uint32_t)c;
}

static __device__ __noinline__ uint32_t code_slow(float a, double scale, int64_t off, int bits,
                                           bool *clipped) {
    const int64_t top = (1ll << bits) - 1;
    const int64_t raw = raw_code(a, scale, off, bits);
    *clipped = raw < 0 || raw > top;
    return (uint32_t)(raw < 0 ? 0 : (raw > top ? top : raw));
}

// Interval-median decode (codec.py:149-154), rounded to the tape dtype.
__device__ __forceinline__ float decode(uint32_t code, double step, int64_t off, int bits) {
    double half = (double)(1 << (bits - 1));
    double inner = __dadd_rn((double)code, 0.5 - half);
    inner = __dadd_rn(inner, (double)off);
    return __double2float_rn(__dmul_rn(step, inner));
}

__device__ __forceinline__ uint32_t get_code(const uint8_t *codes, int64_t i, int bits) {
    if (bits == 8) return codes[i];
    int64_t bit = i * bits;
    return (codes[bit >> 3] >> (bit & 7)) & ((1u << bits) - 1u);
}

// Pre-ReLU activation of element i from a tape (fp32 copy or codes).
__device__ __forceinline__ float tape_value(const qt_tape_t &t, int64_t i, int c) {
    if (t.a2) return t.a2[i];
    return decode(get_code(t.codes, i, t.bits), t.step[c], t.offset[c], t.bits);
}

__device__ __forceinline__ float safe_gamma(float g) {
    float mag = fabsf(g);
    mag = mag > kGammaFloorF ? mag : kGammaFloorF;
    if (isnan(g)) mag = g;
    return g < 0.f ? -mag : mag;
}

// Division by a launch-invariant divisor for numerators below 2^31
// (Granlund-Montgomery: q = (umulhi(x, m) + x) >> s), prepared on the host.
struct FastDiv {
    uint32_t d, m, s;
};
static inline FastDiv make_fastdiv(uint32_t d) {
    FastDiv f;
    f.d = d;
    f.s = 0;
    while ((1ull << f.s) < d) ++f.s;
    f.m = (uint32_t)(((((uint64_t)1) << 32) * ((((uint64_t)1) << f.s) - d)) / d + 1);
    return f;
}
__device__ __forceinline__ uint32_t fast_div(uint32_t x, const FastDiv &f) {
    return (__umulhi(x, f.m) + x) >> f.s;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Convolution geometry (NCHW input n x ci x h x w, kernel co x ci x kh x kw).
struct ConvGeo {
    int64_t n, ci, h, w, co, kh, kw, s, pad, oh, ow;
};

}  // namespace qt
