// K-bit activation codec and the fused forward K1 (BN apply -> tape -> ReLU).
//
// Bit-exact with the reference codec (codec.py:59-156) and BN apply
// (layer.py:245-264): every float op is an explicit round-to-nearest
// intrinsic (no FMA contraction, no FTZ) and the float64 -> int64 cast
// emulates x86 numpy (see common.cuh).
//
// Layout: a thread owns a group of 8 consecutive flat-NCHW elements, i.e.
// K bytes of packed codes (K in {1,2,4,8}); a 256-thread block owns 2048
// consecutive elements.  Loads/stores are 128-bit for the fp32 streams and
// one K-byte store for the codes, so a warp writes 32*K contiguous code
// bytes.  Per-(n,c)-plane constants (mean/inv/gamma/beta/scale/offset) are
// computed once per block into shared memory.
#include <algorithm>

#include "common.cuh"

namespace qt {

constexpr int kThreads = 256;
constexpr int kGroup = 8;
constexpr int kBlockElems = kThreads * kGroup;
constexpr int kMaxPlanes = 258;  // planes a 2048-element block can touch for hw >= 8

struct PlaneConst {
    double scale;
    double step;
    int64_t off;
    float m32, inv32, g, b;
};

enum { MODE_EXACT = 0, MODE_APPROX = 1, MODE_NAIVE = 2 };

struct FwdArgs {
    const float *x;
    int64_t numel, c, hw;
    const double *mean, *var;
    double eps;
    const float *gamma, *beta;
    int mode, bits;  // bits == 0: identity bypass (no codes)
    float *a3_out;
    float *a2_tape;
    uint8_t *codes;
    double *step;
    int64_t *offset;
    unsigned long long *clip_count;
    const BnConst *consts;   // optional: per-channel constants from qt_bn_stats_prep
    FastDiv hw8d, cd;        // stream kernel: group -> plane -> channel (32-bit)
    FastDiv hw4d;            // fused stream kernel: half group -> plane (hw % 4 == 0)
};

__device__ __forceinline__ PlaneConst make_plane(const FwdArgs &a, int64_t ch, bool apply_bn) {
    PlaneConst p;
    if (a.consts) {
        const BnConst k = a.consts[ch];
        p.m32 = k.m32;
        p.inv32 = k.inv32;
        p.g = k.g;
        p.b = k.b;
        p.scale = k.scale;
        p.step = k.step;
        p.off = k.off;
        return p;
    }
    if (apply_bn) {
        double inv = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(a.var[ch], a.eps)));  // layer.py:245
        p.m32 = __double2float_rn(a.mean[ch]);
        p.inv32 = __double2float_rn(inv);
    } else {
        p.m32 = 0.f;
        p.inv32 = 1.f;
    }
    p.g = a.gamma[ch];
    p.b = a.beta[ch];
    if (a.bits) {
        ChanCode cc = chan_code(p.g, p.b, a.bits);
        p.scale = cc.scale;
        p.step = cc.step;
        p.off = cc.off;
    }
    return p;
}

__device__ __forceinline__ float relu_np(float v) {
    // np.maximum(v, 0): keeps NaN and -0.0 (layer.py:264)
    return (v >= 0.f || isnan(v)) ? v : 0.f;
}

template <bool APPLY_BN>
__global__ void __launch_bounds__(kThreads) bn_relu_quant_kernel(FwdArgs a) {
    pdl_enter();
    __shared__ PlaneConst sp[kMaxPlanes];
    __shared__ unsigned long long s_clip[kThreads / 32];

    const int64_t blk0 = (int64_t)blockIdx.x * kBlockElems;
    const int64_t blk1 = min(blk0 + kBlockElems, a.numel);
    const int64_t plane0 = blk0 / a.hw;
    const int64_t nplanes = (blk1 - 1) / a.hw - plane0 + 1;
    const bool staged = nplanes <= kMaxPlanes;
    if (staged) {
        for (int64_t q = threadIdx.x; q < nplanes; q += kThreads)
            sp[q] = make_plane(a, (plane0 + q) % a.c, APPLY_BN);
    }
    // tape constants: frozen step/offset per channel (codec.py:137-143)
    if (a.bits && a.step && !a.consts) {
        for (int64_t ch = (int64_t)blockIdx.x * kThreads + threadIdx.x; ch < a.c;
             ch += (int64_t)gridDim.x * kThreads) {
            ChanCode cc = chan_code(a.gamma[ch], a.beta[ch], a.bits);
            a.step[ch] = cc.step;
            a.offset[ch] = cc.off;
        }
    }
    __syncthreads();

    const int64_t i0 = blk0 + (int64_t)threadIdx.x * kGroup;
    unsigned long long clip = 0;
    if (i0 < a.numel) {
        const int cnt = (int)min((int64_t)kGroup, a.numel - i0);
        float xv[kGroup];
        const bool vec = (cnt == kGroup) && ((((uintptr_t)(a.x + i0)) & 15) == 0);
        if (vec) {
            float4 u = __ldg(reinterpret_cast<const float4 *>(a.x + i0));
            float4 v = __ldg(reinterpret_cast<const float4 *>(a.x + i0) + 1);
            xv[0] = u.x; xv[1] = u.y; xv[2] = u.z; xv[3] = u.w;
            xv[4] = v.x; xv[5] = v.y; xv[6] = v.z; xv[7] = v.w;
        } else {
#pragma unroll
            for (int j = 0; j < kGroup; ++j) xv[j] = j < cnt ? a.x[i0 + j] : 0.f;
        }
        float a2v[kGroup], a3v[kGroup];
        uint64_t word = 0;
        int64_t pl = i0 / a.hw;
        int64_t rem = i0 - pl * a.hw;
        PlaneConst pc = staged ? sp[pl - plane0] : make_plane(a, pl % a.c, APPLY_BN);
#pragma unroll
        for (int j = 0; j < kGroup; ++j) {
            if (j < cnt) {
                if (rem == a.hw) {  // crossed into the next (n,c) plane
                    ++pl;
                    rem = 0;
                    pc = staged ? sp[pl - plane0] : make_plane(a, pl % a.c, APPLY_BN);
                }
                float v = xv[j];
                if (APPLY_BN) {  // four separately rounded ops, layer.py:246-249
                    v = __fsub_rn(v, pc.m32);
                    v = __fmul_rn(v, pc.inv32);
                    v = __fmul_rn(v, pc.g);
                    v = __fadd_rn(v, pc.b);
                }
                a2v[j] = v;
                float pre = v;
                if (a.bits) {
                    int64_t raw = raw_code(v, pc.scale, pc.off, a.bits);
                    const int64_t top = (1ll << a.bits) - 1;
                    clip += (raw < 0 || raw > top);
                    uint32_t code = (uint32_t)(raw < 0 ? 0 : (raw > top ? top : raw));
                    word |= (uint64_t)code << (j * a.bits);
                    if (a.mode == MODE_NAIVE) pre = decode(code, pc.step, pc.off, a.bits);
                }
                a3v[j] = relu_np(pre);
                ++rem;
            } else {
                a2v[j] = 0.f;
                a3v[j] = 0.f;
            }
        }
        if (vec) {
            if (a.a2_tape) {
                float4 *d = reinterpret_cast<float4 *>(a.a2_tape + i0);
                d[0] = make_float4(a2v[0], a2v[1], a2v[2], a2v[3]);
                d[1] = make_float4(a2v[4], a2v[5], a2v[6], a2v[7]);
            }
            if (a.a3_out) {
                float4 *d = reinterpret_cast<float4 *>(a.a3_out + i0);
                d[0] = make_float4(a3v[0], a3v[1], a3v[2], a3v[3]);
                d[1] = make_float4(a3v[4], a3v[5], a3v[6], a3v[7]);
            }
        } else {
            for (int j = 0; j < cnt; ++j) {
                if (a.a2_tape) a.a2_tape[i0 + j] = a2v[j];
                if (a.a3_out) a.a3_out[i0 + j] = a3v[j];
            }
        }
        if (a.bits && a.codes) {
            // group g = i0/8 owns bytes [g*K, g*K + K)
            uint8_t *dst = a.codes + (i0 / kGroup) * a.bits;
            if (cnt == kGroup) {
                switch (a.bits) {
                    case 8: *reinterpret_cast<uint2 *>(dst) = make_uint2((uint32_t)word, (uint32_t)(word >> 32)); break;
                    case 4: *reinterpret_cast<uint32_t *>(dst) = (uint32_t)word; break;
                    case 2: *reinterpret_cast<uint16_t *>(dst) = (uint16_t)word; break;
                    default: *dst = (uint8_t)word; break;
                }
            } else {
                const int nbytes = (cnt * a.bits + 7) / 8;
                for (int b = 0; b < nbytes; ++b) dst[b] = (uint8_t)(word >> (8 * b));
            }
        }
    }
    if (a.clip_count) {
        clip = warp_sum(clip);
        if ((threadIdx.x & 31) == 0) s_clip[threadIdx.x >> 5] = clip;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < kThreads / 32; ++w) t += s_clip[w];
            if (t) atomicAdd(a.clip_count, t);
        }
    }
}

struct DecArgs {
    const uint8_t *codes;
    int64_t numel, c, hw;
    int bits;
    const double *step;
    const int64_t *offset;
    int relu;
    float *out;
};

__global__ void __launch_bounds__(kThreads) unpack_dequant_kernel(DecArgs a) {
    pdl_enter();
    __shared__ double s_step[kMaxPlanes];
    __shared__ int64_t s_off[kMaxPlanes];
    const int64_t blk0 = (int64_t)blockIdx.x * kBlockElems;
    const int64_t blk1 = min(blk0 + kBlockElems, a.numel);
    const int64_t plane0 = blk0 / a.hw;
    const int64_t nplanes = (blk1 - 1) / a.hw - plane0 + 1;
    const bool staged = nplanes <= kMaxPlanes;
    if (staged) {
        for (int64_t q = threadIdx.x; q < nplanes; q += kThreads) {
            int64_t ch = (plane0 + q) % a.c;
            s_step[q] = a.step[ch];
            s_off[q] = a.offset[ch];
        }
    }
    __syncthreads();
    const int64_t i0 = blk0 + (int64_t)threadIdx.x * kGroup;
    if (i0 >= a.numel) return;
    const int cnt = (int)min((int64_t)kGroup, a.numel - i0);
    const uint8_t *src = a.codes + (i0 / kGroup) * a.bits;
    uint64_t word = 0;
    if (cnt == kGroup) {
        switch (a.bits) {
            case 8: { uint2 u = *reinterpret_cast<const uint2 *>(src); word = u.x | ((uint64_t)u.y << 32); break; }
            case 4: word = *reinterpret_cast<const uint32_t *>(src); break;
            case 2: word = *reinterpret_cast<const uint16_t *>(src); break;
            default: word = *src; break;
        }
    } else {
        const int nbytes = (cnt * a.bits + 7) / 8;
        for (int b = 0; b < nbytes; ++b) word |= (uint64_t)src[b] << (8 * b);
    }
    float v[kGroup];
    int64_t pl = i0 / a.hw;
    int64_t rem = i0 - pl * a.hw;
    const uint32_t mask = (1u << a.bits) - 1u;
#pragma unroll
    for (int j = 0; j < kGroup; ++j) {
        if (j < cnt) {
            if (rem == a.hw) { ++pl; rem = 0; }
            double st;
            int64_t of;
            if (staged) { st = s_step[pl - plane0]; of = s_off[pl - plane0]; }
            else { int64_t ch = pl % a.c; st = a.step[ch]; of = a.offset[ch]; }
            float d = decode((uint32_t)(word >> (j * a.bits)) & mask, st, of, a.bits);
            v[j] = a.relu ? relu_np(d) : d;
            ++rem;
        } else {
            v[j] = 0.f;
        }
    }
    if (cnt == kGroup && ((((uintptr_t)(a.out + i0)) & 15) == 0)) {
        float4 *d = reinterpret_cast<float4 *>(a.out + i0);
        d[0] = make_float4(v[0], v[1], v[2], v[3]);
        d[1] = make_float4(v[4], v[5], v[6], v[7]);
    } else {
        for (int j = 0; j < cnt; ++j) a.out[i0 + j] = v[j];
    }
}

__global__ void codec_constants_kernel(const float *gamma, const float *beta, int64_t c,
                                       int bits, double *step, int64_t *offset) {
    pdl_enter();
    int64_t ch = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (ch >= c) return;
    ChanCode cc = chan_code(gamma[ch], beta[ch], bits);
    step[ch] = cc.step;
    offset[ch] = cc.off;
}

__global__ void pack_kernel(const uint8_t *codes, int64_t count, int bits, uint8_t *packed,
                            int64_t nbytes, int32_t *bad) {
    pdl_enter();
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nbytes) return;
    const int per = 8 / bits;
    uint32_t out = 0;
    bool oob = false;
    for (int j = 0; j < per; ++j) {
        int64_t i = b * per + j;
        if (i < count) {
            uint32_t v = codes[i];
            oob |= v >= (1u << bits);
            out |= (v & ((1u << bits) - 1u)) << (j * bits);
        }
    }
    packed[b] = (uint8_t)out;
    if (oob && bad) *bad = 1;
}

__global__ void unpack_kernel(const uint8_t *packed, int64_t count, int bits, uint8_t *codes) {
    pdl_enter();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    codes[i] = (uint8_t)get_code(packed, i, bits);
}

// Streaming K1 for the training path (per-channel constants precomputed by
// qt_bn_stats_prep, hw % 8 == 0): grid-stride over 8-element groups, two
// groups per iteration with all four 128-bit loads issued before any math,
// constants through the read-only cache -- no block prologue, no smem.
// Codes of 8 consecutive A2 values of one channel (approx / naive modes).
// Common path in fp32/int32 (see code_fast in common.cuh for the error
// analysis): a*scale = p + e + a*s2, floor taken from f + floor(fr) when the
// fraction fr is more than 2^-20 from an integer and |p| < 2^20; elements
// failing that (non-finite, huge, near-integer products) and channels whose
// offset is outside +-2^30 are recomputed with the exact float64 recipe.
template <int BITS>
__device__ __forceinline__ void quant8(const float (&v)[8], const BnConst &k, uint32_t (&code)[8],
                                       uint32_t &clipmask) {
    constexpr int top = (1 << BITS) - 1;
    const bool chan_ok = k.off > -(1ll << 30) && k.off < (1ll << 30);
    // u_bits = float bits of (floor(a*scale) + 1.5*2^23); raw = u_bits + bias
    const int bias = (1 << (BITS - 1)) - (int)(chan_ok ? k.off : 0) - 0x4B400000;
    uint32_t slow = chan_ok ? 0u : 0xFFu;
    clipmask = 0u;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const float p = __fmul_rn(v[j], k.s1);
        const float e = __fmaf_rn(v[j], k.s1, -p);
        const float corr = __fmaf_rn(v[j], k.s2, e);
        const float f = floorf(p);
        const float fr = __fadd_rn(__fsub_rn(p, f), corr);
        const float dist = fabsf(__fsub_rn(fr, rintf(fr)));
        if (!(fabsf(p) < 1048576.f && dist > 9.5367431640625e-07f)) slow |= 1u << j;
        const float u = __fadd_rn(__fadd_rn(f, floorf(fr)), 12582912.f);
        const int raw = __float_as_int(u) + bias;
        const int c = min(max(raw, 0), top);
        code[j] = (uint32_t)c;
        clipmask |= (raw != c) ? (1u << j) : 0u;
    }
    if (slow) {
#pragma unroll 1
        for (int j = 0; j < 8; ++j) {
            if (!((slow >> j) & 1u)) continue;
            const int64_t raw = raw_code(v[j], k.scale, k.off, BITS);
            const bool cl = raw < 0 || raw > top;
            code[j] = (uint32_t)(raw < 0 ? 0 : (raw > top ? top : raw));
            clipmask = (clipmask & ~(1u << j)) | (cl ? (1u << j) : 0u);
        }
    }
}

template <int BITS, int MODE, bool A2, bool CLIP, bool H4 = false>
__global__ void __launch_bounds__(kThreads) bn_relu_quant_stream(FwdArgs a) {
    pdl_enter();
    const int64_t ngroups = a.numel >> 3;
    const int64_t stride = (int64_t)gridDim.x * kThreads;
    unsigned long long clip = 0;
    for (int64_t g0 = (int64_t)blockIdx.x * kThreads + threadIdx.x; g0 < ngroups; g0 += 2 * stride) {
        const int64_t gs[2] = {g0, g0 + stride};
        float4 xa[2], xb[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (gs[u] < ngroups) {
                const float4 *src = reinterpret_cast<const float4 *>(a.x) + 2 * gs[u];
                xa[u] = __ldg(src);
                xb[u] = __ldg(src + 1);
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int64_t gg = gs[u];
            if (gg >= ngroups) break;
            // planes of hw % 8 == 4 pixels: a group may start in one channel
            // and end in the next (halves 0-3 / 4-7 never straddle)
            // (H4 instantiation only; hw % 8 == 0 keeps the one-channel group)
            const uint32_t pa = H4 ? fast_div(2u * (uint32_t)gg, a.hw4d) : fast_div((uint32_t)gg, a.hw8d);
            const uint32_t pb = H4 ? fast_div(2u * (uint32_t)gg + 1u, a.hw4d) : pa;
            const uint32_t ch = pa - fast_div(pa, a.cd) * (uint32_t)a.c;
            const BnConst k = a.consts[ch];
            const bool split = H4 && pb != pa;
            const BnConst kb = split ? a.consts[pb - fast_div(pb, a.cd) * (uint32_t)a.c] : k;
            const float xv[8] = {xa[u].x, xa[u].y, xa[u].z, xa[u].w, xb[u].x, xb[u].y, xb[u].z, xb[u].w};
            float a2v[8], a3v[8];
            uint64_t word = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const BnConst &kk = j < 4 ? k : kb;
                float v = __fsub_rn(xv[j], kk.m32);      // layer.py:246-249
                v = __fmul_rn(v, kk.inv32);
                v = __fmul_rn(v, kk.g);
                a2v[j] = __fadd_rn(v, kk.b);
            }
            if (BITS) {
                uint32_t code[8], clipmask;
                quant8<BITS>(a2v, k, code, clipmask);
                if (split) {   // second half with the next channel's constants
                    uint32_t code_b[8], clip_b;
                    quant8<BITS>(a2v, kb, code_b, clip_b);
#pragma unroll
                    for (int j = 4; j < 8; ++j) code[j] = code_b[j];
                    clipmask = (clipmask & 0x0Fu) | (clip_b & 0xF0u);
                }
                if (CLIP) clip += __popc(clipmask);
                if (BITS * 8 <= 32) {
                    uint32_t w32 = 0;
#pragma unroll
                    for (int j = 0; j < 8; ++j) w32 |= code[j] << (j * BITS);
                    word = w32;
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j) word |= (uint64_t)code[j] << (j * BITS);
                }
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    a3v[j] = relu_np(MODE == MODE_NAIVE ? decode(code[j], j < 4 ? k.step : kb.step,
                                                                 j < 4 ? k.off : kb.off, BITS)
                                                        : a2v[j]);
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) a3v[j] = relu_np(a2v[j]);
            }
            float4 *d3 = reinterpret_cast<float4 *>(a.a3_out) + 2 * gg;
            d3[0] = make_float4(a3v[0], a3v[1], a3v[2], a3v[3]);
            d3[1] = make_float4(a3v[4], a3v[5], a3v[6], a3v[7]);
            if (A2) {
                float4 *d2 = reinterpret_cast<float4 *>(a.a2_tape) + 2 * gg;
                d2[0] = make_float4(a2v[0], a2v[1], a2v[2], a2v[3]);
                d2[1] = make_float4(a2v[4], a2v[5], a2v[6], a2v[7]);
            }
            if (BITS) {
                uint8_t *dst = a.codes + gg * BITS;
                if (BITS == 8) *reinterpret_cast<uint2 *>(dst) = make_uint2((uint32_t)word, (uint32_t)(word >> 32));
                else if (BITS == 4) *reinterpret_cast<uint32_t *>(dst) = (uint32_t)word;
                else if (BITS == 2) *reinterpret_cast<uint16_t *>(dst) = (uint16_t)word;
                else *dst = (uint8_t)word;
            }
        }
    }
    if (CLIP) {
        __shared__ unsigned long long s_clip[kThreads / 32];
        clip = warp_sum(clip);
        if ((threadIdx.x & 31) == 0) s_clip[threadIdx.x >> 5] = clip;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < kThreads / 32; ++w) t += s_clip[w];
            if (t) atomicAdd(a.clip_count, t);
        }
    }
}

// Quantize-pack from A2 (codec.quantize, codec.py:123-143) as a streaming
// kernel: 8 elements (one channel, hw % 8 == 0) per group, two groups in
// flight per thread, the per-channel constants recomputed per group (one
// float64 divide per 8 elements, L1-resident gamma/beta), the fp32 fast floor
// with the exact float64 fallback (quant8).  Threads below C also write the
// frozen step / offset.
template <int BITS, bool CLIP>
__global__ void __launch_bounds__(kThreads) quant_pack_stream(FwdArgs a) {
    pdl_enter();
    const int64_t tid = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (tid < a.c && a.step) {
        const ChanCode cc = chan_code(a.gamma[tid], a.beta[tid], BITS);
        a.step[tid] = cc.step;
        a.offset[tid] = cc.off;
    }
    const int64_t ngroups = a.numel >> 3;
    const int64_t stride = (int64_t)gridDim.x * kThreads;
    unsigned long long clip = 0;
    for (int64_t g0 = tid; g0 < ngroups; g0 += 2 * stride) {
        const int64_t gs[2] = {g0, g0 + stride};
        float4 xa[2], xb[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (gs[u] < ngroups) {
                const float4 *src = reinterpret_cast<const float4 *>(a.x) + 2 * gs[u];
                xa[u] = __ldcs(src);
                xb[u] = __ldcs(src + 1);
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int64_t gg = gs[u];
            if (gg >= ngroups) break;
            const uint32_t plane = fast_div((uint32_t)gg, a.hw8d);
            const uint32_t ch = plane - fast_div(plane, a.cd) * (uint32_t)a.c;
            const ChanCode cc = chan_code(__ldg(a.gamma + ch), __ldg(a.beta + ch), BITS);
            BnConst k;
            k.scale = cc.scale;
            k.step = cc.step;
            k.off = cc.off;
            k.s1 = __double2float_rn(cc.scale);
            k.s2 = __double2float_rn(cc.scale - (double)k.s1);
            const float xv[8] = {xa[u].x, xa[u].y, xa[u].z, xa[u].w, xb[u].x, xb[u].y, xb[u].z, xb[u].w};
            uint32_t code[8], clipmask;
            quant8<BITS>(xv, k, code, clipmask);
            if (CLIP) clip += __popc(clipmask);
            uint8_t *dst = a.codes + gg * BITS;
            if (BITS == 8) {
                uint64_t word = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) word |= (uint64_t)code[j] << (j * 8);
                *reinterpret_cast<uint2 *>(dst) = make_uint2((uint32_t)word, (uint32_t)(word >> 32));
            } else {
                uint32_t w32 = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) w32 |= code[j] << (j * BITS);
                if (BITS == 4) *reinterpret_cast<uint32_t *>(dst) = w32;
                else if (BITS == 2) *reinterpret_cast<uint16_t *>(dst) = (uint16_t)w32;
                else *dst = (uint8_t)w32;
            }
        }
    }
    if (CLIP) {
        __shared__ unsigned long long s_clip[kThreads / 32];
        clip = warp_sum(clip);
        if ((threadIdx.x & 31) == 0) s_clip[threadIdx.x >> 5] = clip;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < kThreads / 32; ++w) t += s_clip[w];
            if (t) atomicAdd(a.clip_count, t);
        }
    }
}

// Unpack + dequantize (codec.dequantize, codec.py:146-156) as a streaming
// kernel: 8 codes -> 8 fp32 (two float4 stores) per group; decode in float64
// exactly as the reference (step * ((code + (0.5 - 2^(K-1))) + offset)).
template <int BITS>
__global__ void __launch_bounds__(kThreads) dequant_stream(DecArgs a, FastDiv hw8d, FastDiv cd) {
    pdl_enter();
    const int64_t ngroups = a.numel >> 3;
    const int64_t stride = (int64_t)gridDim.x * kThreads;
    for (int64_t g0 = (int64_t)blockIdx.x * kThreads + threadIdx.x; g0 < ngroups; g0 += 2 * stride) {
        const int64_t gs[2] = {g0, g0 + stride};
        uint64_t words[2] = {0, 0};
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (gs[u] >= ngroups) continue;
            const uint8_t *src = a.codes + gs[u] * BITS;
            if (BITS == 8) {
                const uint2 w = __ldcs(reinterpret_cast<const uint2 *>(src));
                words[u] = w.x | ((uint64_t)w.y << 32);
            } else if (BITS == 4) {
                words[u] = __ldcs(reinterpret_cast<const unsigned int *>(src));
            } else if (BITS == 2) {
                words[u] = __ldcs(reinterpret_cast<const unsigned short *>(src));
            } else {
                words[u] = __ldcs(reinterpret_cast<const unsigned char *>(src));
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int64_t gg = gs[u];
            if (gg >= ngroups) break;
            const uint32_t plane = fast_div((uint32_t)gg, hw8d);
            const uint32_t ch = plane - fast_div(plane, cd) * (uint32_t)a.c;
            const double st = __ldg(a.step + ch);
            const int64_t of = __ldg(a.offset + ch);
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float d = decode((uint32_t)(words[u] >> (j * BITS)) & ((1u << BITS) - 1u), st, of, BITS);
                v[j] = a.relu ? relu_np(d) : d;
            }
            float4 *dst = reinterpret_cast<float4 *>(a.out) + 2 * gg;
            __stcs(dst, make_float4(v[0], v[1], v[2], v[3]));
            __stcs(dst + 1, make_float4(v[4], v[5], v[6], v[7]));
        }
    }
}

template <int BITS>
static void launch_stream(const FwdArgs &a, unsigned blocks, cudaStream_t s) {
    const bool clip = a.clip_count != nullptr;
    const bool h4 = (a.hw & 7) != 0;
#define QT_ST(M, C)                                                                                 \
    (h4 ? launch_pdl(bn_relu_quant_stream<BITS, M, false, C, true>, blocks, kThreads, 0, s, a)       \
        : launch_pdl(bn_relu_quant_stream<BITS, M, false, C, false>, blocks, kThreads, 0, s, a))
    if (a.mode == MODE_NAIVE) {
        if (clip) QT_ST(MODE_NAIVE, true);
        else QT_ST(MODE_NAIVE, false);
    } else {
        if (clip) QT_ST(MODE_APPROX, true);
        else QT_ST(MODE_APPROX, false);
    }
#undef QT_ST
}

static int launch_fwd(const FwdArgs &a0, bool apply_bn, cudaStream_t s) {
    if (a0.numel == 0) return QT_OK;
    FwdArgs a = a0;
    if ((a.hw & 3) == 0 && a.hw < (1ll << 31) && a.c < (1ll << 31)) {
        a.hw8d = make_fastdiv((uint32_t)std::max<int64_t>(1, a.hw >> 3));
        a.hw4d = make_fastdiv((uint32_t)(a.hw >> 2));
        a.cd = make_fastdiv((uint32_t)a.c);
    }
    const bool aligned = ((((uintptr_t)a.x) | ((uintptr_t)a.a3_out) | ((uintptr_t)a.a2_tape)) & 15) == 0;
    if (apply_bn && a.consts && a.a3_out && (a.hw & 3) == 0 && aligned &&
        (a.bits == 0 || a.codes) && (a.numel & 7) == 0 && (a.numel >> 2) < (1ll << 31)) {
        const int64_t ngroups = a.numel >> 3;
        // one 8-element group per thread: more blocks in flight per SM
        // (C2 BN-apply + quantize 1.04 -> 1.00 ms/step; 2 or 4 per thread,
        // and block caps of 592 or 2368, were slower)
        static const int64_t gpt = qt_env_i64("QTAPE_FWD_GPT", 1);
        static const int64_t maxb = qt_env_i64("QTAPE_FWD_MAXB", qt_sm_count() * 8);
        int64_t blocks = std::min<int64_t>(qt_cdiv(ngroups, gpt * kThreads), maxb);
        blocks = std::max<int64_t>(blocks, 1);
        const unsigned b = (unsigned)blocks;
        switch (a.bits) {
            case 0:
                if ((a.hw & 7) != 0) {
                    if (a.a2_tape) launch_pdl(bn_relu_quant_stream<0, MODE_EXACT, true, false, true>, b, kThreads, 0, s, a);
                    else launch_pdl(bn_relu_quant_stream<0, MODE_EXACT, false, false, true>, b, kThreads, 0, s, a);
                } else {
                    if (a.a2_tape) launch_pdl(bn_relu_quant_stream<0, MODE_EXACT, true, false>, b, kThreads, 0, s, a);
                    else launch_pdl(bn_relu_quant_stream<0, MODE_EXACT, false, false>, b, kThreads, 0, s, a);
                }
                break;
            case 1: launch_stream<1>(a, b, s); break;
            case 2: launch_stream<2>(a, b, s); break;
            case 4: launch_stream<4>(a, b, s); break;
            case 8: launch_stream<8>(a, b, s); break;
        }
        QT_CHECK_LAUNCH();
        return QT_OK;
    }
    if (!apply_bn && a.codes && (a.hw & 7) == 0 && a.hw < (1ll << 31) && a.c < (1ll << 31) &&
        (((uintptr_t)a.x) & 15) == 0 &&
        (a.numel >> 3) < (1ll << 31)) {   // quantize-pack from A2: the streaming form
        const int64_t ngroups = a.numel >> 3;
        int64_t blocks = std::min<int64_t>(qt_cdiv(ngroups, 2 * kThreads), qt_sm_count() * 8);
        blocks = std::max<int64_t>(blocks, qt_cdiv(a.c, kThreads));   // constants for every channel
        const unsigned b = (unsigned)std::max<int64_t>(blocks, 1);
        const bool clip = a.clip_count != nullptr;
        switch (a.bits) {
            case 1: clip ? launch_pdl(quant_pack_stream<1, true>, b, kThreads, 0, s, a)
                         : launch_pdl(quant_pack_stream<1, false>, b, kThreads, 0, s, a); break;
            case 2: clip ? launch_pdl(quant_pack_stream<2, true>, b, kThreads, 0, s, a)
                         : launch_pdl(quant_pack_stream<2, false>, b, kThreads, 0, s, a); break;
            case 4: clip ? launch_pdl(quant_pack_stream<4, true>, b, kThreads, 0, s, a)
                         : launch_pdl(quant_pack_stream<4, false>, b, kThreads, 0, s, a); break;
            case 8: clip ? launch_pdl(quant_pack_stream<8, true>, b, kThreads, 0, s, a)
                         : launch_pdl(quant_pack_stream<8, false>, b, kThreads, 0, s, a); break;
        }
        QT_CHECK_LAUNCH();
        return QT_OK;
    }
    int64_t blocks = qt_cdiv(a.numel, kBlockElems);
    if (blocks > 0x7fffffff) return QT_EUNSUPPORTED;
    if (apply_bn)
        launch_pdl(bn_relu_quant_kernel<true>, (unsigned)blocks, kThreads, 0, s, a);
    else
        launch_pdl(bn_relu_quant_kernel<false>, (unsigned)blocks, kThreads, 0, s, a);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

}  // namespace qt

using namespace qt;

extern "C" int qt_codec_constants(const float *gamma, const float *beta, int64_t c, int bits,
                                  double *step, int64_t *offset, qt_stream_t stream) {
    QT_REQUIRE(qt_bits_ok(bits) && c >= 0 && gamma && beta && step && offset);
    if (c == 0) return QT_OK;
    launch_pdl(codec_constants_kernel, (unsigned)qt_cdiv(c, 256), 256, 0, qt_s(stream), gamma, beta, c, bits,
                                                                              step, offset);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

extern "C" int qt_quantize_pack(const float *a, int64_t n, int64_t c, int64_t hw,
                                const float *gamma, const float *beta, int bits, uint8_t *codes,
                                double *step, int64_t *offset, int64_t *clip_count,
                                qt_stream_t stream) {
    QT_REQUIRE(qt_bits_ok(bits) && n >= 0 && c > 0 && hw > 0 && a && gamma && beta && codes);
    FwdArgs f{};
    f.x = a;
    f.numel = n * c * hw;
    f.c = c;
    f.hw = hw;
    f.gamma = gamma;
    f.beta = beta;
    f.mode = MODE_APPROX;
    f.bits = bits;
    f.codes = codes;
    f.step = step;
    f.offset = offset;
    f.clip_count = reinterpret_cast<unsigned long long *>(clip_count);
    return launch_fwd(f, false, qt_s(stream));
}

extern "C" int qt_bn_relu_forward(const float *x, int64_t n, int64_t c, int64_t hw,
                                  const double *mean, const double *var, double eps,
                                  const float *gamma, const float *beta, int mode, int bits,
                                  float *a3_out, float *a2_tape, uint8_t *codes, double *step,
                                  int64_t *offset, int64_t *clip_count, const void *consts,
                                  qt_stream_t stream) {
    QT_REQUIRE(n >= 0 && c > 0 && hw > 0 && x && ((mean && var) || consts) && gamma && beta);
    QT_REQUIRE(mode >= 0 && mode <= 2);
    QT_REQUIRE(bits == 0 || qt_bits_ok(bits));
    QT_REQUIRE(bits == 0 || codes);
    FwdArgs f{};
    f.x = x;
    f.numel = n * c * hw;
    f.c = c;
    f.hw = hw;
    f.mean = mean;
    f.var = var;
    f.eps = eps;
    f.gamma = gamma;
    f.beta = beta;
    f.mode = mode;
    f.bits = bits;
    f.a3_out = a3_out;
    f.a2_tape = a2_tape;
    f.codes = codes;
    f.step = step;
    f.offset = offset;
    f.clip_count = reinterpret_cast<unsigned long long *>(clip_count);
    f.consts = (const BnConst *)consts;
    return launch_fwd(f, true, qt_s(stream));
}

extern "C" int qt_unpack_dequant(const uint8_t *codes, int64_t n, int64_t c, int64_t hw, int bits,
                                 const double *step, const int64_t *offset, int relu, float *out,
                                 qt_stream_t stream) {
    QT_REQUIRE(qt_bits_ok(bits) && n >= 0 && c > 0 && hw > 0 && codes && step && offset && out);
    DecArgs d{codes, n * c * hw, c, hw, bits, step, offset, relu, out};
    if (d.numel == 0) return QT_OK;
    if ((hw & 7) == 0 && hw < (1ll << 31) && c < (1ll << 31) && (((uintptr_t)out) & 15) == 0 &&
        (d.numel >> 3) < (1ll << 31)) {   // the streaming form
        const int64_t ngroups = d.numel >> 3;
        const unsigned b = (unsigned)std::max<int64_t>(
            std::min<int64_t>(qt_cdiv(ngroups, 2 * kThreads), qt_sm_count() * 8), 1);
        const FastDiv hw8d = make_fastdiv((uint32_t)(hw >> 3)), cd = make_fastdiv((uint32_t)c);
        switch (bits) {
            case 1: launch_pdl(dequant_stream<1>, b, kThreads, 0, qt_s(stream), d, hw8d, cd); break;
            case 2: launch_pdl(dequant_stream<2>, b, kThreads, 0, qt_s(stream), d, hw8d, cd); break;
            case 4: launch_pdl(dequant_stream<4>, b, kThreads, 0, qt_s(stream), d, hw8d, cd); break;
            case 8: launch_pdl(dequant_stream<8>, b, kThreads, 0, qt_s(stream), d, hw8d, cd); break;
        }
        QT_CHECK_LAUNCH();
        return QT_OK;
    }
    int64_t blocks = qt_cdiv(d.numel, kBlockElems);
    launch_pdl(unpack_dequant_kernel, (unsigned)blocks, kThreads, 0, qt_s(stream), d);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

extern "C" int qt_pack_codes(const uint8_t *codes, int64_t count, int bits, uint8_t *packed,
                             int32_t *bad, qt_stream_t stream) {
    QT_REQUIRE(qt_bits_ok(bits) && count >= 0 && (count == 0 || (codes && packed)));
    int64_t nbytes = (count * bits + 7) / 8;
    if (nbytes == 0) return QT_OK;
    launch_pdl(pack_kernel, (unsigned)qt_cdiv(nbytes, 256), 256, 0, qt_s(stream), codes, count, bits, packed,
                                                                        nbytes, bad);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

extern "C" int qt_unpack_codes(const uint8_t *packed, int64_t count, int bits, uint8_t *codes,
                               qt_stream_t stream) {
    QT_REQUIRE(qt_bits_ok(bits) && count >= 0 && (count == 0 || (codes && packed)));
    if (count == 0) return QT_OK;
    launch_pdl(unpack_kernel, (unsigned)qt_cdiv(count, 256), 256, 0, qt_s(stream), packed, count, bits, codes);
    QT_CHECK_LAUNCH();
    return QT_OK;
}
