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
#include <climits>

#include "common.cuh"
#include "codec_ops.cuh"

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
                quant8<BITS>(a2v, quant_consts<BITS>(k.s1, k.scale, k.off), code, clipmask);
                if (split) {   // second half with the next channel's constants
                    uint32_t code_b[8], clip_b;
                    quant8<BITS>(a2v, quant_consts<BITS>(kb.s1, kb.scale, kb.off), code_b, clip_b);
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
// Per-channel constants of the quantize-pack stream kernel, staged in shared
// memory once per block (C <= kQuantTable): s1 = fl32(scale), cf = 2^(K-1) -
// offset, lim = 1/2 - marg (see quant8), and the offset for the exact path
// (INT_MIN: |offset| >= 2^20, the whole channel takes the exact path).
constexpr int kQuantTable = 1024;
struct QChan {
    float s1, cf, lim;
    int off;
};

template <int BITS>
__device__ __forceinline__ QChan qchan(float gamma, float beta) {
    const ChanCode cc = chan_code(gamma, beta, BITS);
    const QuantK k = quant_consts<BITS>(__double2float_rn(cc.scale), cc.scale, cc.off);
    return QChan{k.s1, k.cf, __fsub_rn(0.5f, k.marg), k.ok ? (int)cc.off : INT_MIN};
}

// Exact float64 recipe for 4 elements (rare: an element near a code
// boundary, non-finite, huge, or a channel with a huge offset).
template <int BITS>
__device__ __noinline__ uint32_t quant4_exact(float4 x, float gamma, float beta, uint32_t *nclip) {
    constexpr int top = (1 << BITS) - 1;
    const ChanCode cc = chan_code(gamma, beta, BITS);
    const float v[4] = {x.x, x.y, x.z, x.w};
    uint32_t w = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t raw = raw_code(v[j], cc.scale, cc.off, BITS);
        *nclip += (raw < 0 || raw > top) ? 1u : 0u;
        w |= (uint32_t)(raw < 0 ? 0 : (raw > top ? top : raw)) << (j * BITS);
    }
    return w;
}

// Codes of 4 consecutive A2 values of one channel (4K bits), quant8's error
// analysis with fewer instructions: the near-integer test as
// |frac - 1/2| >= 1/2 - marg, the clamp in float, the codes packed by exact
// float accumulation (sum fc_j 2^(jK) < 2^16 for K <= 4; two halves for K = 8).
// Sets `slow` when any element needs the exact recipe (the caller redoes all 4).
template <int BITS>
__device__ __forceinline__ uint32_t quant4(const float4 &x, const QChan &q, uint32_t &nclip,
                                           bool &slow) {
    constexpr float top = (float)((1 << BITS) - 1);
    const float v[4] = {x.x, x.y, x.z, x.w};
    float fc[4];
    bool sl = q.off == INT_MIN;
    uint32_t nc = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float y = __fmaf_rn(v[j], q.s1, q.cf);
        const float f = floorf(y);
        const float fr = __fsub_rn(y, f);
        // near an integer anywhere (also outside the code range: the exact
        // path is just as right there, and the test is one op cheaper)
        sl |= !(fabsf(y) < 1048576.f) | (fabsf(__fsub_rn(fr, 0.5f)) >= q.lim);
        fc[j] = fminf(fmaxf(f, 0.f), top);
        nc += (fc[j] != f) ? 1u : 0u;
    }
    uint32_t w;
    if (BITS == 8) {
        const float lo = __fmaf_rn(fc[1], 256.f, fc[0]), hi = __fmaf_rn(fc[3], 256.f, fc[2]);
        w = (uint32_t)(__float_as_int(__fadd_rn(lo, 8388608.f)) - 0x4B000000) |
            ((uint32_t)(__float_as_int(__fadd_rn(hi, 8388608.f)) - 0x4B000000) << 16);
    } else {
        constexpr float r = (float)(1 << BITS);
        const float acc = __fmaf_rn(__fmaf_rn(__fmaf_rn(fc[3], r, fc[2]), r, fc[1]), r, fc[0]);
        w = (uint32_t)(__float_as_int(__fadd_rn(acc, 8388608.f)) - 0x4B000000);
    }
    if (!sl) nclip += nc;
    slow = sl;
    return w;
}

// Lane-interleaved streaming layout: a warp iteration covers 32 * kSlots
// consecutive float4; slot i of lane l is float4 32 i + l, so every load
// and store instruction of the warp is one contiguous run.  A float4 is half
// of an 8-element group (one channel: hw % 8 == 0); the 4K-bit code pieces of
// 8/K adjacent lanes are OR-combined with shuffles into one 32-bit word,
// which the first of them stores (K = 8: every lane stores its own word).
constexpr int kSlots = 8;       // dequantize: float4 slots per lane per iteration
constexpr int kQSlots = 4;      // quantize: 8-element groups per lane per iteration

template <int BITS>
__device__ __forceinline__ void store_code_piece(uint8_t *codes, int64_t f, uint32_t piece) {
    constexpr int lpw = BITS == 8 ? 1 : 8 / BITS;        // lanes per 32-bit word
    const int lane = threadIdx.x & 31;
    uint32_t w = piece << (((lane & (lpw - 1)) * 4 * BITS) & 31);
    if (lpw > 1) w |= __shfl_xor_sync(0xffffffffu, w, 1);
    if (lpw > 2) w |= __shfl_xor_sync(0xffffffffu, w, 2);
    if (lpw > 4) w |= __shfl_xor_sync(0xffffffffu, w, 4);
    if ((lane & (lpw - 1)) == 0)
        reinterpret_cast<uint32_t *>(codes)[(f * 4 * BITS) >> 5] = w;
}

template <int BITS, bool CLIP, bool TABLE>
__global__ void __launch_bounds__(kThreads, 3) quant_pack_stream(FwdArgs a) {
    pdl_enter();
    __shared__ QChan s_q[TABLE ? kQuantTable : 1];
    const int64_t tid = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    for (int64_t c = tid; c < a.c && a.step; c += (int64_t)gridDim.x * kThreads) {
        const ChanCode cc = chan_code(a.gamma[c], a.beta[c], BITS);
        a.step[c] = cc.step;
        a.offset[c] = cc.off;
    }
    if (TABLE) {
        for (int c = threadIdx.x; c < a.c; c += kThreads)
            s_q[c] = qchan<BITS>(__ldg(a.gamma + c), __ldg(a.beta + c));
        __syncthreads();
    }
    // group-per-lane slots: lane l of a warp takes groups base + 32 i + l
    // (i < kQSlots): its two float4 loads are adjacent (the pair of
    // instructions reads one contiguous 1 KiB run per warp, the second hits
    // L1), and its K-byte code piece is one store -- the warp's store is one
    // contiguous 32K-byte run, no shuffles
    const int lane = threadIdx.x & 31;
    const int64_t warp = tid >> 5, nwarps = ((int64_t)gridDim.x * kThreads) >> 5;
    const int64_t ngroups = a.numel >> 3;
    uint32_t nclip = 0;
    auto chan_of = [&](int64_t gg) {
        const uint32_t plane = fast_div((uint32_t)gg, a.hw8d);
        return plane - fast_div(plane, a.cd) * (uint32_t)a.c;
    };
    auto piece_of = [&](const float4 &x, const QChan &q, uint32_t ch) {
        bool slow;
        uint32_t p = quant4<BITS>(x, q, nclip, slow);
        if (slow) p = quant4_exact<BITS>(x, __ldg(a.gamma + ch), __ldg(a.beta + ch), &nclip);
        return p;
    };
    for (int64_t base = warp * (32 * kQSlots); base < ngroups; base += nwarps * (32 * kQSlots)) {
        float4 xq[2 * kQSlots];
#pragma unroll
        for (int i = 0; i < kQSlots; ++i) {
            const int64_t gg = base + 32 * i + lane;
            if (gg < ngroups) {
                const float4 *src = reinterpret_cast<const float4 *>(a.x) + 2 * gg;
                xq[2 * i] = __ldg(src);
                xq[2 * i + 1] = __ldg(src + 1);
            }
        }
#pragma unroll
        for (int i = 0; i < kQSlots; ++i) {
            const int64_t gg = base + 32 * i + lane;
            if (gg >= ngroups) break;
            const uint32_t ch = chan_of(gg);
            const QChan q = TABLE ? s_q[ch] : qchan<BITS>(__ldg(a.gamma + ch), __ldg(a.beta + ch));
            const uint32_t p0 = piece_of(xq[2 * i], q, ch), p1 = piece_of(xq[2 * i + 1], q, ch);
            uint8_t *dst = a.codes + gg * BITS;
            if (BITS == 8) {
                *reinterpret_cast<uint2 *>(dst) = make_uint2(p0, p1);
            } else {
                const uint32_t w = p0 | (p1 << (4 * BITS));
                if (BITS == 4) *reinterpret_cast<uint32_t *>(dst) = w;
                else if (BITS == 2) *reinterpret_cast<uint16_t *>(dst) = (uint16_t)w;
                else *dst = (uint8_t)w;
            }
        }
    }
    if (CLIP) {
        __shared__ unsigned long long s_clip[kThreads / 32];
        unsigned long long clip = warp_sum((unsigned long long)nclip);
        if ((threadIdx.x & 31) == 0) s_clip[threadIdx.x >> 5] = clip;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < kThreads / 32; ++w) t += s_clip[w];
            if (t) atomicAdd(a.clip_count, t);
        }
    }
}

// Blocks that are co-resident for `kern` (one wave of a grid-stride kernel).
template <typename K>
static int64_t resident_blocks(K kern) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kThreads, 0) != cudaSuccess || nb < 1)
        nb = 1;
    return (int64_t)nb * qt_sm_count();
}

// Unpack + dequantize (codec.dequantize, codec.py:146-156) as a streaming
// kernel: 8 codes -> 8 fp32 (two float4 stores) per group.
// The reference rounds step * z (z = code + 0.5 - 2^(K-1) + offset, exact)
// to float64 and then to float32.  step = 6 |gamma| 2^-K has at most 26
// significant bits (|gamma| a float32 >= 1e-8) and |z| < 2^20 at most 21,
// so step * z is exact in float64 and the reference value is simply
// fl32(step * z).  With step = sh + sl (sh = fl32(step), sl the <= 2-bit
// rest), sl * z is exact in fp32 and fma(sh, z, sl * z) rounds the exact
// product once: bit-identical, in four fp32 ops.  Channels that do not meet
// the conditions (floored gamma, |offset| >= 2^19) decode in float64.
struct DChan {
    float sh, sl, zc;   // zc = offset + 0.5 - 2^(K-1)
    int ok;
};

template <int BITS>
__device__ __forceinline__ DChan dec_consts(double st, int64_t of) {
    DChan d;
    d.sh = __double2float_rn(st);
    d.sl = __double2float_rn(st - (double)d.sh);
    // sh + sl == step, sl <= 3 significant bits within 2^-27 of sh: step spans
    // <= 30 bits, so step * z (|z| < 2^20) is exact in float64
    const bool exact = ((double)d.sh + (double)d.sl == st) &&
                       ((__float_as_uint(d.sl) & 0x1FFFFFu) == 0u) && isfinite(st) && st > 0.0 &&
                       (d.sl == 0.f || fabsf(d.sl) >= __fmul_rn(d.sh, 7.450580596923828e-09f));
    d.ok = exact && of > -(1ll << 19) && of < (1ll << 19);
    d.zc = d.ok ? (float)((double)of + (0.5 - (double)(1 << (BITS - 1)))) : 0.f;
    return d;
}

constexpr int kDecTable = 1024;

// 4 codes (4K bits) of one channel -> 4 fp32 values
template <int BITS, bool TABLE>
__device__ __forceinline__ float4 dequant4(const DecArgs &a, const DChan *s_d, uint32_t ch,
                                           uint32_t piece) {
    float v[4];
    const DChan d = TABLE ? s_d[ch] : dec_consts<BITS>(__ldg(a.step + ch), __ldg(a.offset + ch));
    if (d.ok) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            // 2^23 + code as float bits (one shift-and-or), then exact adds
            const float t = __uint_as_float(((piece >> (j * BITS)) & ((1u << BITS) - 1u)) | 0x4B000000u);
            const float z = __fadd_rn(__fsub_rn(t, 8388608.f), d.zc);   // code + zc, exact
            const float y = __fmaf_rn(d.sh, z, __fmul_rn(d.sl, z));
            v[j] = a.relu ? fmaxf(y, 0.f) : y;                   // y is never 0 or NaN
        }
    } else {
        const double st = __ldg(a.step + ch);
        const int64_t of = __ldg(a.offset + ch);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float dd = decode((piece >> (j * BITS)) & ((1u << BITS) - 1u), st, of, BITS);
            v[j] = a.relu ? relu_np(dd) : dd;
        }
    }
    return make_float4(v[0], v[1], v[2], v[3]);
}

// Lane-interleaved like quant_pack_stream: slot i of lane l is float4
// 32 i + l of the warp's 256-float4 run, so every store instruction writes
// one contiguous 512-byte run; a lane loads the 32-bit code word holding its
// 4 codes (shared with 8/K - 1 neighbours: one contiguous code run per warp).
template <int BITS, bool TABLE>
__global__ void __launch_bounds__(kThreads) dequant_stream(DecArgs a, FastDiv hw8d, FastDiv cd) {
    pdl_enter();
    __shared__ DChan s_d[TABLE ? kDecTable : 1];
    if (TABLE) {
        for (int c = threadIdx.x; c < a.c; c += kThreads)
            s_d[c] = dec_consts<BITS>(__ldg(a.step + c), __ldg(a.offset + c));
        __syncthreads();
    }
    // lane-interleaved float4 slots: every store instruction of the warp is
    // one contiguous 512-byte run (measured: 0.80 of HBM peak, against 0.52
    // with a group -- two adjacent float4 -- per lane)
    const int64_t tid = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const int64_t nf4 = (a.numel >> 7) << 5;
    const int lane = threadIdx.x & 31;
    const int64_t warp = tid >> 5, nwarps = ((int64_t)gridDim.x * kThreads) >> 5;
    auto chan_of = [&](int64_t gg) {
        const uint32_t plane = fast_div((uint32_t)gg, hw8d);
        return plane - fast_div(plane, cd) * (uint32_t)a.c;
    };
    constexpr int lpw = BITS == 8 ? 1 : 8 / BITS;
    const uint32_t *cw = reinterpret_cast<const uint32_t *>(a.codes);
    for (int64_t base = warp * (32 * kSlots); base < nf4; base += nwarps * (32 * kSlots)) {
        uint32_t word[kSlots];
#pragma unroll
        for (int i = 0; i < kSlots; ++i) {
            const int64_t f = base + 32 * i + lane;
            if (base + 32 * i < nf4) word[i] = __ldcs(cw + ((f * 4 * BITS) >> 5));
        }
#pragma unroll
        for (int i = 0; i < kSlots; ++i) {
            if (base + 32 * i >= nf4) break;
            const int64_t f = base + 32 * i + lane;
            const uint32_t piece = BITS == 8 ? word[i] : (word[i] >> (((lane & (lpw - 1)) * 4 * BITS) & 31));
            __stcs(reinterpret_cast<float4 *>(a.out) + f,
                   dequant4<BITS, TABLE>(a, s_d, chan_of(f >> 1), piece));
        }
    }
    const int64_t ngroups = a.numel >> 3;
    for (int64_t gg = (nf4 >> 1) + tid; gg < ngroups; gg += (int64_t)gridDim.x * kThreads) {
        const uint8_t *src = a.codes + gg * BITS;
        uint64_t w;
        if (BITS == 8) {
            const uint2 u = *reinterpret_cast<const uint2 *>(src);
            w = u.x | ((uint64_t)u.y << 32);
        } else if (BITS == 4) {
            w = *reinterpret_cast<const unsigned int *>(src);
        } else if (BITS == 2) {
            w = *reinterpret_cast<const unsigned short *>(src);
        } else {
            w = *src;
        }
        const uint32_t ch = chan_of(gg);
        float4 *dst = reinterpret_cast<float4 *>(a.out) + 2 * gg;
        dst[0] = dequant4<BITS, TABLE>(a, s_d, ch, (uint32_t)(w & ((1ull << (4 * BITS)) - 1)));
        dst[1] = dequant4<BITS, TABLE>(a, s_d, ch, (uint32_t)(w >> (4 * BITS)));
    }
}

// Fused K1 (approx tapes, hw % 8 == 0, C <= kQuantTable) in the
// lane-interleaved layout of dequant_stream: every x load and A3 store of a
// warp is one contiguous 512-byte run; the per-channel BN and code constants
// come from a shared table (one block prologue); the codes of a float4 go
// through quant4 and store_code_piece.  Bit-identical to bn_relu_quant_stream.
struct K1Chan {
    float m32, inv32, g, b;   // BN apply (layer.py:246-249)
    QChan q;                   // codes
};

template <int BITS, bool CLIP>
__global__ void __launch_bounds__(kThreads) bn_relu_quant_lanes(FwdArgs a) {
    pdl_enter();
    __shared__ K1Chan s_k[kQuantTable];
    for (int c = threadIdx.x; c < a.c; c += kThreads) {
        const BnConst k = a.consts[c];
        const QuantK qk = quant_consts<BITS>(k.s1, k.scale, k.off);
        s_k[c] = K1Chan{k.m32, k.inv32, k.g, k.b,
                        QChan{qk.s1, qk.cf, __fsub_rn(0.5f, qk.marg), qk.ok ? (int)k.off : INT_MIN}};
    }
    __syncthreads();
    const int64_t tid = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const int64_t nf4 = (a.numel >> 7) << 5;
    const int lane = threadIdx.x & 31;
    const int64_t warp = tid >> 5, nwarps = ((int64_t)gridDim.x * kThreads) >> 5;
    uint32_t nclip = 0;
    auto chan_of = [&](int64_t gg) {
        const uint32_t plane = fast_div((uint32_t)gg, a.hw8d);
        return plane - fast_div(plane, a.cd) * (uint32_t)a.c;
    };
    // BN apply + ReLU of one float4 (A3 out) and its 4K-bit code piece
    auto one = [&](const float4 &x, uint32_t ch, float4 &a3) {
        const K1Chan k = s_k[ch];
        const float xv[4] = {x.x, x.y, x.z, x.w};
        float a2[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float v = __fsub_rn(xv[j], k.m32);
            v = __fmul_rn(v, k.inv32);
            v = __fmul_rn(v, k.g);
            a2[j] = __fadd_rn(v, k.b);
        }
        a3 = make_float4(relu_np(a2[0]), relu_np(a2[1]), relu_np(a2[2]), relu_np(a2[3]));
        const float4 a24 = make_float4(a2[0], a2[1], a2[2], a2[3]);
        bool slow;
        uint32_t p = quant4<BITS>(a24, k.q, nclip, slow);
        if (slow) p = quant4_exact<BITS>(a24, __ldg(a.gamma + ch), __ldg(a.beta + ch), &nclip);
        return p;
    };
    constexpr int S = 4;
    for (int64_t base = warp * (32 * S); base < nf4; base += nwarps * (32 * S)) {
        float4 xq[S];
#pragma unroll
        for (int i = 0; i < S; ++i)
            if (base + 32 * i < nf4) xq[i] = __ldg(reinterpret_cast<const float4 *>(a.x) + base + 32 * i + lane);
#pragma unroll
        for (int i = 0; i < S; ++i) {
            if (base + 32 * i >= nf4) break;                 // warp-uniform
            const int64_t f = base + 32 * i + lane;
            float4 a3;
            const uint32_t piece = one(xq[i], chan_of(f >> 1), a3);
            reinterpret_cast<float4 *>(a.a3_out)[f] = a3;
            store_code_piece<BITS>(a.codes, f, piece);
        }
    }
    const int64_t ngroups = a.numel >> 3;
    for (int64_t gg = (nf4 >> 1) + tid; gg < ngroups; gg += (int64_t)gridDim.x * kThreads) {
        const float4 *src = reinterpret_cast<const float4 *>(a.x) + 2 * gg;
        const uint32_t ch = chan_of(gg);
        float4 a30, a31;
        const uint32_t p0 = one(src[0], ch, a30), p1 = one(src[1], ch, a31);
        reinterpret_cast<float4 *>(a.a3_out)[2 * gg] = a30;
        reinterpret_cast<float4 *>(a.a3_out)[2 * gg + 1] = a31;
        uint8_t *dst = a.codes + gg * BITS;
        if (BITS == 8) {
            *reinterpret_cast<uint2 *>(dst) = make_uint2(p0, p1);
        } else {
            const uint32_t w = p0 | (p1 << (4 * BITS));
            if (BITS == 4) *reinterpret_cast<uint32_t *>(dst) = w;
            else if (BITS == 2) *reinterpret_cast<uint16_t *>(dst) = (uint16_t)w;
            else *dst = (uint8_t)w;
        }
    }
    if (CLIP) {
        __shared__ unsigned long long s_clip[kThreads / 32];
        unsigned long long clip = warp_sum((unsigned long long)nclip);
        if ((threadIdx.x & 31) == 0) s_clip[threadIdx.x >> 5] = clip;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < kThreads / 32; ++w) t += s_clip[w];
            if (t) atomicAdd(a.clip_count, t);
        }
    }
}

// The lane-interleaved K1 pays a per-block table prologue: measured slower
// on the C2 step's <= 8.4 M-element layers (1.19 vs 1.05 ms/step), so it is
// used from QTAPE_K1_LANES elements up (default 2^24: ImageNet-sized layers).
static bool lanes_k1(int64_t numel) {
    static const int64_t v = qt_env_i64("QTAPE_K1_LANES", 1ll << 24);
    return v > 0 && numel >= v;
}

template <int BITS>
static void launch_stream(const FwdArgs &a, unsigned blocks, cudaStream_t s) {
    const bool clip = a.clip_count != nullptr;
    const bool h4 = (a.hw & 7) != 0;
    if (!h4 && a.mode != MODE_NAIVE && a.c <= kQuantTable && !a.a2_tape && lanes_k1(a.numel)) {
        const int64_t ngroups = a.numel >> 3;
        auto kern = clip ? bn_relu_quant_lanes<BITS, true> : bn_relu_quant_lanes<BITS, false>;
        const unsigned b = (unsigned)std::max<int64_t>(
            1, std::min<int64_t>(qt_cdiv(ngroups, 4 * kThreads), resident_blocks(kern)));
        launch_pdl(kern, b, kThreads, 0, s, a);
        return;
    }
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
        const bool clip = a.clip_count != nullptr;
        const bool table = a.c <= kQuantTable;
        // one wave of co-resident blocks, 4 groups per thread per iteration
#define QT_QK(B, C, T) quant_pack_stream<B, C, T>
#define QT_QL(B, C, T)                                                                        \
    launch_pdl(QT_QK(B, C, T),                                                                \
               (unsigned)std::max<int64_t>(1, std::min<int64_t>(qt_cdiv(ngroups, 4 * kThreads),     \
                                                                resident_blocks(QT_QK(B, C, T)))), \
               kThreads, 0, s, a)
#define QT_QP(B)                                                                              \
    (table ? (clip ? QT_QL(B, true, true) : QT_QL(B, false, true))                          \
           : (clip ? QT_QL(B, true, false) : QT_QL(B, false, false)))
        switch (a.bits) {
            case 1: QT_QP(1); break;
            case 2: QT_QP(2); break;
            case 4: QT_QP(4); break;
            case 8: QT_QP(8); break;
        }
#undef QT_QP
#undef QT_QL
#undef QT_QK
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
        const FastDiv hw8d = make_fastdiv((uint32_t)(hw >> 3)), cd = make_fastdiv((uint32_t)c);
        const bool table = c <= kDecTable;
        // one wave of co-resident blocks, 4 groups per thread per iteration
#define QT_DL(B, T)                                                                           \
    launch_pdl(dequant_stream<B, T>,                                                          \
               (unsigned)std::max<int64_t>(1, std::min<int64_t>(qt_cdiv(ngroups, 4 * kThreads),     \
                                                                resident_blocks(dequant_stream<B, T>))), \
               kThreads, 0, qt_s(stream), d, hw8d, cd)
#define QT_DQ(B) (table ? QT_DL(B, true) : QT_DL(B, false))
        switch (bits) {
            case 1: QT_DQ(1); break;
            case 2: QT_DQ(2); break;
            case 4: QT_DQ(4); break;
            case 8: QT_DQ(8); break;
        }
#undef QT_DQ
#undef QT_DL
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
