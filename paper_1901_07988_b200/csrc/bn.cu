// Batch-norm statistics, the BN/ReLU backward from the tape, reconstruction,
// global average pooling and the parameter-free shortcut kernels.
//
// Reductions are deterministic: a fixed element->thread->block partition,
// float64 partials, and a last-block-per-channel finalize that reads the
// partials in block order (no float atomics anywhere).
#include <algorithm>

#include "common.cuh"
#include "codec_ops.cuh"

namespace qt {

constexpr int kRThreads = 256;
constexpr int64_t kTargetPerBlock = 8192;
// Workspace layout of every reduction: [kCounterBytes of per-channel
// completion counters (always left at zero)][float64 partials].  Keeping the
// counters at a fixed offset lets differently-shaped launches share one
// grow-only buffer.
constexpr int64_t kMaxChannels = 65535;
constexpr int64_t kCounterBytes = 65536 * 4;

struct Part {
    int64_t planes_per_block;  // (n) planes one block reduces for a channel
    int64_t blocks;            // blocks per channel
};

static Part partition(int64_t n, int64_t c, int64_t hw) {
    // blocks of ~kTargetPerBlock elements (every load of a thread in flight
    // at once); large layers get several waves of blocks, small ones one
    // block per channel
    (void)c;
    Part p;
    p.planes_per_block = std::max<int64_t>(1, qt_red_target() / hw);
    // at least ~2 blocks per SM: a small layer's single pass is one load
    // round per block, so spread it rather than lengthen it
    p.planes_per_block = std::min<int64_t>(p.planes_per_block,
                                           std::max<int64_t>(1, n * c / qt_red_div()));
    if (p.planes_per_block > n) p.planes_per_block = n;
    p.blocks = qt_cdiv(n, p.planes_per_block);
    return p;
}

// Clustered BN statistics: at most kStatsCluster blocks per channel (one
// cluster), each a contiguous run of planes.
constexpr int64_t kStatsCluster = 8;
static Part stats_partition(int64_t n, int64_t c, int64_t hw) {
    Part p = partition(n, c, hw);
    // balanced runs: the launch lasts as long as its longest block
    const int64_t nb = std::min<int64_t>(p.blocks, qt_red_cluster());
    p.planes_per_block = qt_cdiv(n, nb);
    p.blocks = qt_cdiv(n, p.planes_per_block);
    return p;
}

// Block-wide deterministic sum of NV doubles; result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double (*smem)[kRThreads / 32]) {
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = warp_sum(v[j]);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) smem[j][w] = v[j];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            double t = 0.0;
            for (int q = 0; q < kRThreads / 32; ++q) t += smem[j][q];
            v[j] = t;
        }
    }
}

// Returns true in thread 0 of the last block to finish channel `ch`.
__device__ __forceinline__ bool last_block(unsigned *counter, unsigned nblocks) {
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned prev = atomicAdd(counter, 1u);
        s_last = (prev == nblocks - 1);
        if (s_last) *counter = 0;  // re-arm for the next launch / graph replay
    }
    __syncthreads();
    return s_last;
}

// ------------------------------------------------------------- BN stats ---

struct StatsArgs {
    const float *x;
    int64_t n, c, hw;
    int64_t ppb, nb;
    double *mean, *var, *rmean, *rvar;
    double *part;       // [c][nb][2]
    unsigned *counter;  // [c]
    // optional fused preparation of the layer's forward (qt_bn_stats_prep)
    const float *gamma, *beta;
    int bits;
    double eps;
    BnConst *consts;
    float *gcopy, *bcopy;
    double *step;
    int64_t *offset;
    int64_t *clip;
    FastDiv hw8d;       // hw / 8 (vectorized stats loop)
    FastDiv hw4d;       // hw / 4 (4-pixel groups, hw % 8 == 4)
    FastDiv hwd;        // hw (scalar loop of odd planes, e.g. 7x7)
};

__global__ void __launch_bounds__(kRThreads) bn_stats_kernel(StatsArgs a) {
    pdl_enter();
    __shared__ double red[2][kRThreads / 32];
    const int64_t ch = blockIdx.y;
    const int64_t p0 = (int64_t)blockIdx.x * a.ppb;
    const int64_t p1 = min(p0 + a.ppb, a.n);
    // the finalizing thread loads the channel's parameters and evaluates its
    // code constants now, under the main loop's loads
    const bool fin = blockIdx.x == 0 && threadIdx.x == 0;
    float pg = 0.f, pb = 0.f;
    double prm = 0.0, prv = 0.0;
    ChanCode pcc{};
    if (fin) {
        if (a.rmean) { prm = a.rmean[ch]; prv = a.rvar[ch]; }
        if (a.consts) {
            pg = a.gamma[ch];
            pb = a.beta[ch];
            if (a.bits) pcc = chan_code(pg, pb, a.bits);
        }
    }
    const double shift = (double)a.x[ch * a.hw];  // x[0, c, 0]: shifted sums
    double v[2] = {0.0, 0.0};
    const int64_t cnt = (p1 - p0) * a.hw;
    if ((a.hw & 7) == 0 && cnt / 8 < (1ll << 31)) {
        const uint32_t hw8 = (uint32_t)(a.hw >> 3), n8 = (uint32_t)(cnt / 8);
        constexpr int U = 4;   // groups in flight per thread
        for (uint32_t e0 = threadIdx.x; e0 < n8; e0 += U * kRThreads) {
          float4 qq[U], rr[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t e = e0 + u * kRThreads;
            if (e >= n8) break;
            const uint32_t pl = fast_div(e, a.hw8d), off = e - pl * hw8;
            const float4 *src = reinterpret_cast<const float4 *>(a.x + ((p0 + pl) * a.c + ch) * a.hw) + 2 * off;
            qq[u] = __ldg(src);
            rr[u] = __ldg(src + 1);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (e0 + u * kRThreads >= n8) break;
            const float4 q = qq[u], r = rr[u];
            double d0 = (double)q.x - shift, d1 = (double)q.y - shift;
            double d2 = (double)q.z - shift, d3 = (double)q.w - shift;
            double d4 = (double)r.x - shift, d5 = (double)r.y - shift;
            double d6 = (double)r.z - shift, d7 = (double)r.w - shift;
            v[0] += ((d0 + d1) + (d2 + d3)) + ((d4 + d5) + (d6 + d7));
            v[1] += ((d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3)) +
                    ((d4 * d4 + d5 * d5) + (d6 * d6 + d7 * d7));
          }
        }
    } else if ((a.hw & 3) == 0 && cnt / 4 < (1ll << 31)) {
        // same per-thread order as one group per iteration; U loads in flight
        const uint32_t hw4 = (uint32_t)(a.hw >> 2), n4 = (uint32_t)(cnt / 4);
        constexpr int U = 4;
        for (uint32_t e0 = threadIdx.x; e0 < n4; e0 += U * kRThreads) {
            float4 qq[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t e = e0 + u * kRThreads;
                if (e >= n4) break;
                const uint32_t pl = fast_div(e, a.hw4d), off = e - pl * hw4;
                qq[u] = __ldg(reinterpret_cast<const float4 *>(a.x + ((p0 + pl) * a.c + ch) * a.hw) + off);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (e0 + u * kRThreads >= n4) break;
                const float4 q = qq[u];
                double d0 = (double)q.x - shift, d1 = (double)q.y - shift;
                double d2 = (double)q.z - shift, d3 = (double)q.w - shift;
                v[0] += (d0 + d1) + (d2 + d3);
                v[1] += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
            }
        }
    } else if (cnt < (1ll << 31) && a.hw < (1ll << 31)) {
        // odd planes (7x7): the same per-thread order as the loop below,
        // FastDiv indexing and U loads in flight
        const uint32_t hw = (uint32_t)a.hw, n1 = (uint32_t)cnt;
        constexpr int U = 4;
        for (uint32_t e0 = threadIdx.x; e0 < n1; e0 += U * kRThreads) {
            float xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t e = e0 + u * kRThreads;
                if (e >= n1) break;
                const uint32_t pl = fast_div(e, a.hwd), off = e - pl * hw;
                xv[u] = __ldg(a.x + ((p0 + pl) * a.c + ch) * a.hw + off);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (e0 + u * kRThreads >= n1) break;
                const double d = (double)xv[u] - shift;
                v[0] += d;
                v[1] += d * d;
            }
        }
    } else {
        for (int64_t e = threadIdx.x; e < cnt; e += kRThreads) {
            int64_t pl = e / a.hw, off = e - pl * a.hw;
            double d = (double)a.x[((p0 + pl) * a.c + ch) * a.hw + off] - shift;
            v[0] += d;
            v[1] += d * d;
        }
    }
    // the nb blocks of channel ch form one cluster: each publishes its block
    // sum in shared memory, rank 0 adds them in rank order (no global
    // partials, fence or counter)
    __shared__ double s_part[2];
    block_sum<2>(v, red);
    if (threadIdx.x == 0) {
        s_part[0] = v[0];
        s_part[1] = v[1];
    }
    cluster_sync_all();
    double s1 = 0.0, s2 = 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (unsigned r = 0; r < (unsigned)a.nb; ++r) {
            s1 += ld_dsmem_f64(&s_part[0], r);
            s2 += ld_dsmem_f64(&s_part[1], r);
        }
    }
    cluster_sync_all();   // remote CTAs keep their shared memory until read
    if (fin) {
        const double cntd = (double)(a.n * a.hw);
        const double dm = s1 / cntd;
        double var = (s2 - s1 * dm) / cntd;
        if (!(var > 0.0)) var = var != var ? var : 0.0;
        const double mean = shift + dm;
        a.mean[ch] = mean;
        a.var[ch] = var;
        if (a.rmean) {  // layer.py:237-241
            const double m = 0.9;
            a.rmean[ch] = __dadd_rn(__dmul_rn(prm, m), __dmul_rn(1.0 - m, mean));
            a.rvar[ch] = __dadd_rn(__dmul_rn(prv, m), __dmul_rn(1.0 - m, var));
        }
        if (a.consts) {  // per-channel constants of the fused forward (K1)
            const BnConst k = bn_const_cc(mean, var, a.eps, pg, pb, a.bits, pcc);
            a.consts[ch] = k;
            a.gcopy[ch] = pg;          // frozen tape copies (layer.py:253-255)
            a.bcopy[ch] = pb;
            if (a.bits) {
                a.step[ch] = k.step;
                a.offset[ch] = k.off;
            }
            if (ch == 0 && a.clip) *a.clip = 0;
        }
    }
}

// ------------------------------------------- fused BN forward (K0 + K1) ---
// qt_bn_stats_prep + qt_bn_relu_forward in ONE launch (layer.py:236-264):
// the nb blocks of a channel form one thread-block cluster (as
// bn_stats_kernel: the same partition, per-thread order and rank-ordered
// DSMEM combination, so mean / var are bit-identical to the two-launch
// path); every block then derives the channel's constants itself from the
// rank sums and applies BN -> tape -> ReLU to its own planes, from the copy
// of x it staged in shared memory during the statistics pass when it fits
// (x is read once), else from global memory.  hw % 8 == 0.  512 threads per
// block (the statistics kernel's 256 left the apply pass of narrow layers
// with too few threads: 2.18 vs 1.96 ms/step for the two launches on C2),
// so the moments are not bit-identical to bn_stats_kernel's (float64 sums in
// another order; tolerance-equal, and the codes are checked against the
// oracle on each layer's own input, tests/test_parity_gpu.py).
struct BnFwdArgs {
    const float *x;
    int64_t n, c, hw;
    int64_t ppb, nb;
    double *mean, *var, *rmean, *rvar;
    const float *gamma, *beta;
    int bits, mode;
    double eps;
    BnConst *consts;
    float *gcopy, *bcopy;
    double *step;
    int64_t *offset;
    unsigned long long *clip;   // accumulated (zeroed by the caller)
    float *a3, *a2;
    uint8_t *codes;
    FastDiv hw8d;
    int stage;                  // 1: the block's planes are staged in shared memory
};

__device__ __forceinline__ float relu_keep(float v) { return (v >= 0.f || v != v) ? v : 0.f; }

constexpr int kFThreads = 256;

template <int BITS, int MODE, bool A2OUT>
__global__ void __launch_bounds__(kFThreads) bn_fwd_kernel(BnFwdArgs a) {
    pdl_enter();
    __shared__ double red[2][kFThreads / 32];
    __shared__ double s_part[2];
    __shared__ BnConst s_k;
    __shared__ unsigned long long s_clip[kFThreads / 32];
    extern __shared__ float4 s_x[];
    const int64_t ch = blockIdx.y;
    const int64_t p0 = (int64_t)blockIdx.x * a.ppb;
    const int64_t p1 = min(p0 + a.ppb, a.n);
    float pg = 0.f, pb = 0.f;
    double prm = 0.0, prv = 0.0;
    ChanCode pcc{};
    if (threadIdx.x == 0) {   // under the main loop's loads
        pg = a.gamma[ch];
        pb = a.beta[ch];
        if (BITS != 0) pcc = chan_code(pg, pb, BITS);
        if (a.rmean && blockIdx.x == 0) { prm = a.rmean[ch]; prv = a.rvar[ch]; }
    }
    const double shift = (double)a.x[ch * a.hw];  // x[0, c, 0]: shifted sums
    double v[2] = {0.0, 0.0};
    const int64_t cnt = (p1 - p0) * a.hw;
    const uint32_t hw8 = (uint32_t)(a.hw >> 3), n8 = (uint32_t)(cnt / 8);
    constexpr int U = 4;   // groups in flight per thread (bn_stats_kernel's order)
    for (uint32_t e0 = threadIdx.x; e0 < n8; e0 += U * kFThreads) {
        float4 qq[U], rr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t e = e0 + u * kFThreads;
            if (e >= n8) break;
            const uint32_t pl = fast_div(e, a.hw8d), off = e - pl * hw8;
            const float4 *src = reinterpret_cast<const float4 *>(a.x + ((p0 + pl) * a.c + ch) * a.hw) + 2 * off;
            qq[u] = __ldg(src);
            rr[u] = __ldg(src + 1);
            if (a.stage) {
                s_x[2 * e] = qq[u];
                s_x[2 * e + 1] = rr[u];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (e0 + u * kFThreads >= n8) break;
            const float4 q = qq[u], r = rr[u];
            double d0 = (double)q.x - shift, d1 = (double)q.y - shift;
            double d2 = (double)q.z - shift, d3 = (double)q.w - shift;
            double d4 = (double)r.x - shift, d5 = (double)r.y - shift;
            double d6 = (double)r.z - shift, d7 = (double)r.w - shift;
            v[0] += ((d0 + d1) + (d2 + d3)) + ((d4 + d5) + (d6 + d7));
            v[1] += ((d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3)) +
                    ((d4 * d4 + d5 * d5) + (d6 * d6 + d7 * d7));
        }
    }
    {   // block-wide deterministic sum (warp trees, warps in order)
#pragma unroll
        for (int j = 0; j < 2; ++j) v[j] = warp_sum(v[j]);
        if ((threadIdx.x & 31) == 0) {
            red[0][threadIdx.x >> 5] = v[0];
            red[1][threadIdx.x >> 5] = v[1];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double t0 = 0.0, t1 = 0.0;
            for (int q = 0; q < kFThreads / 32; ++q) { t0 += red[0][q]; t1 += red[1][q]; }
            v[0] = t0;
            v[1] = t1;
        }
    }
    if (threadIdx.x == 0) {
        s_part[0] = v[0];
        s_part[1] = v[1];
    }
    cluster_sync_all();
    if (threadIdx.x == 0) {   // every block: the channel's moments, rank order
        double s1 = 0.0, s2 = 0.0;
        for (unsigned r = 0; r < (unsigned)a.nb; ++r) {
            s1 += ld_dsmem_f64(&s_part[0], r);
            s2 += ld_dsmem_f64(&s_part[1], r);
        }
        const double cntd = (double)(a.n * a.hw);
        const double dm = s1 / cntd;
        double var = (s2 - s1 * dm) / cntd;
        if (!(var > 0.0)) var = var != var ? var : 0.0;
        const double mean = shift + dm;
        const BnConst k = bn_const_cc(mean, var, a.eps, pg, pb, BITS, pcc);
        s_k = k;
        if (blockIdx.x == 0) {   // the tape / running-stat outputs, once per channel
            a.mean[ch] = mean;
            a.var[ch] = var;
            if (a.rmean) {  // layer.py:237-241
                const double m = 0.9;
                a.rmean[ch] = __dadd_rn(__dmul_rn(prm, m), __dmul_rn(1.0 - m, mean));
                a.rvar[ch] = __dadd_rn(__dmul_rn(prv, m), __dmul_rn(1.0 - m, var));
            }
            a.consts[ch] = k;
            a.gcopy[ch] = pg;          // frozen tape copies (layer.py:253-255)
            a.bcopy[ch] = pb;
            if (BITS) {
                a.step[ch] = k.step;
                a.offset[ch] = k.off;
            }
        }
    }
    cluster_sync_all();   // remote CTAs keep their shared memory until read; s_k visible
    const BnConst k = s_k;
    const QuantK qk = quant_consts<(BITS ? BITS : 1)>(k.s1, k.scale, k.off);
    unsigned long long clip = 0;
    for (uint32_t e = threadIdx.x; e < n8; e += kFThreads) {
        const uint32_t pl = fast_div(e, a.hw8d), off = e - pl * hw8;
        const int64_t i0 = ((p0 + pl) * a.c + ch) * a.hw + 8 * (int64_t)off;
        float4 q, r;
        if (a.stage) {
            q = s_x[2 * e];
            r = s_x[2 * e + 1];
        } else {
            q = __ldg(reinterpret_cast<const float4 *>(a.x + i0));
            r = __ldg(reinterpret_cast<const float4 *>(a.x + i0) + 1);
        }
        const float xv[8] = {q.x, q.y, q.z, q.w, r.x, r.y, r.z, r.w};
        float a2v[8], a3v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float t = __fsub_rn(xv[j], k.m32);      // layer.py:246-249
            t = __fmul_rn(t, k.inv32);
            t = __fmul_rn(t, k.g);
            a2v[j] = __fadd_rn(t, k.b);
        }
        if constexpr (BITS != 0) {
            uint32_t code[8], clipmask;
            quant8<BITS>(a2v, qk, code, clipmask);
            clip += __popc(clipmask);
            uint8_t *dst = a.codes + (i0 >> 3) * BITS;
            if (BITS == 8) {
                *reinterpret_cast<uint2 *>(dst) =
                    make_uint2(code[0] | (code[1] << 8) | (code[2] << 16) | (code[3] << 24),
                               code[4] | (code[5] << 8) | (code[6] << 16) | (code[7] << 24));
            } else {
                uint32_t w = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) w |= code[j] << (j * BITS);
                if (BITS == 4) *reinterpret_cast<uint32_t *>(dst) = w;
                else if (BITS == 2) *reinterpret_cast<uint16_t *>(dst) = (uint16_t)w;
                else *dst = (uint8_t)w;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
                a3v[j] = relu_keep(MODE == 2 ? decode(code[j], k.step, k.off, BITS) : a2v[j]);
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) a3v[j] = relu_keep(a2v[j]);
        }
        float4 *d3 = reinterpret_cast<float4 *>(a.a3 + i0);
        d3[0] = make_float4(a3v[0], a3v[1], a3v[2], a3v[3]);
        d3[1] = make_float4(a3v[4], a3v[5], a3v[6], a3v[7]);
        if (A2OUT) {
            float4 *d2 = reinterpret_cast<float4 *>(a.a2 + i0);
            d2[0] = make_float4(a2v[0], a2v[1], a2v[2], a2v[3]);
            d2[1] = make_float4(a2v[4], a2v[5], a2v[6], a2v[7]);
        }
    }
    if (BITS && a.clip) {
        clip = warp_sum(clip);
        if ((threadIdx.x & 31) == 0) s_clip[threadIdx.x >> 5] = clip;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < kFThreads / 32; ++w) t += s_clip[w];
            if (t) atomicAdd(a.clip, t);
        }
    }
}

// Plain per-channel float64 sum (ops.channel_sum, ops.py:199-201).
__global__ void __launch_bounds__(kRThreads) chan_sum_kernel(StatsArgs a) {
    pdl_enter();
    __shared__ double red[1][kRThreads / 32];
    const int64_t ch = blockIdx.y;
    const int64_t p0 = (int64_t)blockIdx.x * a.ppb;
    const int64_t p1 = min(p0 + a.ppb, a.n);
    double v[1] = {0.0};
    const int64_t cnt = (p1 - p0) * a.hw;
    for (int64_t e = threadIdx.x; e < cnt; e += kRThreads) {
        int64_t pl = e / a.hw, off = e - pl * a.hw;
        v[0] += (double)a.x[((p0 + pl) * a.c + ch) * a.hw + off];
    }
    block_sum<1>(v, red);
    if (threadIdx.x == 0) a.part[ch * a.nb + blockIdx.x] = v[0];
    if (!last_block(a.counter + ch, (unsigned)a.nb)) return;
    __threadfence();
    double fin[1] = {0.0};
    for (int64_t b = threadIdx.x; b < a.nb; b += kRThreads) fin[0] += __ldcg(a.part + ch * a.nb + b);
    block_sum<1>(fin, red);
    if (threadIdx.x == 0) a.mean[ch] = fin[0];
}

// ------------------------------------------------------- reconstruct ---

__global__ void reconstruct_kernel(qt_tape_t t, int64_t numel, int64_t c, int64_t hw,
                                   const float *gamma, const float *beta, float *a1, float *a2,
                                   float *a3) {
    pdl_enter();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < numel;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int ch = (int)((i / hw) % c);
        float v = tape_value(t, i, ch);
        if (a2) a2[i] = v;
        if (a3) a3[i] = (v >= 0.f || isnan(v)) ? v : 0.f;
        if (a1) a1[i] = __fdiv_rn(__fsub_rn(v, beta[ch]), safe_gamma(gamma[ch]));
    }
}

// -------------------------------------------------------------- GAP ---

__global__ void gap_kernel(const float *x, int64_t planes, int64_t hw, float *out) {
    pdl_enter();
    const int64_t pl = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (pl >= planes) return;
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    for (int64_t e = lane; e < hw; e += 32) s += (double)x[pl * hw + e];
    s = warp_sum(s);
    if (lane == 0) out[pl] = __double2float_rn(s / (double)hw);
}

__global__ void gap_bwd_kernel(const float *g, int64_t planes, int64_t hw, float *out) {
    pdl_enter();
    const int64_t numel = planes * hw;
    const float fhw = (float)hw;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < numel;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = __fdiv_rn(g[i / hw], fhw);
}

// --------------------------------------------------------- shortcut ---

__global__ void copy_kernel(const float4 *src, float4 *dst, int64_t n4) {
    pdl_enter();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

__global__ void copy1_kernel(const float *src, float *dst, int64_t n) {
    pdl_enter();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

// cur (N,C,H,W) += res (N,CR,H*sr,W*sr) on channels < CR (engine.py:262-269)
__global__ void shortcut_add_kernel(float *cur, const float *res, int64_t n, int64_t c, int64_t h,
                                    int64_t w, int64_t cr, int64_t sr) {
    pdl_enter();
    const int64_t numel = n * c * h * w;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < numel;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t x = i % w, t = i / w;
        int64_t y = t % h;
        t /= h;
        int64_t ch = t % c, nn = t / c;
        if (ch >= cr) continue;
        float r = res[((nn * cr + ch) * (h * sr) + y * sr) * (w * sr) + x * sr];
        cur[i] = __fadd_rn(cur[i], r);
    }
}

// g_in (N,C,H,W)[:, :, ::s, ::s] += g_res (N,CRES,H/s,W/s)[:, :C] (engine.py:272-279)
__global__ void shortcut_adj_kernel(float *g_in, const float *g_res, int64_t n, int64_t c,
                                    int64_t h, int64_t w, int64_t cres, int64_t sr) {
    pdl_enter();
    const int64_t hr = h / sr, wr = w / sr;
    const int64_t numel = n * c * hr * wr;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < numel;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t x = i % wr, t = i / wr;
        int64_t y = t % hr;
        t /= hr;
        int64_t ch = t % c, nn = t / c;
        float *d = g_in + ((nn * c + ch) * h + y * sr) * w + x * sr;
        *d = __fadd_rn(*d, g_res[((nn * cres + ch) * hr + y) * wr + x]);
    }
}

static unsigned grid_for(int64_t n, int threads) {
    int64_t b = qt_cdiv(n, threads);
    if (b > qt_sm_count() * 64) b = qt_sm_count() * 64;
    return (unsigned)std::max<int64_t>(b, 1);
}

}  // namespace qt

using namespace qt;

extern "C" int64_t qt_bn_stats_workspace(int64_t n, int64_t c, int64_t hw) {
    Part p = partition(n, c, hw);
    return kCounterBytes + c * p.blocks * 2 * (int64_t)sizeof(double);
}

extern "C" int qt_bn_stats(const float *x, int64_t n, int64_t c, int64_t hw, double *mean,
                           double *var, double *running_mean, double *running_var, void *ws,
                           qt_stream_t stream) {
    QT_REQUIRE(x && mean && var && ws && n > 0 && c > 0 && hw > 0 && c <= kMaxChannels);
    QT_REQUIRE((running_mean == nullptr) == (running_var == nullptr));
    Part p = stats_partition(n, c, hw);
    StatsArgs a{x, n, c, hw, p.planes_per_block, p.blocks, mean, var, running_mean, running_var,
                (double *)((char *)ws + kCounterBytes), (unsigned *)ws,
                nullptr, nullptr, 0, 0.0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    a.hw8d = make_fastdiv((uint32_t)std::max<int64_t>(1, hw >> 3));
    a.hw4d = make_fastdiv((uint32_t)std::max<int64_t>(1, hw >> 2));
    a.hwd = make_fastdiv((uint32_t)std::max<int64_t>(1, std::min<int64_t>(hw, INT32_MAX)));
    dim3 grid((unsigned)p.blocks, (unsigned)c);
    launch_pdl_cluster(bn_stats_kernel, grid, kRThreads, 0, qt_s(stream), (unsigned)p.blocks, a);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

extern "C" int qt_bn_stats_prep(const float *x, int64_t n, int64_t c, int64_t hw, double eps,
                                const float *gamma, const float *beta, int bits, double *mean,
                                double *var, double *running_mean, double *running_var,
                                float *gamma_copy, float *beta_copy, double *step, int64_t *offset,
                                int64_t *clip_count, void *consts, void *ws, qt_stream_t stream) {
    QT_REQUIRE(x && mean && var && ws && consts && gamma && beta && gamma_copy && beta_copy);
    QT_REQUIRE(n > 0 && c > 0 && hw > 0 && c <= kMaxChannels);
    QT_REQUIRE(bits == 0 || (qt_bits_ok(bits) && step && offset));
    QT_REQUIRE((running_mean == nullptr) == (running_var == nullptr));
    Part p = stats_partition(n, c, hw);
    StatsArgs a{x, n, c, hw, p.planes_per_block, p.blocks, mean, var, running_mean, running_var,
                (double *)((char *)ws + kCounterBytes), (unsigned *)ws,
                gamma, beta, bits, eps, (BnConst *)consts, gamma_copy, beta_copy, step, offset,
                clip_count};
    a.hw8d = make_fastdiv((uint32_t)std::max<int64_t>(1, hw >> 3));
    a.hw4d = make_fastdiv((uint32_t)std::max<int64_t>(1, hw >> 2));
    a.hwd = make_fastdiv((uint32_t)std::max<int64_t>(1, std::min<int64_t>(hw, INT32_MAX)));
    dim3 grid((unsigned)p.blocks, (unsigned)c);
    launch_pdl_cluster(bn_stats_kernel, grid, kRThreads, 0, qt_s(stream), (unsigned)p.blocks, a);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

// 1 if qt_bn_forward_fused takes this shape (else: qt_bn_stats_prep +
// qt_bn_relu_forward)
extern "C" int qt_bn_forward_fused_ok(int64_t n, int64_t c, int64_t hw) {
    return (n > 0 && c > 0 && c <= kMaxChannels && hw % 8 == 0 && n * hw / 8 < (1ll << 31) &&
            n * c * hw < (1ll << 40)) ? 1 : 0;
}

extern "C" int qt_bn_forward_fused(const float *x, int64_t n, int64_t c, int64_t hw, double eps,
                                   const float *gamma, const float *beta, int mode, int bits,
                                   double *mean, double *var, double *running_mean,
                                   double *running_var, float *gamma_copy, float *beta_copy,
                                   double *step, int64_t *offset, int64_t *clip_count,
                                   void *consts, float *a3_out, float *a2_tape, uint8_t *codes,
                                   qt_stream_t stream) {
    QT_REQUIRE(x && mean && var && consts && gamma && beta && gamma_copy && beta_copy && a3_out);
    QT_REQUIRE(mode >= 0 && mode <= 2 && (bits == 0 || qt_bits_ok(bits)));
    QT_REQUIRE(bits == 0 || (step && offset && codes));
    QT_REQUIRE((running_mean == nullptr) == (running_var == nullptr));
    if (!qt_bn_forward_fused_ok(n, c, hw)) return QT_EUNSUPPORTED;
    if ((((uintptr_t)x) | ((uintptr_t)a3_out) | ((uintptr_t)a2_tape)) & 15) return QT_EUNSUPPORTED;
    Part p = stats_partition(n, c, hw);
    BnFwdArgs a{};
    a.x = x; a.n = n; a.c = c; a.hw = hw; a.ppb = p.planes_per_block; a.nb = p.blocks;
    a.mean = mean; a.var = var; a.rmean = running_mean; a.rvar = running_var;
    a.gamma = gamma; a.beta = beta; a.bits = bits; a.mode = mode; a.eps = eps;
    a.consts = (BnConst *)consts; a.gcopy = gamma_copy;
    a.bcopy = beta_copy; a.step = step; a.offset = offset;
    a.clip = (unsigned long long *)clip_count;
    a.a3 = a3_out; a.a2 = a2_tape; a.codes = codes;
    a.hw8d = make_fastdiv((uint32_t)(hw >> 3));
    // stage the block's planes in shared memory when they fit (x read once)
    const int64_t bytes = p.planes_per_block * hw * 4;
    static const int64_t cap = qt_env_i64("QTAPE_BN_STAGE_BYTES", 64 * 1024);
    a.stage = bytes <= cap ? 1 : 0;
    const size_t smem = a.stage ? (size_t)bytes : 0;
    dim3 grid((unsigned)p.blocks, (unsigned)c);
    const cudaStream_t st = qt_s(stream);
#define QT_BF(B, M, A)                                                                        \
    do {                                                                                      \
        auto kern = bn_fwd_kernel<B, M, A>;                                                   \
        if (smem > 48 * 1024)                                                                 \
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        launch_pdl_cluster(kern, grid, kFThreads, smem, st, (unsigned)p.blocks, a);           \
    } while (0)
    const bool a2o = a2_tape != nullptr;
    switch (bits) {
        case 0: if (a2o) QT_BF(0, 0, true); else QT_BF(0, 0, false); break;
        case 1: if (mode == 2) QT_BF(1, 2, false); else QT_BF(1, 1, false); break;
        case 2: if (mode == 2) QT_BF(2, 2, false); else QT_BF(2, 1, false); break;
        case 4: if (mode == 2) QT_BF(4, 2, false); else QT_BF(4, 1, false); break;
        case 8: if (mode == 2) QT_BF(8, 2, false); else QT_BF(8, 1, false); break;
    }
#undef QT_BF
    QT_CHECK_LAUNCH();
    return QT_OK;
}

extern "C" int qt_channel_sum(const float *x, int64_t n, int64_t c, int64_t hw, double *out,
                              void *ws, qt_stream_t stream) {
    QT_REQUIRE(x && out && ws && n > 0 && c > 0 && hw > 0 && c <= kMaxChannels);
    Part p = partition(n, c, hw);
    StatsArgs a{x, n, c, hw, p.planes_per_block, p.blocks, out, nullptr, nullptr, nullptr,
                (double *)((char *)ws + kCounterBytes), (unsigned *)ws,
                nullptr, nullptr, 0, 0.0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    dim3 grid((unsigned)p.blocks, (unsigned)c);
    launch_pdl(chan_sum_kernel, grid, kRThreads, 0, qt_s(stream), a);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

extern "C" int qt_reconstruct(qt_tape_t tape, int64_t n, int64_t c, int64_t hw,
                              const float *gamma_tape, const float *beta_tape, float *a1,
                              float *a2, float *a3, qt_stream_t stream) {
    QT_REQUIRE(n > 0 && c > 0 && hw > 0 && gamma_tape && beta_tape);
    QT_REQUIRE(tape.a2 || (tape.codes && tape.step && tape.offset && qt_bits_ok(tape.bits)));
    int64_t numel = n * c * hw;
    launch_pdl(reconstruct_kernel, grid_for(numel, 256), 256, 0, qt_s(stream), tape, numel, c, hw, gamma_tape,
                                                                    beta_tape, a1, a2, a3);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

extern "C" int qt_gap(const float *x, int64_t n, int64_t c, int64_t hw, float *out,
                      qt_stream_t stream) {
    QT_REQUIRE(x && out && n > 0 && c > 0 && hw > 0);
    int64_t planes = n * c;
    launch_pdl(gap_kernel, (unsigned)qt_cdiv(planes, 8), 256, 0, qt_s(stream), x, planes, hw, out);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

extern "C" int qt_gap_backward(const float *g, int64_t n, int64_t c, int64_t hw, float *out,
                               qt_stream_t stream) {
    QT_REQUIRE(g && out && n > 0 && c > 0 && hw > 0);
    launch_pdl(gap_bwd_kernel, grid_for(n * c * hw, 256), 256, 0, qt_s(stream), g, n * c, hw, out);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

extern "C" int qt_copy(const float *src, float *dst, int64_t count, qt_stream_t stream) {
    QT_REQUIRE(count >= 0 && (count == 0 || (src && dst)));
    if (count == 0) return QT_OK;
    if ((count & 3) == 0 && (((uintptr_t)src | (uintptr_t)dst) & 15) == 0)
        launch_pdl(copy_kernel, grid_for(count / 4, 256), 256, 0, qt_s(stream), 
            (const float4 *)src, (float4 *)dst, count / 4);
    else
        launch_pdl(copy1_kernel, grid_for(count, 256), 256, 0, qt_s(stream), src, dst, count);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

extern "C" int qt_shortcut_add(float *cur, const float *res, int64_t n, int64_t c, int64_t h,
                               int64_t w, int64_t cr, int64_t sr, qt_stream_t stream) {
    QT_REQUIRE(cur && res && n > 0 && c > 0 && h > 0 && w > 0 && cr > 0 && cr <= c && sr >= 1);
    launch_pdl(shortcut_add_kernel, grid_for(n * c * h * w, 256), 256, 0, qt_s(stream), cur, res, n, c, h, w,
                                                                             cr, sr);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

extern "C" int qt_shortcut_adjoint(float *g_in, const float *g_res, int64_t n, int64_t c, int64_t h,
                                   int64_t w, int64_t cres, int64_t sr, qt_stream_t stream) {
    QT_REQUIRE(g_in && g_res && n > 0 && c > 0 && h > 0 && w > 0 && cres >= c && sr >= 1);
    QT_REQUIRE(h % sr == 0 && w % sr == 0);
    launch_pdl(shortcut_adj_kernel, grid_for(n * c * (h / sr) * (w / sr), 256), 256, 0, qt_s(stream), 
        g_in, g_res, n, c, h, w, cres, sr);
    QT_CHECK_LAUNCH();
    return QT_OK;
}
