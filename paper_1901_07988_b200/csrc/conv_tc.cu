// Convolution on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Forward (and stride-1 data gradient, as a forward conv of g_out with the
// transposed / flipped kernel) as an implicit GEMM over NCHW fp32:
//
//   D[m = output pixel][n = out channel] = sum_{(u,v), ci} A_uv[m][ci] * B[n][(u,v), ci]
//
// For every kernel tap (u,v) and channel chunk, TMA loads the SHIFTED input
// box straight from NCHW (tensor-map dims (w, c, h, n); negative / past-the-
// end coordinates are zero-filled by the TMA unit, which is the conv's zero
// padding) into shared memory in the UMMA MN-major swizzled layout
// (swizzle width = one image row: 32/64/128 B for rows of 8/16/32 px).
// The weights are pre-split once per call into (hi, lo) TF32 halves in a
// [co][(u,v) ci] K-major buffer and TMA-loaded the same way.
//
// Precision: 3xTF32 -- transform warps split each activation tile in place
// into hi (low 13 mantissa bits cleared) and lo = x - hi, and the MMA warp
// issues hi*hi + hi*lo + lo*hi, so products are accurate to ~2^-22 relative
// (fp32-level) while running on the tensor pipe.
//
// Warp roles (6 warps): w0 TMA producer, w1 TMEM owner + single-thread MMA
// issuer, w2..w5 split transform then epilogue (TMEM -> registers ->
// coalesced NCHW stores with the fused shortcut add).  S-stage mbarrier ring:
// full (TMA tx) -> ready (split done) -> empty (tcgen05.commit).
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "tc_common.cuh"

namespace qt {

using namespace tc;


template <int BN, int OWT, int KC, int KW>
struct FwdCfg {
    static constexpr int BM = 128;
    static constexpr int NM = KW * BN;                               // MMA N: (column tap, channel)
    static constexpr int A_BYTES = BM * KC * 4;                      // raw activation box
    static constexpr int B_BYTES = NM * KC * 4;                      // weights, one of (hi, lo)
    static constexpr int B_SLOT = (B_BYTES + 1023) / 1024 * 1024;    // keep every tile 1 KiB aligned
    static constexpr int RAW_BYTES = A_BYTES + 2 * B_SLOT;           // raw ring slot
    static constexpr int OUT_BYTES = BM * BN * 4;                    // output staging tile
    static constexpr int ACC_COLS = 2 * NM;                          // double-buffered accumulator
    static constexpr int OP_COLS = 2 * KC;                           // one A operand stage (hi, lo)
    static_assert(NM <= 256 && NM % 16 == 0, "UMMA N");
    static_assert(ACC_COLS + OP_COLS <= 512, "TMEM budget");
    static constexpr int A_SW = OWT * 4;     // swizzle bytes of the raw activation box
    static constexpr int K_SW = KC * 4;      // swizzle bytes of the weight tiles
};

struct FwdGeo {
    int n, ci, h, w, co, kh, kw, pad, oh, ow;
    int rows, nimg, tiles_per_img;  // tile = nimg images x rows x OW pixels
    int hw;                         // true pixels per plane (the activation map's extent)
    int flat;                       // 1x1 on any plane: 128-pixel runs of the flattened plane
    int mtiles, ntiles;             // output tiles along pixels / channels
    int R, NOUT;                    // raw ring and output staging depths
    int G;                          // split warpgroups (1, 2)
    int OPS;                        // operand ring depth in TMEM (a multiple of G, <= kFwdMaxOps)
    int wres;                       // 1: the CTA's weight tiles stay resident in smem
    int slot;                       // raw ring slot bytes (A box [+ B tiles])
    FastDiv ntd, tpid;              // / ntiles, / tiles_per_img (no runtime IDIV)
};

struct EpiParams {
    float *out;
    const float *res;
    int cr, sr;
    int res_tma;   // 1: shortcut tile TMA-loaded into the output staging buffer
};

// Layer fusion around the forward GEMM (qt_conv_forward_fused).
//
// Prologue (bits != 0): the activation boxes hold the layer's PRE-BN input x;
// the split warps form A3 = relu(((x - mean32) * inv32) * gamma + beta)
// (layer.py:245-249, 264: four rounded fp32 ops, no FMA) from the channel's
// BnConst and feed it to the MMA -- the rectified activation never exists in
// HBM -- and, on the centre-row stage of the CTA's first channel tile, emit
// the K-bit packed tape of A2 (codec.quantize, codec.py:107-143, bit-exact
// through code_fast) with the clip count.  Pixels outside the image (the
// conv's zero padding, the flat path's partial last run) are forced to 0
// after the BN apply, as the reference pads the rectified activation.
//
// Epilogue (stats != 0): the BN statistics of the OUTPUT (the next layer's
// input, after the fused shortcut add) -- the next layer's
// channel_moments (ops.py:186-196) + qt_bn_stats_prep outputs.  Every CTA
// owns one channel tile (grid % ntiles == 0); per output tile the epilogue
// warps take the tile mean and M2 of each channel from the staged tile (two
// passes, float64) and merge them into the CTA's running (n, mean, M2) in
// tile order (Chan et al.).  At the end each CTA publishes its (mean, M2) per
// channel and takes a ticket; the last `nfin` CTAs wait for the rest and
// finalize nfin disjoint channel ranges: mean = sum n_b mean_b / N,
// M2 = sum M2_b + n_b (mean_b - mean)^2 over the CTAs b of the channel's
// tile, in CTA order (deterministic), then var, running stats, BnConst,
// frozen gamma/beta, step/offset and the next tape's clip counter reset.
struct FuseParams {
    const BnConst *bn;             // [ci] constants of THIS layer (prologue)
    uint32_t *codes;               // packed K-bit tape, as 32-bit words
    unsigned long long *clip;      // clip counter of this layer's tape
    int bits;                      // 0: prologue off
    int stats;                     // 1: epilogue statistics of the output
    int nfin;                      // finalizer CTAs
    double *part;                  // [grid][BN] (mean, M2)
    double *pcnt;                  // [grid] pixel count per CTA
    unsigned *counter;             // [2] arrivals, finalizers done (left at 0)
    double eps;                    // next layer's BN: epsilon, gamma, beta, K
    const float *gamma, *beta;
    int nbits;
    double *mean, *var, *rmean, *rvar;
    BnConst *consts;
    float *gcopy, *bcopy;
    double *step;
    int64_t *offset;
    unsigned long long *nclip;
};

// w0 TMA, w1 TMEM + MMA, w2..w17 up to 4 split warpgroups, w18..w21 epilogue.
// Split group g owns operand stage g and every G-th (u, chunk) stage, so G
// stages are transformed concurrently and every mbarrier has one waiter
// group that consumes its phases in order (R is a multiple of G).
constexpr int kFwdGroups = 2;
// Operand (TMEM A) ring depth: up to kFwdMaxOps stages, a multiple of the
// split groups -- group g alternates over stages g, g + G, ... so it can
// transform stage gi while the MMAs of gi - G still read theirs
constexpr int kFwdMaxOps = 8;

// debug timeline (qt_debug_conv_trace): clock64 stamps of CTA trace_cta.
// Per stage gi < 64: [8*gi + 0] producer issue, +1 split raw_full ok, +2 split
// op_empty ok, +3 split done, +4 MMA op_full ok, +5 MMA committed;
// per tile lt < 32: [600 + 4*lt + 0] epi acc_full ok, +1 epi stored.
__device__ long long *g_cv_trace = nullptr;
__device__ int g_cv_trace_cta = 0;
#define CV_TRACE(idx)                  \
    do {                               \
        if (tr_) tr_[idx] = clock64(); \
    } while (0)
constexpr int kFwdEpiWarps = 8;   // two warps per TMEM lane quarter, alternate 16-channel blocks
constexpr int kFwdThreads = 64 + 128 * kFwdGroups + 32 * kFwdEpiWarps;
constexpr int kFwdEpiWarp = 2 + 4 * kFwdGroups;

// --- epilogue BN statistics (FuseParams.stats) ------------------------------
constexpr int kEpiThreads = 32 * kFwdEpiWarps;
constexpr int kFwdDualThreads = 64 + 128 + 32 * 4;   // DUAL form: 1 split group, 4 epilogue warps
constexpr int kFwdDualSmem = 113 * 1024;             // dynamic smem per CTA, two CTAs per SM

// One output tile's per-channel (mean, M2) from the staged tile
// s_out[img][BN][tpx] (valid pixels q < nvalid of the flattened 128), merged
// into the CTA's running (n, mean, M2) per channel (first: initialise).
// TPC = 256 / BN threads per channel (adjacent lanes); each sums a fixed,
// bank-rotated subset in float64, the group combines by a fixed xor tree.
template <int BN>
__device__ __forceinline__ void epi_tile_stats(const float *s_out, int tpx_log, int nvalid,
                                               bool nfirst, double *s_acc) {
    constexpr int TPC = kEpiThreads / BN;      // threads per channel (adjacent lanes)
    constexpr int PER4 = 32 / TPC;             // float4 chunks per thread (128 px / 4)
    const int tid = (int)threadIdx.x - 32 * kFwdEpiWarp;
    const int cc = tid / TPC, sub = tid % TPC;
    const int tmask = (1 << tpx_log) - 1;
    // one pass, float64, shifted by the channel's first value of the tile
    // (|mean - shift| ~ sigma: no cancellation in M2 = Q - S^2/n); chunk
    // r = sub + TPC * ((i + cc) mod PER4) keeps the float4 reads conflict-free
    const double sft = (double)s_out[cc << tpx_log];
    double S = 0.0, Q = 0.0;
#pragma unroll 4
    for (int i = 0; i < PER4; ++i) {
        const int q = 4 * (sub + TPC * ((i + cc) & (PER4 - 1)));
        if (q < nvalid) {
            const float4 v = *reinterpret_cast<const float4 *>(
                s_out + (((q >> tpx_log) * BN + cc) << tpx_log) + (q & tmask));
            const double d0 = (double)v.x - sft, d1 = (double)v.y - sft;
            const double d2 = (double)v.z - sft, d3 = (double)v.w - sft;
            S += (d0 + d1) + (d2 + d3);
            Q += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
        }
    }
#pragma unroll
    for (int o = TPC / 2; o > 0; o >>= 1) {
        S += __shfl_xor_sync(0xffffffffu, S, o);
        Q += __shfl_xor_sync(0xffffffffu, Q, o);
    }
    if (sub == 0) {   // re-centre on the CTA's shift (its first tile's) and accumulate
        const double n_t = (double)nvalid;
        double *a = s_acc + 3 * cc;
        if (nfirst) a[0] = sft;
        const double d = sft - a[0];
        a[1] += S + n_t * d;
        a[2] += Q + d * (2.0 * S + n_t * d);
    }
}

// Publish the CTA's per-channel shifted sums (shift, S, Q) and pixel count,
// take a ticket; the last nfin CTAs wait for the rest and finalize nfin
// disjoint channel ranges in ONE load round: every CTA's sums re-centred on
// the first CTA's shift s0 (S' = S + n d, Q' = Q + d (2 S + n d), d = s - s0),
// mean = s0 + sum S' / N, M2 = sum Q' - (sum S')^2 / N, in CTA order through
// a fixed warp tree (deterministic).
template <int BN>
__device__ __forceinline__ void epi_stats_finalize(const FuseParams &fz, const double *s_acc,
                                                   double cta_px, int *s_fin, int co, int ntiles) {
    const int tid = (int)threadIdx.x - 32 * kFwdEpiWarp;
    const int lane = tid & 31, w = tid >> 5;
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
    const int b = (int)blockIdx.x;
    for (int c = tid; c < BN; c += kEpiThreads) {
        double *dst = fz.part + ((size_t)b * BN + c) * 3;
        dst[0] = s_acc[3 * c + 0];
        dst[1] = s_acc[3 * c + 1];
        dst[2] = s_acc[3 * c + 2];
    }
    if (tid == 0) fz.pcnt[b] = cta_px;
    __threadfence();
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
    const int grid = (int)gridDim.x;
    if (tid == 0) {
        const unsigned t = atomicAdd(&fz.counter[0], 1u);
        const int f = (int)t - (grid - fz.nfin);
        if (f >= 0) {   // finalizer: wait for every CTA's partials
            while (*(volatile unsigned *)&fz.counter[0] < (unsigned)grid) {
            }
            __threadfence();
        }
        *s_fin = f;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
    const int f = *s_fin;
    if (f < 0) return;
    const int per = (co + fz.nfin - 1) / fz.nfin;
    const int cbeg = f * per, cend = min(co, cbeg + per);
    const int cpt = grid / ntiles;           // CTAs per channel tile
    for (int c = cbeg + w; c < cend; c += kFwdEpiWarps) {
        const int t = c / BN, cl = c - t * BN;
        double nb[5], sb[5], Sb[5], Qb[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) {          // every load of the lane in flight at once
            const int j = lane + 32 * k;
            const int bb = t + (j < cpt ? j : 0) * ntiles;
            const double *src = fz.part + ((size_t)bb * BN + cl) * 3;
            nb[k] = j < cpt ? __ldcg(fz.pcnt + bb) : 0.0;
            sb[k] = __ldcg(src);
            Sb[k] = __ldcg(src + 1);
            Qb[k] = __ldcg(src + 2);
        }
        const double s0 = __shfl_sync(0xffffffffu, sb[0], 0);
        double nn = 0.0, S = 0.0, Q = 0.0;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const double d = sb[k] - s0;
            if (nb[k] > 0.0) {
                nn += nb[k];
                S += Sb[k] + nb[k] * d;
                Q += Qb[k] + d * (2.0 * Sb[k] + nb[k] * d);
            }
        }
        for (int j = lane + 160; j < cpt; j += 32) {   // more than 160 CTAs per tile
            const int bb = t + j * ntiles;
            const double *src = fz.part + ((size_t)bb * BN + cl) * 3;
            const double cn = __ldcg(fz.pcnt + bb);
            const double d = __ldcg(src) - s0, Sj = __ldcg(src + 1);
            if (cn > 0.0) {
                nn += cn;
                S += Sj + cn * d;
                Q += __ldcg(src + 2) + d * (2.0 * Sj + cn * d);
            }
        }
        nn = warp_sum(nn);
        S = warp_sum(S);
        Q = warp_sum(Q);
        if (lane == 0) {
            const double mean = s0 + S / nn;
            double var = (Q - S * (S / nn)) / nn;
            if (!(var > 0.0)) var = var != var ? var : 0.0;
            fz.mean[c] = mean;
            fz.var[c] = var;
            if (fz.rmean) {   // layer.py:237-241
                const double m = 0.9;
                fz.rmean[c] = __dadd_rn(__dmul_rn(fz.rmean[c], m), __dmul_rn(1.0 - m, mean));
                fz.rvar[c] = __dadd_rn(__dmul_rn(fz.rvar[c], m), __dmul_rn(1.0 - m, var));
            }
            const float pg = fz.gamma[c], pb = fz.beta[c];
            const BnConst k = bn_const(mean, var, fz.eps, pg, pb, fz.nbits);
            fz.consts[c] = k;
            fz.gcopy[c] = pg;     // frozen tape copies (layer.py:253-255)
            fz.bcopy[c] = pb;
            if (fz.nbits) {
                fz.step[c] = k.step;
                fz.offset[c] = k.off;
            }
            if (c == 0 && fz.nclip) *fz.nclip = 0;
        }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
    if (tid == 0) {   // the last finalizer re-arms the counters for the next launch
        __threadfence();
        if (atomicAdd(&fz.counter[1], 1u) == (unsigned)fz.nfin - 1) {
            fz.counter[0] = 0;
            fz.counter[1] = 0;
        }
    }
}

// Persistent implicit-GEMM conv: each CTA walks output tiles (128 pixels x BN
// channels) with a grid-stride loop.
//
// Column taps as MMA columns: for kernel row u and a channel chunk the A
// operand is the UNSHIFTED input box (whole image rows shifted by u -- TMA
// handles the row offset and the zero rows); the B operand stacks the KW
// column taps, D[p][(v, co)] = sum_ci x[p][ci] W[co][ci][u][v], and the
// epilogue forms out[x] = D_0[x-1] + D_1[x] + D_2[x+1] with warp shuffles
// (a warp holds whole image rows, so neighbours are lanes +-1 and the zero
// padding is a lane mask).  This keeps N = KW*BN large and the MMA count per
// tile small (each tcgen05.mma costs ~46 cycles whatever N <= 64).
//   raw ring (TMA -> split / MMA): activation box + (hi, lo) weight tiles;
//            freed by the MMA commit.
//   A in TMEM (split -> MMA): each split thread owns one pixel = one TMEM lane
//            and writes its TF32 (hi, lo) halves with tcgen05.st.
//   TMEM acc x2 (MMA -> epilogue): tile j's epilogue (TMEM -> regs -> taps ->
//            + shortcut (TMA-prefetched) -> smem -> TMA store) overlaps tile
//            j+1's main loop.
// Precision: 3xTF32 (hi*hi + hi*lo + lo*hi).
// DUAL: two CTAs per SM (one split group, four epilogue warps, 256 TMEM
// columns each) for the small-N CIFAR layers, whose tiles are bound by fixed
// per-tile latencies (barrier round trips, epilogue hand-offs) rather than by
// the tensor pipe: the two CTAs' pipelines interleave on the SM.
template <int BN, int OWT, int KC, int KW, bool FUSE, bool DUAL = false>
__global__ void __launch_bounds__(DUAL ? 64 + 128 + 32 * 4 : kFwdThreads, DUAL ? 2 : 1)
    conv_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmA,
                       const __grid_constant__ CUtensorMap tmBh,
                       const __grid_constant__ CUtensorMap tmBl,
                       const __grid_constant__ CUtensorMap tmOut,
                       const __grid_constant__ CUtensorMap tmRes, FwdGeo g, EpiParams ep,
                       FuseParams fz) {
    using C = FwdCfg<BN, OWT, KC, KW>;
    static_assert(!(DUAL && FUSE), "fused prologue / epilogue: single-CTA form only");
    constexpr int NG = DUAL ? 1 : kFwdGroups;          // split warpgroups
    constexpr int NEPI = DUAL ? 4 : kFwdEpiWarps;      // epilogue warps
    constexpr int EPIW = 2 + 4 * NG;                   // first epilogue warp
    constexpr int TMEM_COLS = DUAL ? 256 : 512;
    const int R = g.R, NOUT = g.NOUT, G = g.G;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1 KiB alignment by pointer arithmetic on the __shared__ array (an
    // integer round trip would turn every access into a generic LD/ST)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *raw_base = smem;
    float *out_base = (float *)(raw_base + R * g.slot);
    // resident weights (wres): every stage's (hi, lo) tile, loaded once per CTA
    uint8_t *wres_base = (uint8_t *)out_base + NOUT * C::OUT_BYTES;
    uint64_t *bars = (uint64_t *)(wres_base + (g.wres ? g.kh * (g.ci / KC) * 2 * C::B_SLOT : 0));
    uint64_t *raw_full = bars, *raw_empty = bars + R;
    uint64_t *op_full = bars + 2 * R, *op_empty = op_full + kFwdMaxOps;
    uint64_t *acc_full = op_empty + kFwdMaxOps, *acc_empty = acc_full + 2;
    uint64_t *res_full = acc_empty + 2;
    uint64_t *w_full = res_full + 2;
    uint32_t *tmem_slot = (uint32_t *)(w_full + 1);
    // fusion scratch (16-byte aligned): the layer's BnConst table, the CTA's
    // running (n, mean, M2) per channel of its tile, the finalizer index
    // (pointer arithmetic from the shared base keeps every access LDS/STS)
    // (bars is 1 KiB aligned; this is the first 16-byte boundary past tmem_slot)
    uint8_t *fbase = (uint8_t *)(bars + 2 * R + 2 * kFwdMaxOps + 8);
    BnConst *s_bn = (BnConst *)fbase;
    double *s_acc = (double *)(fbase + (FUSE && fz.bits ? g.ci * (int)sizeof(BnConst) : 0));   // [BN][3]
    int *s_fin = (int *)(s_acc + (FUSE && fz.stats ? 3 * BN : 0));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    long long *const tr_ = (g_cv_trace && blockIdx.x == (unsigned)g_cv_trace_cta) ? g_cv_trace : nullptr;
    if (threadIdx.x == 0) CV_TRACE(1000);
    if (threadIdx.x == 0 && tr_) { tr_[990] = R; tr_[991] = G; tr_[992] = g.OPS; }
    const int kchunks = g.ci / KC;
    const int nst = g.kh * kchunks;             // (u, channel chunk) stages per tile
    const int total = g.mtiles * g.ntiles;

    if (threadIdx.x == 0) {
        for (int s = 0; s < R; ++s) { mbar_init(&raw_full[s], 1); mbar_init(&raw_empty[s], 1); }
        for (int s = 0; s < g.OPS; ++s) { mbar_init(&op_full[s], 128); mbar_init(&op_empty[s], 1); }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&acc_full[a], 1);
            mbar_init(&acc_empty[a], 32 * NEPI);
            mbar_init(&res_full[a], 1);
        }
        mbar_init(w_full, 1);
        fence_barrier_init();
    }
    if (FUSE && fz.stats && (int)threadIdx.x < 3 * BN) s_acc[threadIdx.x] = 0.0;
    if (warp == 1) tmem_alloc<TMEM_COLS>(tmem_slot);
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmBh);
        tma_prefetch(&tmBl);
        tma_prefetch(&tmOut);
        if (ep.res_tma) tma_prefetch(&tmRes);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // setup above touched only smem / TMEM / the tensor maps: overlap it with
    // the previous kernel, then wait for that kernel's results
    pdl_wait();
    pdl_trigger();

    auto tile_coords = [&](int T, int &n0, int &h0, int &co0) {
        const int mt = (int)fast_div((uint32_t)T, g.ntd);
        co0 = (T - mt * g.ntiles) * BN;
        const int im = (int)fast_div((uint32_t)mt, g.tpid);
        n0 = (g.nimg > 1) ? mt * g.nimg : im;
        h0 = (g.nimg > 1) ? 0 : (mt - im * g.tiles_per_img) * g.rows;
    };
    auto sRaw = [&](int s) { return raw_base + s * g.slot; };
    // B tiles of ring slot s / stage i: in the slot, or resident
    auto sBh = [&](int s, int i) {
        return g.wres ? wres_base + (2 * i) * C::B_SLOT : raw_base + s * g.slot + C::A_BYTES;
    };
    auto sBl = [&](int s, int i) {
        return g.wres ? wres_base + (2 * i + 1) * C::B_SLOT
                      : raw_base + s * g.slot + C::A_BYTES + C::B_SLOT;
    };
    auto a_col = [&](int o) { return (uint32_t)(C::ACC_COLS + o * C::OP_COLS); };

    if (warp == 0) {
        if (lane == 0) {  // ---------------------------------------- TMA producer
            if (g.wres && (int)blockIdx.x < total) {   // this CTA's co tile is fixed
                int n0, h0, co0;
                tile_coords(blockIdx.x, n0, h0, co0);
                mbar_expect_tx(w_full, nst * 2 * C::B_BYTES);
                for (int i = 0; i < nst; ++i) {
                    const int u = i / kchunks, c0 = (i % kchunks) * KC;
                    tma_load_3d(sBh(0, i), &tmBh, w_full, c0, co0, u * KW);
                    tma_load_3d(sBl(0, i), &tmBl, w_full, c0, co0, u * KW);
                }
            }
            int gi = 0, s = 0;
            uint32_t phe = 0;
            for (int T = blockIdx.x; T < total; T += gridDim.x) {
                int n0, h0, co0;
                tile_coords(T, n0, h0, co0);
                for (int i = 0, u = 0, c0 = 0; i < nst; ++i, ++gi) {
                    mbar_wait(&raw_empty[s], phe ^ 1u);
                    if (gi < 64) CV_TRACE(8 * gi);
                    mbar_expect_tx(&raw_full[s], C::A_BYTES + (g.wres ? 0 : 2 * C::B_BYTES));
                    // flattened (h*w) plane: the tile's rows shifted by u - pad are one
                    // contiguous pixel run (rows above / below the image are OOB -> 0)
                    tma_load_3d(sRaw(s), &tmA, &raw_full[s], (h0 + u - g.pad) * g.w, c0, n0);
                    if (!g.wres) {
                        tma_load_3d(sBh(s, i), &tmBh, &raw_full[s], c0, co0, u * KW);
                        tma_load_3d(sBl(s, i), &tmBl, &raw_full[s], c0, co0, u * KW);
                    }
                    if (++s == R) { s = 0; phe ^= 1u; }
                    c0 += KC;
                    if (c0 == g.ci) { c0 = 0; ++u; }
                }
            }
        }
    } else if (warp == 1) {  // ------------------ MMA issuer (whole warp, one lane issues)
        constexpr uint32_t idesc = instr_desc(128, C::NM, 2, 0, 0);  // A (TMEM) x B (K-major)
        constexpr uint32_t k_sbo = 8 * KC * 4;        // stride between 8-row groups
        constexpr uint32_t lay = swizzle_layout(C::K_SW);
        int s = 0, o = 0, lt = 0;
        uint32_t phs = 0, pho = 0;
        if (g.wres && (int)blockIdx.x < total) mbar_wait(w_full, 0);
        for (int T = blockIdx.x; T < total; T += gridDim.x, ++lt) {
            const int acc = lt & 1;
            mbar_wait(&acc_empty[acc], ((uint32_t)(lt >> 1) & 1u) ^ 1u);
            tc_fence_after();
            const uint32_t d = tmem + (uint32_t)(acc * C::NM);
            for (int i = 0; i < nst; ++i) {
                const int gi_ = lt * nst + i;
                if (lane == 0 && gi_ < 64) CV_TRACE(8 * gi_ + 6);
                mbar_wait(&op_full[o], pho);
                if (lane == 0 && gi_ < 64) CV_TRACE(8 * gi_ + 4);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t ah = tmem + a_col(o), al = ah + KC;
                    // descriptor = base + (byte offset >> 4) (tiles below 256 KiB)
                    const uint64_t dbh = smem_desc(smem_u32(sBh(s, i)), 16, k_sbo, lay);
                    const uint64_t dbl = smem_desc(smem_u32(sBl(s, i)), 16, k_sbo, lay);
#pragma unroll
                    for (int j = 0; j < KC / 8; ++j) {
                        mma_tf32_ts(d, ah + j * 8, dbh + j * 2, idesc, (i | j) ? 1u : 0u);
                        mma_tf32_ts(d, ah + j * 8, dbl + j * 2, idesc, 1u);
                        mma_tf32_ts(d, al + j * 8, dbh + j * 2, idesc, 1u);
                    }
                    mma_commit(&raw_empty[s]);
                    mma_commit(&op_empty[o]);
                    if (i == nst - 1) mma_commit(&acc_full[acc]);
                }
                __syncwarp();
                if (lane == 0 && gi_ < 64) CV_TRACE(8 * gi_ + 5);
                if (++s == R) { s = 0; phs ^= 1u; }
                if (++o == g.OPS) { o = 0; pho ^= 1u; }
            }
        }
    } else if (warp < EPIW) {  // ------------ split warpgroups -> TMEM (A operand)
        const int grp = (warp - 2) >> 2;
        const int quarter = warp & 3;
        const int row = 32 * quarter + lane;          // this thread's TMEM lane = pixel
        // raw A box: [img][channel][tile pixels of that image], unswizzled
        const uint32_t tpx = (uint32_t)(g.rows * OWT);
        const uint32_t aimg = (uint32_t)row / tpx, apx = (uint32_t)row % tpx;
        const uint32_t lane_base = tmem + ((uint32_t)(32 * quarter) << 16);
        // stages of this CTA: (its tiles) x nst, in MMA order
        const int my_tiles = (int)blockIdx.x < total ? (total - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
        const int nstages = my_tiles * nst;
        int gi = grp < G ? grp : nstages;
        int s = gi % R;
        int o = gi % g.OPS;                           // operand stage of stage gi
        uint32_t phr = (uint32_t)(gi / R) & 1u, pho = (uint32_t)(gi / g.OPS) & 1u;
        const int bits = FUSE ? fz.bits : 0;
        unsigned long long nclip = 0;
        if (bits) {   // the layer's BnConst table (written by the stats kernel / producer)
            const int st = threadIdx.x - 64;
            const float4 *src = reinterpret_cast<const float4 *>(fz.bn);
            float4 *dst = reinterpret_cast<float4 *>(s_bn);
            for (int q = st; q < g.ci * 3; q += 128 * NG) dst[q] = src[q];
            asm volatile("bar.sync 2, %0;" ::"n"(128 * NG) : "memory");
        }
        const int lpw_log = bits ? 5 - (bits == 1 ? 0 : bits == 2 ? 1 : bits == 4 ? 2 : 3) : 0;
        const int lpw = 1 << lpw_log;                      // lanes (pixels) per 32-bit code word
        for (; gi < nstages; gi += G) {
            mbar_wait(&raw_full[s], phr);
            if (quarter == 2 && lane == 0 && gi < 64) CV_TRACE(8 * gi + 1);
            mbar_wait(&op_empty[o], pho ^ 1u);
            if (quarter == 2 && lane == 0 && gi < 64) CV_TRACE(8 * gi + 2);
            tc_fence_after();
            const uint8_t *raw = sRaw(s);
            // stage -> (tile, kernel row u, channel chunk c0); pixel validity
            // (zero padding / partial flat run) and whether this stage emits
            // the tape (centre row of the CTA's first channel tile)
            int u = 0, c0 = 0, nimg0 = 0, pix = 0;
            bool valid = true, emit = false;
            if (bits) {
                const int lt_ = gi / nst, ist = gi - lt_ * nst;
                u = ist / kchunks;
                c0 = (ist - u * kchunks) * KC;
                int h0_, co0_;
                tile_coords((int)blockIdx.x + lt_ * (int)gridDim.x, nimg0, h0_, co0_);
                pix = (h0_ + u - g.pad) * g.w + (int)apx;
                valid = pix >= 0 && pix < g.hw;
                emit = (u == g.pad) && (co0_ == 0);
                nimg0 += (int)aimg;
            }
#pragma unroll
            for (int cg = 0; cg < KC; cg += 16) {
                uint32_t hi[16], lo[16];
                float a2[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const uint32_t off = ((aimg * KC + cg + j) * tpx + apx) * 4;
                    float x = *reinterpret_cast<const float *>(raw + off);
                    if (bits) {   // A3 = relu(BN(x)), 0 outside the image
                        const float4 k4 = *reinterpret_cast<const float4 *>(&s_bn[c0 + cg + j]);
                        float v = __fsub_rn(x, k4.x);           // layer.py:246-249
                        v = __fmul_rn(v, k4.y);
                        v = __fmul_rn(v, k4.z);
                        a2[j] = __fadd_rn(v, k4.w);
                        x = valid ? ((a2[j] >= 0.f || a2[j] != a2[j]) ? a2[j] : 0.f) : 0.f;
                    }
                    float h, l;
                    split_tf32(x, h, l);
                    hi[j] = __float_as_uint(h);
                    lo[j] = __float_as_uint(l);
                }
                tmem_st16(lane_base + a_col(o) + cg, hi);
                tmem_st16(lane_base + a_col(o) + KC + cg, lo);
                if (emit) {   // the K-bit tape of A2: lanes = consecutive pixels
                    // phase 1: 16 independent codes; phase 2: OR-reduce each
                    // over the lpw lanes of its word; phase 3: one lane stores
                    const int64_t ebase = ((int64_t)nimg0 * g.ci + c0 + cg) * g.hw + pix;
                    const uint32_t sh_l = (uint32_t)(bits * (lane & (lpw - 1)));
                    uint32_t wv[16];
                    uint32_t slowm = 0;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const BnConst &k = s_bn[c0 + cg + j];
                        bool cl, slow;
                        const uint32_t cj = code_fast_only(a2[j], k.s1, k.s2, k.off, bits, &cl, &slow);
                        slowm |= slow ? (1u << j) : 0u;
                        nclip += (valid && cl && !slow) ? 1u : 0u;
                        wv[j] = cj << sh_l;
                    }
                    if (slowm) {   // rare: exact float64 recipe (codec.py:118-120)
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            if (slowm & (1u << j)) {
                                const BnConst &k = s_bn[c0 + cg + j];
                                bool cl;
                                wv[j] = code_slow(a2[j], k.scale, k.off, bits, &cl) << sh_l;
                                nclip += (valid && cl) ? 1u : 0u;
                            }
                        }
                    }
#pragma unroll
                    for (int sh = 1; sh < 32; sh <<= 1) {
                        if (sh < lpw) {
#pragma unroll
                            for (int j = 0; j < 16; ++j) wv[j] |= __shfl_xor_sync(0xffffffffu, wv[j], sh);
                        }
                    }
                    if (valid && (lane & (lpw - 1)) == 0) {
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            __stcg(fz.codes + ((ebase + (int64_t)j * g.hw) >> lpw_log), wv[j]);
                    }
                }
            }
            tmem_wait_st();
            tc_fence_before();
            if (quarter == 2 && lane == 0 && gi < 64) CV_TRACE(8 * gi + 3);
            if (quarter == 0 && lane == 0 && gi < 64) CV_TRACE(8 * gi + 7);
            mbar_arrive(&op_full[o]);
            s += G;
            if (s >= R) { s -= R; phr ^= 1u; }    // R is a multiple of G
            o += G;
            if (o >= g.OPS) { o -= g.OPS; pho ^= 1u; }   // OPS is a multiple of G
        }
        if (bits) {   // clip count of the tape (codec.py:133-135), integer atomics
            nclip = warp_sum(nclip);
            if (lane == 0 && nclip) atomicAdd(fz.clip, nclip);
        }
    } else {  // ------------------------------------------------ epilogue warps
        const int quarter = warp & 3;
        const int ehalf = DUAL ? 0 : (warp - EPIW) >> 2;  // which alternate channel chunks
        const int row = 32 * quarter + lane;
        const int ratom = row / OWT, wcol = row % OWT;
        const int img = ratom / g.rows, rr = ratom % g.rows;
        const size_t cstride = (size_t)g.rows * OWT;
        const bool leader = (warp == EPIW && lane == 0);
        const bool res_ldg = ep.res && !ep.res_tma;
        const int kw_pad = (KW > 1) ? g.pad : 0;
        if (leader && ep.res_tma && (int)blockIdx.x < total) {  // prefetch the first shortcut tile
            int n0, h0, co0;
            tile_coords(blockIdx.x, n0, h0, co0);
            mbar_expect_tx(&res_full[0], C::OUT_BYTES);
            tma_load_4d(out_base, &tmRes, &res_full[0], g.flat ? h0 * OWT : 0, g.flat ? 0 : h0,
                        co0, n0);
        }
        int lt = 0;
        int cta_px = 0;      // pixels this CTA's tiles contributed (statistics epilogue)
        for (int T = blockIdx.x; T < total; T += gridDim.x, ++lt) {
            int n0, h0, co0;
            tile_coords(T, n0, h0, co0);
            const int acc = lt & 1, ob = (NOUT > 1) ? (lt & 1) : 0;
            float *s_out = out_base + (size_t)ob * (C::OUT_BYTES / 4);
            asm volatile("bar.sync 1, %0;" ::"n"(32 * NEPI) : "memory");   // staging free
            mbar_wait(&acc_full[acc], (uint32_t)(lt >> 1) & 1u);
            if (leader && lt < 32) CV_TRACE(600 + 4 * lt);
            tc_fence_after();
            if (ep.res_tma) mbar_wait(&res_full[ob], (uint32_t)((NOUT > 1 ? lt >> 1 : lt)) & 1u);
            const int nn = n0 + img, y = h0 + rr;
            const uint32_t tbase = tmem + ((uint32_t)(32 * quarter) << 16) + (uint32_t)(acc * C::NM);
            float *so = s_out + (img * BN * g.rows + rr) * OWT + wcol;
            const int64_t hr = (int64_t)g.oh * ep.sr, wr = (int64_t)g.ow * ep.sr;
            // channel chunks of CW dealt to the two warps of each lane quarter
            // (8-channel chunks when BN = 16, so both warps work)
            constexpr int CW = BN >= 32 ? 16 : 8;
#pragma unroll 1
            for (int cb = CW * ehalf; cb < BN; cb += (DUAL ? 1 : 2) * CW) {
                float rv[CW];
                if (res_ldg) {  // strided shortcut (sr > 1): gather, CW loads in flight
#pragma unroll
                    for (int j = 0; j < CW; ++j) {
                        const int co = co0 + cb + j;
                        rv[j] = co < ep.cr ? __ldg(ep.res + (((int64_t)nn * ep.cr + co) * hr +
                                                             (int64_t)y * ep.sr) * wr +
                                                    (int64_t)wcol * ep.sr)
                                           : 0.f;
                    }
                }
                uint32_t r[KW][CW];
                // per column tap: source lane and zero-padding mask (branch-free
                // so the CW channels' shuffle chains interleave)
                int src[KW];
                bool okt[KW];
#pragma unroll
                for (int t = 0; t < KW; ++t) {
                    const int dx = t - kw_pad;
                    src[t] = (lane + dx) & 31;
                    okt[t] = (wcol + dx >= 0) && (wcol + dx < OWT);
                }
#pragma unroll
                for (int v = 0; v < KW; ++v) {
                    if constexpr (CW == 16) tmem_ld16(tbase + v * BN + cb, r[v]);
                    else tmem_ld8(tbase + v * BN + cb, r[v]);
                }
                tmem_wait_ld();
                if (leader && lt < 32 && cb == 0) CV_TRACE(600 + 4 * lt + 2);
#pragma unroll
                for (int j = 0; j < CW; ++j) {
                    float v;
                    if (KW == 1) {
                        v = __uint_as_float(r[0][j]);
                    } else {
                        // out[x] = sum_v D_v[x + v - pad]  (zero outside the image row)
                        v = 0.f;
#pragma unroll
                        for (int t = 0; t < KW; ++t) {
                            const float nb = __shfl_sync(0xffffffffu, __uint_as_float(r[t][j]), src[t]);
                            v = __fadd_rn(v, okt[t] ? nb : 0.f);
                        }
                    }
                    float *dst = so + (cb + j) * (int)cstride;
                    // out = fp32(conv); cur += shortcut(res)  (engine.py:262-269)
                    if (ep.res_tma) {
                        if (co0 + cb + j < ep.cr) v = __fadd_rn(v, *dst);
                    } else if (res_ldg && co0 + cb + j < ep.cr) {
                        v = __fadd_rn(v, rv[j]);
                    }
                    *dst = v;
                }
            }
            if (leader && lt < 32) CV_TRACE(600 + 4 * lt + 3);
            tc_fence_before();
            mbar_arrive(&acc_empty[acc]);            // TMEM buffer free for tile lt+2
            fence_async_smem();
            asm volatile("bar.sync 1, %0;" ::"n"(32 * NEPI) : "memory");
            if (leader && lt < 32) CV_TRACE(600 + 4 * lt + 1);
            if (leader) {
                tma_store_4d(&tmOut, s_out, g.flat ? h0 * OWT : 0, g.flat ? 0 : h0, co0, n0);
                bulk_commit();
                // the next tile's staging buffer must have been read by its previous store;
                // then prefetch the next shortcut tile into it
                if (NOUT > 1) bulk_wait_read1(); else bulk_wait_read0();
                const int Tn = T + gridDim.x;
                if (ep.res_tma && Tn < total) {
                    int n1, h1, c1;
                    tile_coords(Tn, n1, h1, c1);
                    const int ob1 = (NOUT > 1) ? ((lt + 1) & 1) : 0;
                    mbar_expect_tx(&res_full[ob1], C::OUT_BYTES);
                    tma_load_4d(out_base + (size_t)ob1 * (C::OUT_BYTES / 4), &tmRes, &res_full[ob1],
                                g.flat ? h1 * OWT : 0, g.flat ? 0 : h1, c1, n1);
                }
            }
            if (FUSE && fz.stats) {   // BN statistics of this output tile (reads the staged tile)
                const int nvalid = g.flat ? min(128, g.hw - h0 * OWT) : 128;
                epi_tile_stats<BN>(s_out, cstride == 64 ? 6 : 7, nvalid, lt == 0, s_acc);
                cta_px += nvalid;
            }
        }
        if (leader) bulk_wait_read0();
        if (FUSE && fz.stats) epi_stats_finalize<BN>(fz, s_acc, (double)cta_px, s_fin, g.co, g.ntiles);
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) CV_TRACE(1001);
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<TMEM_COLS>(tmem);
    }
}

// Weight prep: B[co'][(u,v)*ci' + c] = hi/lo of W[co'][c][u][v] (forward) or of
// W[c][co'][kh-1-u][kw-1-v] (data gradient: transposed + flipped kernel).
__global__ void weight_prep_kernel(const float *w, int co_n, int ci_n, int kh, int kw, int flip,
                                   float *bhi, float *blo) {
    pdl_enter();
    // output rows co' (co_n of them), K' = kh*kw*ci_n
    const int kk = kh * kw;
    const int64_t total = (int64_t)co_n * kk * ci_n;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        // layout [uv][co'][ci'] (uv = u*kw + v): the TMA box (KC, BN, KW) at
        // (c0, co0, u*kw) is the stacked column-tap B tile of kernel row u
        const int c = (int)(idx % ci_n);
        const int o = (int)((idx / ci_n) % co_n);
        const int uv = (int)(idx / ((int64_t)ci_n * co_n));
        const int u = uv / kw, v = uv % kw;
        float x;
        if (!flip)
            x = w[(((int64_t)o * ci_n + c) * kh + u) * kw + v];
        else  // original W is [c][o][kh][kw] with c = original out channel
            x = w[(((int64_t)c * co_n + o) * kh + (kh - 1 - u)) * kw + (kw - 1 - v)];
        float hi, lo;
        split_tf32(x, hi, lo);
        bhi[idx] = hi;
        blo[idx] = lo;
    }
}

// Many layers' preparations in one launch: blockIdx.y selects the descriptor.
__global__ void weight_prep_batch_kernel(const qt_wprep_t *descs) {
    pdl_enter();
    const qt_wprep_t d = descs[blockIdx.y];
    const int kk = d.kh * d.kw;
    const int64_t total = (int64_t)d.rows * kk * d.cols;
    float *bhi = d.out, *blo = d.out + total;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(idx % d.cols);
        const int o = (int)((idx / d.cols) % d.rows);
        const int uv = (int)(idx / ((int64_t)d.cols * d.rows));
        const int u = uv / d.kw, v = uv % d.kw;
        float x;
        if (!d.flip)
            x = d.w[(((int64_t)o * d.cols + c) * d.kh + u) * d.kw + v];
        else
            x = d.w[(((int64_t)c * d.rows + o) * d.kh + (d.kh - 1 - u)) * d.kw + (d.kw - 1 - v)];
        float hi, lo;
        split_tf32(x, hi, lo);
        bhi[idx] = hi;
        blo[idx] = lo;
    }
}

// --------------------------------------------------------------- host side

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    });
    return fn;
}

static CUtensorMapSwizzle swz(int bytes) {
    return bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                        : (bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
}

// activations (n, c, h*w) as 3D (pixel, c, n), box = the tile's pixels of
// each image (rows*ow <= 128, one contiguous run per channel) x KC x nimg;
// no swizzle (the split warps read it pixel-per-lane, conflict-free), so
// a stage is KC*nimg TMA rows of up to 512 B instead of KC*rows 128-B rows
static bool make_map_act(CUtensorMap *m, const float *x, const FwdGeo &g, int owt, int kc) {
    auto enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)g.hw, (cuuint64_t)g.ci, (cuuint64_t)g.n};
    cuuint64_t strides[2] = {(cuuint64_t)g.hw * 4, (cuuint64_t)g.ci * g.hw * 4};
    cuuint32_t box[3] = {(cuuint32_t)(g.rows * owt), (cuuint32_t)kc, (cuuint32_t)g.nimg};
    cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void *)x, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// prepared weights [kh*kw][co][ci] as 3D (ci, co, uv); box = KC x BN x KW
static bool make_map_w(CUtensorMap *m, const float *b, int co, int ci, int kk, int bn, int kc,
                       int kw) {
    auto enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)ci, (cuuint64_t)co, (cuuint64_t)kk};
    cuuint64_t strides[2] = {(cuuint64_t)ci * 4, (cuuint64_t)co * ci * 4};
    cuuint32_t box[3] = {(cuuint32_t)kc, (cuuint32_t)bn, (cuuint32_t)kw};
    cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void *)b, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, swz(kc * 4), CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct Maps {
    CUtensorMap a, bh, bl, out, res;
};

static int num_sms() { return qt_sm_count(); }

// CTA cap of the current launch (0 = every SM); set per call by tc_conv_s1
static int s_cta_cap = 0;
static int dgrad_cta_cap() {
    static const int v = [] {
        const char *e = getenv("QTAPE_DGRAD_CTAS");
        return e && atoi(e) > 0 ? atoi(e) : 0;
    }();
    return v;
}

template <int BN, int OWT, int KC, int KW>
static int launch_fwd(const Maps &m, const FwdGeo &g, const EpiParams &ep, const FuseParams &fz,
                      int tiles, int ntiles, cudaStream_t st, bool allow_dual = true) {
    using C = FwdCfg<BN, OWT, KC, KW>;
    const bool fuse = fz.bits || fz.stats;
    const int total = tiles * ntiles;
    // two CTAs per SM (DUAL) for small-N layers with more tiles than SMs:
    // 256 TMEM columns and about half the shared memory each (QTAPE_FWD_DUAL=0: off)
    static const bool dual_on = [] {
        const char *e = getenv("QTAPE_FWD_DUAL");
        return !(e && *e == '0');
    }();
    // also under the concurrent-backward SM cap (the data gradient beside the
    // side-stream weight gradients): C2 dgrad 1.84 -> 1.60 ms/step
    static const bool dual_capped = [] {
        const char *e = getenv("QTAPE_FWD_DUAL_CAP");
        return !(e && *e == '0');
    }();
    // CIFAR-sized layers only: the ImageNet ones are closer to the tensor
    // bound and measured 1 % slower in pairs (C4 43.9 vs 44.3 ms/step)
    const double macs = (double)g.n * g.oh * g.ow * (double)g.co * g.ci * g.kh * g.kw;
    bool dual = allow_dual && dual_on && !fuse && macs < kSmallLayerMacs &&
                (s_cta_cap == 0 || dual_capped) && BN <= 64 &&
                total > (s_cta_cap > 0 ? s_cta_cap : num_sms()) && C::ACC_COLS + C::OP_COLS <= 256;
    auto kern = fuse ? conv_fwd_tc_kernel<BN, OWT, KC, KW, true>
                : dual ? conv_fwd_tc_kernel<BN, OWT, KC, KW, false, true>
                       : conv_fwd_tc_kernel<BN, OWT, KC, KW, false>;
    const int variant = fuse ? 1 : (dual ? 2 : 0);
    static bool attr[3] = {false, false, false};
    if (!attr[variant]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             dual ? kFwdDualSmem : 227 * 1024);
        attr[variant] = true;
    }
    FwdGeo gg = g;
    gg.mtiles = tiles;
    gg.ntiles = ntiles;
    const int tmem_cols = dual ? 256 : 512;
    // split groups G (operand ring depth) limited by TMEM; smem: output
    // staging x2 when it fits, raw ring a multiple of G (>= G, up to 8)
    int G = dual ? 1 : kFwdGroups;
    while (G > 1 && C::ACC_COLS + G * C::OP_COLS > tmem_cols) G /= 2;
    if (C::ACC_COLS + G * C::OP_COLS > tmem_cols) return QT_EUNSUPPORTED;
    // resident weights: every CTA keeps one co tile (grid a multiple of
    // ntiles) and its nst stages' (hi, lo) tiles fit next to the rings
    const int nst = g.kh * (g.ci / KC);
    const int wbytes = nst * 2 * C::B_SLOT;
    const int sms = (s_cta_cap > 0 ? std::min(num_sms(), s_cta_cap) : num_sms()) * (dual ? 2 : 1);
    int grid = std::min(total, sms);
    gg.wres = 0;
    if (ntiles <= sms && wbytes <= (dual ? 40 : 96) * 1024) {
        gg.wres = 1;
        grid = std::max(ntiles, std::min(total, sms) / ntiles * ntiles);
    }
    FuseParams fzl = fz;
    if (fz.stats) {   // every CTA keeps one channel tile: grid a multiple of ntiles
        if (ntiles > sms) return QT_EUNSUPPORTED;
        grid = std::max(ntiles, std::min(total, sms) / ntiles * ntiles);
        fzl.nfin = std::max(1, std::min(grid, g.co / 8));
    }
    const int fuse_bytes = 16 + (fz.bits ? g.ci * (int)sizeof(BnConst) : 0) +
                           (fz.stats ? 3 * BN * 8 : 0) + 16;
    gg.slot = gg.wres ? (C::A_BYTES + 1023) / 1024 * 1024 : C::RAW_BYTES;
    gg.ntd = make_fastdiv((uint32_t)ntiles);
    gg.tpid = make_fastdiv((uint32_t)std::max(1, g.tiles_per_img));
    const int budget = (dual ? kFwdDualSmem : 227 * 1024) - 1024 - 512 - fuse_bytes -
                       (gg.wres ? wbytes : 0);
    auto raw_fit = [&](int no) { return (budget - no * C::OUT_BYTES) / gg.slot; };
    int nout = 2;
    while (G > 1 && raw_fit(1) < G) G /= 2;
    if (raw_fit(nout) < G) nout = 1;
    int r = raw_fit(nout);
    if (r < G || r < 1) {
        if (dual)   // does not fit half an SM: the single-CTA form
            return launch_fwd<BN, OWT, KC, KW>(m, g, ep, fz, tiles, ntiles, st, false);
        return QT_EUNSUPPORTED;
    }
    r = std::min(r, 8) / G * G;
    gg.R = r;
    gg.NOUT = nout;
    gg.G = G;
    static const int ops_env = [] {
        const char *e = getenv("QTAPE_FWD_OPS");
        return e ? atoi(e) : 0;
    }();
    int ops = std::min(kFwdMaxOps, (tmem_cols - C::ACC_COLS) / C::OP_COLS) / G * G;
    if (ops_env > 0) ops = std::max(G, std::min(ops, ops_env / G * G));   // tuning
    gg.OPS = std::max(G, ops);
    const int smem = r * gg.slot + nout * C::OUT_BYTES + (gg.wres ? wbytes : 0) + 1024 + 512 +
                     fuse_bytes;
    launch_pdl(kern, grid, dual ? kFwdDualThreads : kFwdThreads, smem, st, m.a, m.bh, m.bl, m.out,
               m.res, gg, ep, fzl);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

template <int OWT, int KC, int KW>
static int dispatch_bn(int bn, const Maps &m, const FwdGeo &g, const EpiParams &ep,
                       const FuseParams &fz, int tiles, int ntiles, cudaStream_t st) {
    switch (bn) {
        case 16: return launch_fwd<16, OWT, KC, KW>(m, g, ep, fz, tiles, ntiles, st);
        case 32: return launch_fwd<32, OWT, KC, KW>(m, g, ep, fz, tiles, ntiles, st);
        case 64: return launch_fwd<64, OWT, KC, KW>(m, g, ep, fz, tiles, ntiles, st);
        case 128:
            if constexpr (KW == 1) return launch_fwd<128, OWT, KC, KW>(m, g, ep, fz, tiles, ntiles, st);
            return QT_EUNSUPPORTED;
        default: return QT_EUNSUPPORTED;
    }
}

template <int OWT>
static int dispatch_kc(int kc, int kw, int bn, const Maps &m, const FwdGeo &g,
                       const EpiParams &ep, const FuseParams &fz, int tiles, int ntiles,
                       cudaStream_t st) {
    if (kw == 1) {
        switch (kc) {
            case 16: return dispatch_bn<OWT, 16, 1>(bn, m, g, ep, fz, tiles, ntiles, st);
            case 32: return dispatch_bn<OWT, 32, 1>(bn, m, g, ep, fz, tiles, ntiles, st);
        }
    } else if (kw == 3) {
        if (kc == 16) return dispatch_bn<OWT, 16, 3>(bn, m, g, ep, fz, tiles, ntiles, st);
    }
    return QT_EUNSUPPORTED;
}

// (w, h, c, n) view of an NCHW fp32 tensor, box = one output tile of BN channels
static bool make_map_nchw(CUtensorMap *m, const float *t, int n, int c, int h, int w, int rows,
                          int bn, int nimg) {
    auto enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[4] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)c, (cuuint64_t)n};
    cuuint64_t strides[3] = {(cuuint64_t)w * 4, (cuuint64_t)h * w * 4, (cuuint64_t)c * h * w * 4};
    cuuint32_t box[4] = {(cuuint32_t)w, (cuuint32_t)rows, (cuuint32_t)bn, (cuuint32_t)nimg};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void *)t, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// (hw, 1, c, n) view of an NCHW fp32 tensor for the flattened 1x1 mode: box =
// 128 consecutive pixels of one plane x BN channels (the last run of a plane
// is partial: TMA zero-fills the load and clips the store)
static bool make_map_flat(CUtensorMap *m, const float *t, int n, int c, int hw, int bn) {
    auto enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[4] = {(cuuint64_t)hw, 1, (cuuint64_t)c, (cuuint64_t)n};
    cuuint64_t strides[3] = {(cuuint64_t)hw * 4, (cuuint64_t)hw * 4, (cuuint64_t)c * hw * 4};
    cuuint32_t box[4] = {128, 1, (cuuint32_t)bn, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void *)t, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Row-tiled form: output rows of 8/16/32 px, whole rows (or whole images) per
// 128-pixel tile.
static bool tc_rows_ok(int n, int ci, int h, int wd, int co, int kh, int kw, int pad) {
    const int oh = h + 2 * pad - kh + 1, ow = wd + 2 * pad - kw + 1;
    if (kw != 1 && kw != 3) return false;
    if (kw == 1 && pad != 0) return false;
    if (ow != 8 && ow != 16 && ow != 32) return false;
    if (ow != wd || ci % 16 || co % 16) return false;
    const int per = 128 / ow;
    if (oh >= per) return oh % per == 0;
    return per % oh == 0 && n % (per / oh) == 0;
}

// Flattened form: a 1x1 conv is a per-pixel GEMM, so any plane whose byte
// stride is a 16-byte multiple (TMA) tiles as 128-pixel runs
static bool tc_flat_ok(int ci, int h, int wd, int co, int kh, int kw, int pad) {
    if (kh != 1 || kw != 1 || pad != 0 || ci % 16 || co % 16) return false;
    const int64_t hw = (int64_t)h * wd;
    return hw % 4 == 0 && hw >= 16 && hw < (1 << 30);
}

// Shape predicate of the tensor-core path (also used by qt_conv_uses_tc).
static bool tc_shape_ok(int n, int ci, int h, int wd, int co, int kh, int kw, int pad) {
    return tc_rows_ok(n, ci, h, wd, co, kh, kw, pad) || tc_flat_ok(ci, h, wd, co, kh, kw, pad);
}

// Runs out = conv_s1(x, W') with W' the (possibly transposed+flipped) kernel.
// x: (n, ci, h, w); out: (n, co, oh, ow); weights w in the ORIGINAL layout.
static const FuseParams kNoFuse{};

static int tc_conv_s1(const float *x, const float *w, float *out, int n, int ci, int h, int wd,
                      int co, int kh, int kw, int pad, int flip, const float *res, int cr, int sr,
                      void *ws, cudaStream_t st, const FuseParams &fz = kNoFuse) {
    FwdGeo g{};
    {   // data gradient beside the side-stream weight gradients: half the SMs
        const double macs = (double)n * (h + 2 * pad - kh + 1) * (wd + 2 * pad - kw + 1) *
                            (double)co * ci * kh * kw;
        s_cta_cap = !flip ? 0
                    : dgrad_cta_cap() > 0 ? dgrad_cta_cap()
                    : (g_concurrent_bwd && macs < kSmallLayerMacs) ? num_sms() / 2 : 0;
    }
    g.n = n; g.ci = ci; g.h = h; g.w = wd; g.co = co; g.kh = kh; g.kw = kw; g.pad = pad;
    g.oh = h + 2 * pad - kh + 1;
    g.ow = wd + 2 * pad - kw + 1;
    g.hw = h * wd;
    if (tc_rows_ok(n, ci, h, wd, co, kh, kw, pad)) {
        const int per = 128 / g.ow;                     // rows per 128-pixel tile
        if (g.oh >= per) {
            g.rows = per; g.nimg = 1; g.tiles_per_img = g.oh / per;
        } else {
            g.rows = g.oh; g.nimg = per / g.oh; g.tiles_per_img = 1;
        }
    } else if (tc_flat_ok(ci, h, wd, co, kh, kw, pad)) {
        if (res && sr != 1) {   // strided shortcut: the conv, then the standalone add
            if (fz.stats) return QT_EUNSUPPORTED;    // statistics must see the sum
            int rc = tc_conv_s1(x, w, out, n, ci, h, wd, co, kh, kw, pad, flip, nullptr, 0, 1, ws, st, fz);
            if (rc) return rc;
            return qt_shortcut_add(out, res, n, co, h, wd, cr, sr, st);
        }
        // virtual rows of 32 px: tile t = pixels [128 t, 128 t + 128) of the plane
        g.flat = 1;
        g.w = g.ow = 32;
        g.h = g.oh = (g.hw + 31) / 32;
        g.rows = 4; g.nimg = 1; g.tiles_per_img = (g.hw + 127) / 128;
    } else {
        return QT_EUNSUPPORTED;
    }
    if (fz.bits && (flip || g.hw % (32 / fz.bits) != 0 || ci > 512)) return QT_EUNSUPPORTED;
    const int kc = (kw == 1 && ci % 32 == 0) ? 32 : 16;
    int bn = co <= 16 ? 16 : (co <= 32 ? 32 : (co <= 64 ? 64 : 128));
    if (kw == 3 && bn > 64) bn = 64;         // stacked taps: KW * BN <= 256 (UMMA N)
    while (co % bn) bn /= 2;                 // co % 16 == 0 (tc_shape_ok): 48, 80, 96, 160, 192 ...
    {   // split the channels further while there are fewer tiles than SMs
        const int mt = (n / g.nimg) * g.tiles_per_img;
        const int sm_target = s_cta_cap > 0 ? std::min(num_sms(), s_cta_cap) : num_sms();
        while (bn > 16 && (int64_t)mt * (co / bn) < sm_target && co % (bn / 2) == 0) bn /= 2;
    }
    const int kdim = kh * kw * ci;
    float *bhi = (float *)ws;
    float *blo = bhi + (int64_t)co * kdim;
    if (!ws) return QT_EINVAL;
    if (w) {   // w == NULL: ws already holds the prepared operand (qt_conv_prepare_weights)
        launch_pdl(weight_prep_kernel, (unsigned)std::min<int64_t>(qt_cdiv((int64_t)co * kdim, 256), 1024), 256, 0, st, w, co, ci, kh, kw, flip, bhi, blo);
        QT_CHECK_LAUNCH();
    }
    Maps mp;
    if (!make_map_act(&mp.a, x, g, g.ow, kc) ||
        !make_map_w(&mp.bh, bhi, co, ci, kh * kw, bn, kc, kw) ||
        !make_map_w(&mp.bl, blo, co, ci, kh * kw, bn, kc, kw) ||
        !(g.flat ? make_map_flat(&mp.out, out, n, co, g.hw, bn)
                 : make_map_nchw(&mp.out, out, n, co, g.oh, g.ow, g.rows, bn, g.nimg)))
        return QT_EUNSUPPORTED;
    EpiParams ep{out, res, cr, sr, 0};
    mp.res = mp.out;
    if (res && sr == 1) {  // same-resolution shortcut: one TMA box per tile (channels >= cr -> 0)
        if (!(g.flat ? make_map_flat(&mp.res, res, n, cr, g.hw, bn)
                     : make_map_nchw(&mp.res, res, n, cr, g.oh, g.ow, g.rows, bn, g.nimg)))
            return QT_EUNSUPPORTED;
        ep.res_tma = 1;
    }
    const int tiles = (n / g.nimg) * g.tiles_per_img;
    const int ntiles = co / bn;
    switch (g.ow) {
        case 8: return dispatch_kc<8>(kc, kw, bn, mp, g, ep, fz, tiles, ntiles, st);
        case 16: return dispatch_kc<16>(kc, kw, bn, mp, g, ep, fz, tiles, ntiles, st);
        case 32: return dispatch_kc<32>(kc, kw, bn, mp, g, ep, fz, tiles, ntiles, st);
    }
    return QT_EUNSUPPORTED;
}

}  // namespace qt

using namespace qt;

static bool tc_disabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("QTAPE_NO_TC");
        v = (e && *e && *e != '0') ? 1 : 0;
    }
    return v == 1;
}

extern "C" int qt_conv_uses_tc(int64_t n, int64_t ci, int64_t h, int64_t wd, int64_t co,
                               int64_t kh, int64_t kw, int64_t stride, int64_t pad, int dgrad) {
    if (tc_disabled() || stride != 1) return 0;
    if (!dgrad) return tc_shape_ok((int)n, (int)ci, (int)h, (int)wd, (int)co, (int)kh, (int)kw,
                                   (int)pad) ? 1 : 0;
    if (kh != kw || pad > kh - 1) return 0;
    const int64_t oh = h + 2 * pad - kh + 1, ow = wd + 2 * pad - kw + 1;
    return tc_shape_ok((int)n, (int)co, (int)oh, (int)ow, (int)ci, (int)kh, (int)kw,
                       (int)(kh - 1 - pad)) ? 1 : 0;
}

// debug hook (not part of the public ABI): buf = 1002 int64 stamps or NULL
extern "C" int qt_debug_conv_trace(void *buf, int cta) {
    long long *b = (long long *)buf;
    if (cudaMemcpyToSymbol(g_cv_trace, &b, sizeof(b)) != cudaSuccess) return QT_EINVAL;
    if (cudaMemcpyToSymbol(g_cv_trace_cta, &cta, sizeof(cta)) != cudaSuccess) return QT_EINVAL;
    return QT_OK;
}

extern "C" int qt_conv_prepare_weights(const qt_wprep_t *descs, int64_t count, int64_t max_elems,
                                       qt_stream_t stream) {
    QT_REQUIRE(descs && count >= 0 && count <= 65535 && max_elems >= 0);
    if (count == 0) return QT_OK;
    const unsigned bx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(qt_cdiv(max_elems, 256), 64));
    launch_pdl(weight_prep_batch_kernel, dim3(bx, (unsigned)count), 256, 0, qt_s(stream), descs);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

extern "C" int64_t qt_conv_workspace(int64_t ci, int64_t co, int64_t kh, int64_t kw) {
    return 2 * ci * co * kh * kw * (int64_t)sizeof(float) + 1024;
}

int qt_tc_conv_forward(const float *x, const float *w, float *out, const qt::ConvGeo &g,
                       const float *res, int64_t cr, int64_t sr, void *ws, cudaStream_t s) {
    if (tc_disabled() || g.s != 1 || !ws) return QT_EUNSUPPORTED;
    if (g.n > INT32_MAX || g.ci * g.h * g.w > INT32_MAX) return QT_EUNSUPPORTED;
    return tc_conv_s1(x, w, out, (int)g.n, (int)g.ci, (int)g.h, (int)g.w, (int)g.co, (int)g.kh,
                      (int)g.kw, (int)g.pad, 0, res, (int)cr, (int)sr, ws, s);
}

// data gradient of a stride-1 conv = forward conv of g_out with the
// transposed, flipped kernel and padding k-1-pad
int qt_tc_conv_dgrad(const float *gr, const float *w, float *gx, const qt::ConvGeo &g, void *ws,
                     cudaStream_t s) {
    if (tc_disabled() || g.s != 1 || !ws) return QT_EUNSUPPORTED;
    if (g.kh != g.kw || g.pad > g.kh - 1) return QT_EUNSUPPORTED;
    const int pad2 = (int)(g.kh - 1 - g.pad);
    return tc_conv_s1(gr, w, gx, (int)g.n, (int)g.co, (int)g.oh, (int)g.ow, (int)g.ci, (int)g.kh,
                      (int)g.kw, pad2, 1, nullptr, 0, 1, ws, s);
}

// ---------------------------------------------------------------------------
// Non-overlapping convs (kernel == stride, no padding: the 2x2/s2 transition
// convs of SURVEY.md Appendix C) are 1x1 convs of the space-to-depth input:
//   x'[n][(c*s + u)*s + v][y][x] = x[n][c][y*s + u][x*s + v]
// with the kernel viewed as (co, ci*s*s) -- the same memory.  Forward: s2d
// into the workspace, then the tensor-core 1x1 path; data gradient: the 1x1
// data gradient into the workspace, then depth-to-space.
namespace qt {

template <bool TO_DEPTH>
__global__ void space_depth_kernel(const float *src, float *dst, int64_t n, int64_t c, int64_t h,
                                   int64_t w, int s) {
    pdl_enter();
    // iterate over the full-resolution tensor in memory order (coalesced side)
    const int64_t total = n * c * h * w;
    const int64_t hs = h / s, ws = w / s;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t xx = i % w, t1 = i / w, yy = t1 % h, t2 = t1 / h, cc = t2 % c, nn = t2 / c;
        const int64_t u = yy % s, v = xx % s;
        const int64_t j = (((nn * c + cc) * s + u) * s + v) * hs * ws + (yy / s) * ws + xx / s;
        if (TO_DEPTH)
            dst[j] = src[i];
        else
            dst[i] = src[j];
    }
}

// s == 2 with w % 4 == 0: a thread moves a 2-row x 4-column patch -- two
// float4 on the full-resolution side, four float2 (one per (u, v) plane) on
// the depth side; 32-bit indices through FastDiv
template <bool TO_DEPTH>
__global__ void space_depth2_kernel(const float *src, float *dst, uint32_t total, uint32_t h,
                                    uint32_t w, FastDiv qd, FastDiv yd) {
    pdl_enter();
    const uint32_t w4 = w >> 2, h2 = h >> 1, w2 = w >> 1, plane2 = h2 * w2;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const uint32_t r = fast_div(t, qd), q = t - r * w4;       // r = plane * h2 + Y
        const uint32_t pl = fast_div(r, yd), Y = r - pl * h2;
        const size_t full = ((size_t)pl * h + 2 * Y) * w + 4 * q;
        const size_t dep = (size_t)pl * 4 * plane2 + (size_t)Y * w2 + 2 * q;
        float4 *f0 = const_cast<float4 *>(reinterpret_cast<const float4 *>((TO_DEPTH ? src : dst) + full));
        float4 *f1 = const_cast<float4 *>(reinterpret_cast<const float4 *>((TO_DEPTH ? src : dst) + full + w));
        float2 *d = const_cast<float2 *>(reinterpret_cast<const float2 *>((TO_DEPTH ? dst : src) + dep));
        if (TO_DEPTH) {
            const float4 a = __ldg(f0), b = __ldg(f1);
            d[0] = make_float2(a.x, a.z);                   // (u, v) = (0, 0)
            d[plane2 / 2] = make_float2(a.y, a.w);          // (0, 1)
            d[plane2] = make_float2(b.x, b.z);              // (1, 0)
            d[3 * plane2 / 2] = make_float2(b.y, b.w);      // (1, 1)
        } else {
            const float2 p00 = d[0], p01 = d[plane2 / 2], p10 = d[plane2], p11 = d[3 * plane2 / 2];
            *f0 = make_float4(p00.x, p01.x, p00.y, p01.y);
            *f1 = make_float4(p10.x, p11.x, p10.y, p11.y);
        }
    }
}

static int space_depth(const float *src, float *dst, int64_t n, int64_t c, int64_t h, int64_t w,
                       int s, bool to_depth, cudaStream_t st) {
    const int64_t total = n * c * h * w;
    if (s == 2 && w % 4 == 0 && h % 2 == 0 && (h / 2) * (w / 2) % 2 == 0 && total / 8 < (1ll << 31)) {
        const uint32_t t8 = (uint32_t)(total / 8);
        const unsigned blocks = (unsigned)std::min<int64_t>(qt_cdiv(t8, 256), qt_sm_count() * 8);
        const FastDiv qd = make_fastdiv((uint32_t)(w / 4)), yd = make_fastdiv((uint32_t)(h / 2));
        if (to_depth)
            launch_pdl(space_depth2_kernel<true>, blocks, 256, 0, st, src, dst, t8, (uint32_t)h,
                       (uint32_t)w, qd, yd);
        else
            launch_pdl(space_depth2_kernel<false>, blocks, 256, 0, st, src, dst, t8, (uint32_t)h,
                       (uint32_t)w, qd, yd);
        QT_CHECK_LAUNCH();
        return QT_OK;
    }
    const unsigned blocks = (unsigned)std::min<int64_t>(qt_cdiv(total, 256), qt_sm_count() * 16);
    if (to_depth)
        launch_pdl(space_depth_kernel<true>, blocks, 256, 0, st, src, dst, n, c, h, w, s);
    else
        launch_pdl(space_depth_kernel<false>, blocks, 256, 0, st, src, dst, n, c, h, w, s);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

static bool s2d_shape(const ConvGeo &g) {
    return g.s > 1 && g.kh == g.s && g.kw == g.s && g.pad == 0 && g.h % g.s == 0 && g.w % g.s == 0;
}

}  // namespace qt

static int64_t s2d_weights_bytes(const qt::ConvGeo &g) {
    return (qt_conv_workspace(g.ci * g.kh * g.kw, g.co, 1, 1) + 255) / 256 * 256;
}

int64_t qt_tc_s2d_workspace(const qt::ConvGeo &g) {
    if (!s2d_shape(g)) return 0;
    return s2d_weights_bytes(g) + g.n * g.ci * g.h * g.w * (int64_t)sizeof(float);
}

// 1 if the s2d form of this non-overlapping conv runs on the tensor cores
int qt_tc_s2d_ok(const qt::ConvGeo &g, int dgrad) {
    if (tc_disabled() || !s2d_shape(g)) return 0;
    const int64_t c4 = g.ci * g.kh * g.kw, h2 = g.h / g.s, w2 = g.w / g.s;
    if (!dgrad) return tc_shape_ok((int)g.n, (int)c4, (int)h2, (int)w2, (int)g.co, 1, 1, 0) ? 1 : 0;
    return tc_shape_ok((int)g.n, (int)g.co, (int)h2, (int)w2, (int)c4, 1, 1, 0) ? 1 : 0;
}

int qt_tc_conv_s2d_forward(const float *x, const float *w, float *out, const qt::ConvGeo &g,
                           const float *res, int64_t cr, int64_t sr, void *ws, cudaStream_t s) {
    if (!ws || !w || !qt_tc_s2d_ok(g, 0)) return QT_EUNSUPPORTED;
    float *xd = (float *)((char *)ws + s2d_weights_bytes(g));
    int rc = space_depth(x, xd, g.n, g.ci, g.h, g.w, (int)g.s, true, s);
    if (rc) return rc;
    return tc_conv_s1(xd, w, out, (int)g.n, (int)(g.ci * g.kh * g.kw), (int)g.oh, (int)g.ow,
                      (int)g.co, 1, 1, 0, 0, res, (int)cr, (int)sr, ws, s);
}

// ---------------------------------------------------------------------------
// Fused forward (qt_conv_forward_fused): BN-apply + ReLU + K-bit tape in the
// operand prologue and/or the next layer's BN statistics in the epilogue.
namespace qt {

// 1: stride-1 row-tiled or flat tensor-core path; 2: kernel == stride via
// space-to-depth (stats epilogue only); 0: neither
static int fused_route(int64_t n, int64_t ci, int64_t h, int64_t wd, int64_t co, int64_t kh,
                       int64_t kw, int64_t stride, int64_t pad) {
    if (tc_disabled() || n <= 0 || n > INT32_MAX || ci * h * wd > INT32_MAX) return 0;
    if (stride == 1 && tc_shape_ok((int)n, (int)ci, (int)h, (int)wd, (int)co, (int)kh, (int)kw,
                                   (int)pad))
        return 1;
    if (stride > 1 && kh == stride && kw == stride && pad == 0 && h % stride == 0 &&
        wd % stride == 0 &&
        tc_shape_ok((int)n, (int)(ci * kh * kw), (int)(h / stride), (int)(wd / stride), (int)co,
                    1, 1, 0))
        return 2;
    return 0;
}

static bool flat_only(int64_t n, int64_t ci, int64_t h, int64_t wd, int64_t co, int64_t kh,
                      int64_t kw, int64_t pad) {
    return !tc_rows_ok((int)n, (int)ci, (int)h, (int)wd, (int)co, (int)kh, (int)kw, (int)pad);
}

}  // namespace qt

extern "C" int64_t qt_conv_stats_workspace(int64_t co) {
    return 256 + (int64_t)qt_sm_count() * (8 + co * 24);
}

extern "C" int qt_conv_fused_support(int64_t n, int64_t ci, int64_t h, int64_t wd, int64_t co,
                                     int64_t kh, int64_t kw, int64_t stride, int64_t pad,
                                     int64_t sr, int bits) {
    const int route = fused_route(n, ci, h, wd, co, kh, kw, stride, pad);
    if (!route) return 0;
    int r = 0;
    if (route == 1 && qt_bits_ok(bits) && ci <= 512 && (h * wd) % (32 / bits) == 0) r |= 1;
    // the statistics must see the shortcut sum: the flat path adds a strided
    // shortcut in a separate kernel
    const int64_t oh = route == 2 ? h / stride : h + 2 * pad - kh + 1;
    const int64_t ow = route == 2 ? wd / stride : wd + 2 * pad - kw + 1;
    const int64_t cin = route == 2 ? ci * kh * kw : ci;
    const bool flat = route == 2 ? flat_only(n, cin, oh, ow, co, 1, 1, 0)
                                 : flat_only(n, ci, h, wd, co, kh, kw, pad);
    (void)oh; (void)ow;
    if (!(flat && sr > 1) && co % 16 == 0 && co <= 4096) r |= 2;
    return r;
}

extern "C" int qt_conv_forward_fused(const float *x, const float *w, float *out, int64_t n,
                                     int64_t ci, int64_t h, int64_t wd, int64_t co, int64_t kh,
                                     int64_t kw, int64_t stride, int64_t pad, const float *res,
                                     int64_t cr, int64_t sr, const qt_bn_prologue_t *pro,
                                     const qt_bn_stats_epilogue_t *epi, void *ws,
                                     qt_stream_t stream) {
    if (!pro && !epi)
        return qt_conv_forward(x, w, out, n, ci, h, wd, co, kh, kw, stride, pad, res, cr, sr, ws,
                               stream);
    QT_REQUIRE(x && out && ws && n > 0 && ci > 0 && co > 0);
    QT_REQUIRE(!res || (cr > 0 && cr <= co && sr >= 1));
    const int sup = qt_conv_fused_support(n, ci, h, wd, co, kh, kw, stride, pad, res ? sr : 1,
                                          pro ? pro->bits : 4);
    if ((pro && !(sup & 1)) || (epi && !(sup & 2))) return QT_EUNSUPPORTED;
    FuseParams fz{};
    if (pro) {
        QT_REQUIRE(pro->consts && pro->codes && pro->clip_count && qt_bits_ok(pro->bits));
        QT_REQUIRE(((uintptr_t)pro->codes & 3) == 0);
        fz.bn = (const BnConst *)pro->consts;
        fz.codes = (uint32_t *)pro->codes;
        fz.clip = (unsigned long long *)pro->clip_count;
        fz.bits = pro->bits;
    }
    if (epi) {
        QT_REQUIRE(epi->ws && epi->mean && epi->var && epi->gamma && epi->beta && epi->consts &&
                   epi->gamma_copy && epi->beta_copy);
        QT_REQUIRE(epi->bits == 0 || (qt_bits_ok(epi->bits) && epi->step && epi->offset));
        char *b = (char *)epi->ws;
        fz.stats = 1;
        fz.counter = (unsigned *)b;
        fz.pcnt = (double *)(b + 256);
        fz.part = fz.pcnt + qt_sm_count();
        fz.eps = epi->eps;
        fz.gamma = epi->gamma;
        fz.beta = epi->beta;
        fz.nbits = epi->bits;
        fz.mean = epi->mean;
        fz.var = epi->var;
        fz.rmean = epi->running_mean;
        fz.rvar = epi->running_var;
        fz.consts = (BnConst *)epi->consts;
        fz.gcopy = epi->gamma_copy;
        fz.bcopy = epi->beta_copy;
        fz.step = epi->step;
        fz.offset = epi->offset;
        fz.nclip = (unsigned long long *)epi->clip_count;
    }
    const cudaStream_t st = qt_s(stream);
    if (fused_route(n, ci, h, wd, co, kh, kw, stride, pad) == 1)
        return tc_conv_s1(x, w, out, (int)n, (int)ci, (int)h, (int)wd, (int)co, (int)kh, (int)kw,
                          (int)pad, 0, res, (int)cr, (int)sr, ws, st, fz);
    // kernel == stride: space-to-depth, then the 1x1 with the stats epilogue
    QT_REQUIRE(w);
    ConvGeo g{};
    g.n = n; g.ci = ci; g.h = h; g.w = wd; g.co = co; g.kh = kh; g.kw = kw; g.s = stride;
    g.pad = pad; g.oh = h / stride; g.ow = wd / stride;
    float *xd = (float *)((char *)ws + s2d_weights_bytes(g));
    int rc = space_depth(x, xd, g.n, g.ci, g.h, g.w, (int)g.s, true, st);
    if (rc) return rc;
    return tc_conv_s1(xd, w, out, (int)g.n, (int)(g.ci * g.kh * g.kw), (int)g.oh, (int)g.ow,
                      (int)g.co, 1, 1, 0, 0, res, (int)cr, (int)sr, ws, st, fz);
}

int qt_tc_conv_s2d_dgrad(const float *gr, const float *w, float *gx, const qt::ConvGeo &g,
                         void *ws, cudaStream_t s) {
    if (!ws || !w || !qt_tc_s2d_ok(g, 1)) return QT_EUNSUPPORTED;
    float *gd = (float *)((char *)ws + s2d_weights_bytes(g));
    int rc = tc_conv_s1(gr, w, gd, (int)g.n, (int)g.co, (int)g.oh, (int)g.ow,
                        (int)(g.ci * g.kh * g.kw), 1, 1, 0, 1, nullptr, 0, 1, ws, s);
    if (rc) return rc;
    return space_depth(gd, gx, g.n, g.ci, g.h, g.w, (int)g.s, false, s);
}

// ---------------------------------------------------------------------------
// "Same"-padded stride-1 convs whose width is not a tensor-core row width
// (the ImageNet 56/28/14/7 planes of SURVEY.md Appendix C) run on the
// row-tiled tensor-core path over a SEGMENTED copy of the plane:
//   * W <= 32: each row is zero-padded on the right to OWT = 8/16/32 px;
//   * W > 32: each row is cut into segments of 30 output columns carrying a
//     one-column halo on both sides (32 px), and segment j of image n becomes
//     image n * nseg + j of a (N * nseg, C, Hp, 32) tensor.
// Rows are zero-padded to Hp so tiles hold whole rows (and whole images for
// small planes).  The kernel's own row-edge mask supplies the left zero
// column; the padding supplies the right one, so every output column that
// maps back to the image is exact, and the unsegment pass drops the rest.
// For the weight gradient the g_out copy is zero outside those columns, so
// each output pixel contributes exactly once.
namespace qt {

struct SegGeo {
    int ok, owt, halo, nseg, step, hp;
    int flat;   // weight gradient of a kernel == stride conv (1x1 included): the
                // (space-to-depth) plane flattened and zero-padded to 64-px multiples
    int sd;     // flat: the stride (space-to-depth factor of the activation)
};

constexpr int kWgSubRows = 2;   // = kWgSub (conv_tc_wgrad.cuh): 32-px chunks per wgrad stage

static SegGeo seg_geo(int64_t n, int64_t h, int64_t w, int64_t kh, int64_t kw, int64_t pad) {
    SegGeo s{};
    s.sd = 1;
    if (kh != 3 || kw != 3 || pad != 1 || h < 1 || w < 1) return s;
    if (w <= 32) {
        s.owt = w <= 8 ? 8 : (w <= 16 ? 16 : 32);
        s.halo = 0; s.nseg = 1; s.step = s.owt;
    } else {
        s.owt = 32; s.halo = 1; s.step = 30; s.nseg = (int)((w + 29) / 30);
    }
    const int per = 128 / s.owt;
    auto wg_rows_ok = [&](int hp) {   // weight-gradient row tiling (conv_tc_wgrad.cu:wg_plan)
        const int chunks = hp * s.owt / 32;
        return (hp * s.owt) % 32 == 0 && hp % (32 / s.owt) == 0 && chunks % kWgSubRows == 0;
    };
    int hp;
    if (h >= per) {
        hp = (int)((h + per - 1) / per * per);
    } else {
        hp = 1;
        while (hp < h) hp *= 2;
        if ((n * s.nseg) % (per / hp) || !wg_rows_ok(hp)) hp = per;
    }
    if (!wg_rows_ok(hp)) return s;
    s.hp = hp;
    s.ok = 1;
    return s;
}

// Weight gradient of a non-overlapping conv (kernel == stride, no padding; 1x1
// stride 1 included) whose plane is not a multiple of 64 px: dW is the 1x1
// weight gradient of the space-to-depth activation (dW viewed as (co, ci s s),
// the same memory), so both operands are flattened to (n, c, hp * 32) planes,
// zero-padded to whole 64-pixel pairs of 32-px rows.
static SegGeo seg_geo_flat(int64_t h, int64_t w, int64_t kh, int64_t kw, int64_t st, int64_t pad) {
    SegGeo s{};
    if (kh != kw || kh != st || pad != 0 || h % st || w % st) return s;
    const int64_t plane = (h / st) * (w / st);
    s.flat = 1; s.sd = (int)st;
    s.owt = 32; s.halo = 0; s.nseg = 1; s.step = 32;
    s.hp = (int)((plane + 63) / 64 * 2);
    s.ok = 1;
    return s;
}

// dst (n*nseg, c, hp, owt) from src (n, c, h, w).  mode 0: fp32 source, copied;
// 1: g_out, zero outside the segment's own output columns; 2: tape (relu of
// the decoded pre-activation, layer.py:356) or plain fp32 when src != NULL.
// launch-invariant divisors of seg_in_kernel (no runtime IDIV in the loop)
struct SegDiv {
    FastDiv hp, c, nseg, plane, wd, sd2, sd;
    uint32_t owt_log2;
};

static SegDiv seg_div(const SegGeo &s, int64_t c, int64_t w) {
    SegDiv d;
    d.hp = make_fastdiv((uint32_t)s.hp);
    d.c = make_fastdiv((uint32_t)c);
    d.nseg = make_fastdiv((uint32_t)s.nseg);
    d.plane = make_fastdiv((uint32_t)(s.hp * s.owt));
    const int sd = s.sd > 0 ? s.sd : 1;
    d.wd = make_fastdiv((uint32_t)std::max<int64_t>(1, w / sd));
    d.sd2 = make_fastdiv((uint32_t)(sd * sd));
    d.sd = make_fastdiv((uint32_t)sd);
    d.owt_log2 = s.owt == 8 ? 3 : (s.owt == 16 ? 4 : 5);
    return d;
}

// source of element i of a segmented plane: its (n, c, h, w) index si and
// channel tc, or false for a zero (padding) element (MODE as seg_in_kernel)
template <int MODE>
__device__ __forceinline__ bool seg_src(uint32_t i, int c, int h, int w, const SegGeo &s,
                                        const SegDiv &dv, int64_t &si, int &tc) {
    bool ok;
    if (s.flat) {   // c = source channels x sd^2; (h, w) = source extent
        const uint32_t m = fast_div(i, dv.plane), p = i - m * (uint32_t)(s.hp * s.owt);
        const uint32_t wd = (uint32_t)w / (uint32_t)s.sd;
        ok = p < (uint32_t)h / (uint32_t)s.sd * wd;
        if (s.sd == 1) {
            si = (int64_t)m * (uint32_t)(h * w) + p;
            tc = (int)(m - fast_div(m, dv.c) * (uint32_t)c);
        } else {
            const uint32_t nn = fast_div(m, dv.c), ch = m - nn * (uint32_t)c;
            const uint32_t Y = fast_div(p, dv.wd), X = p - Y * wd;
            const uint32_t sd2 = (uint32_t)(s.sd * s.sd), c0 = fast_div(ch, dv.sd2), uv = ch - c0 * sd2;
            const uint32_t u = fast_div(uv, dv.sd), v = uv - u * (uint32_t)s.sd;
            const uint32_t cs = (uint32_t)c / sd2;
            si = (((int64_t)nn * cs + c0) * h + Y * s.sd + u) * w + X * s.sd + v;
            tc = (int)c0;
        }
    } else {
        const uint32_t k = i & ((uint32_t)s.owt - 1u), r = i >> dv.owt_log2;
        const uint32_t r2 = fast_div(r, dv.hp), y = r - r2 * (uint32_t)s.hp;
        const uint32_t m = fast_div(r2, dv.c), ch = r2 - m * (uint32_t)c;
        const uint32_t nn = fast_div(m, dv.nseg), j = m - nn * (uint32_t)s.nseg;
        const int col = (int)(j * s.step + k) - s.halo;
        ok = y < (uint32_t)h && col >= 0 && col < w;
        if (MODE == 1) ok = ok && (int)k >= s.halo && (int)k < s.halo + s.step;
        si = (((int64_t)nn * c + ch) * h + y) * w + col;
        tc = (int)ch;
    }
    return ok;
}

// Four consecutive elements i0..i0+3 of a segmented plane (i0 % 4 == 0: owt
// and the flat plane are multiples of 4, so they share one source row): the
// source index of the first and the valid positions [klo, khi); false for
// the space-to-depth flat form (sd > 1), which maps element by element.
template <int MODE>
__device__ __forceinline__ bool seg_src4(uint32_t i0, int c, int h, int w, const SegGeo &s,
                                         const SegDiv &dv, int64_t &si, int &tc, int &klo,
                                         int &khi) {
    klo = 0;
    khi = 4;
    if (s.flat) {
        if (s.sd != 1) return false;
        const uint32_t m = fast_div(i0, dv.plane), p = i0 - m * (uint32_t)(s.hp * s.owt);
        si = (int64_t)m * (uint32_t)(h * w) + p;
        tc = (int)(m - fast_div(m, dv.c) * (uint32_t)c);
        khi = max(0, min(4, h * w - (int)p));
        return true;
    }
    const uint32_t k = i0 & ((uint32_t)s.owt - 1u), r = i0 >> dv.owt_log2;
    const uint32_t r2 = fast_div(r, dv.hp), y = r - r2 * (uint32_t)s.hp;
    const uint32_t m = fast_div(r2, dv.c), ch = r2 - m * (uint32_t)c;
    const uint32_t nn = fast_div(m, dv.nseg), j = m - nn * (uint32_t)s.nseg;
    const int col = (int)(j * s.step + k) - s.halo;
    si = (((int64_t)nn * c + ch) * h + y) * w + col;
    tc = (int)ch;
    klo = max(0, -col);
    khi = min(4, w - col);
    if (MODE == 1) {
        klo = max(klo, s.halo - (int)k);
        khi = min(khi, s.halo + s.step - (int)k);
    }
    if (y >= (uint32_t)h) khi = 0;
    return true;
}

template <int MODE>
__global__ void seg_in4_kernel(const float *src, qt_tape_t t, float *dst, uint32_t total, int c,
                               int h, int w, SegGeo s, SegDiv dv) {
    pdl_enter();
    const uint32_t quads = total >> 2;
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < quads; q += gridDim.x * blockDim.x) {
        int64_t si;
        int tc, klo, khi;
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (seg_src4<MODE>(4 * q, c, h, w, s, dv, si, tc, klo, khi)) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (k < klo || k >= khi) continue;
                if (MODE != 2 || src) {
                    v[k] = __ldg(src + si + k);
                } else {
                    const float a = tape_value(t, si + k, tc);
                    v[k] = (a >= 0.f || isnan(a)) ? a : 0.f;
                }
            }
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                int64_t sk;
                int tk;
                if (seg_src<MODE>(4 * q + k, c, h, w, s, dv, sk, tk)) {
                    if (MODE != 2 || src) {
                        v[k] = __ldg(src + sk);
                    } else {
                        const float a = tape_value(t, sk, tk);
                        v[k] = (a >= 0.f || isnan(a)) ? a : 0.f;
                    }
                }
            }
        }
        reinterpret_cast<float4 *>(dst)[q] = make_float4(v[0], v[1], v[2], v[3]);
    }
}

template <int MODE>
__global__ void seg_in_kernel(const float *src, qt_tape_t t, float *dst, uint32_t total, int c,
                              int h, int w, SegGeo s, SegDiv dv) {
    pdl_enter();
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        int64_t si;
        int tc;
        const bool ok = seg_src<MODE>(i, c, h, w, s, dv, si, tc);
        float v = 0.f;
        if (ok) {
            if (MODE != 2 || src) {
                v = __ldg(src + si);
            } else {
                const float a = tape_value(t, si, tc);
                v = (a >= 0.f || isnan(a)) ? a : 0.f;
            }
        }
        dst[i] = v;
    }
}

// g_out of a segmented plane straight into the weight gradient's pre-split B
// layout (conv_tc_wgrad.cuh, PRE-SPLIT): per (image, 32-px chunk) three
// piece blocks [co][32 px] of bf16 hi / mid / lo (hi + mid + lo == g to fp32
// precision), pixels pair-permuted in 8-px groups (word k = pixels k, k + 4).
// One thread per (image, chunk, channel, 8-px group): 3 x 16-byte stores.
__global__ void seg_pieces_kernel(const float *g, uint4 *dst, uint32_t groups, int co, int h, int w,
                                  SegGeo s, SegDiv dv, FastDiv cod, FastDiv cpid) {
    pdl_enter();
    const uint32_t plane = (uint32_t)(s.hp * s.owt);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < groups;
         i += gridDim.x * blockDim.x) {
        const uint32_t q = i & 3u, r = i >> 2;
        const uint32_t r2 = fast_div(r, cod), ch = r - r2 * (uint32_t)co;    // r2 = image * cpi + chunk
        const uint32_t nn = fast_div(r2, cpid), chunk = r2 - nn * (plane / 32u);
        const uint32_t p0 = chunk * 32u + 8u * q;     // first pixel of the group in the plane
        // the group's 8 pixels are one run of a source row (owt and the
        // flat plane are multiples of 8): map the first, clip the run
        int64_t si;
        int klo = 0, khi = 8;
        if (s.flat) {   // g_out planes are flat with sd == 1
            si = (int64_t)(nn * (uint32_t)co + ch) * (uint32_t)(h * w) + p0;
            khi = max(0, min(8, h * w - (int)p0));
        } else {
            const uint32_t nimg = fast_div(nn, dv.nseg), j = nn - nimg * (uint32_t)s.nseg;
            const uint32_t y = p0 >> dv.owt_log2, k0 = p0 & ((uint32_t)s.owt - 1u);
            const int col = (int)(j * s.step + k0) - s.halo;
            si = (((int64_t)nimg * co + ch) * h + y) * w + col;
            klo = max(max(0, -col), s.halo - (int)k0);
            khi = min(min(8, w - col), s.halo + s.step - (int)k0);
            if ((int)y >= h) khi = 0;
        }
        float v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = (k >= klo && k < khi) ? __ldg(g + si + k) : 0.f;
        uint32_t H[4], M[4], L[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            H[k] = pack_bf16x2(v[k], v[k + 4]);
            const float rx = __fsub_rn(v[k], bf16_lo(H[k])), ry = __fsub_rn(v[k + 4], bf16_hi(H[k]));
            M[k] = pack_bf16x2(rx, ry);
            L[k] = pack_bf16x2(__fsub_rn(rx, bf16_lo(M[k])), __fsub_rn(ry, bf16_hi(M[k])));
        }
        // [image][chunk][piece][co][4 groups of 16 B]
        uint4 *o = dst + ((size_t)r2 * 3u * (uint32_t)co + ch) * 4u + q;
        const size_t pstride = (size_t)co * 4u;
        o[0] = make_uint4(H[0], H[1], H[2], H[3]);
        o[pstride] = make_uint4(M[0], M[1], M[2], M[3]);
        o[2 * pstride] = make_uint4(L[0], L[1], L[2], L[3]);
    }
}

// Flat weight-gradient operand from a packed tape: codes of the (space-to-
// depth) plane repacked into zero-padded (n, c sd^2, hp * owt) planes in the
// same K-bit little-endian order (codec.pack_codes, codec.py:59-78), plus the
// per-channel step / offset repeated sd^2 times.  Padding pixels carry code 0:
// their g is zero, so any finite decode contributes nothing.
__global__ void seg_codes_kernel(const uint8_t *codes, uint32_t *dst, uint32_t words, int bits,
                                 int c4, int h, int w, SegGeo s, const double *step,
                                 const int64_t *offset, double *step4, int64_t *offset4,
                                 FastDiv pwd, FastDiv c4d, FastDiv nsegd) {
    pdl_enter();
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t sd = (uint32_t)s.sd, sd2 = sd * sd;
    if (tid < (uint32_t)c4) {
        step4[tid] = step[tid / sd2];
        offset4[tid] = offset[tid / sd2];
    }
    const uint32_t per = 32u / (uint32_t)bits;
    const uint32_t pw = (uint32_t)(s.hp * s.owt) / per;       // words per padded plane
    const uint32_t wd = (uint32_t)w / sd, pl = (uint32_t)h / sd * wd;
    const uint32_t cs = (uint32_t)c4 / sd2;
    const uint32_t *src32 = reinterpret_cast<const uint32_t *>(codes);   // 16-byte aligned tape
    const uint32_t owt_log2 = s.owt == 8 ? 3u : (s.owt == 16 ? 4u : 5u);
    for (uint32_t o = tid; o < words; o += gridDim.x * blockDim.x) {
        const uint32_t m = fast_div(o, pwd), wi = o - m * pw;
        uint32_t acc = 0;
        // the word's codes are one run of a source row (flat plane, or a
        // segment row: owt is a multiple of the codes per word): the valid
        // codes [klo, khi) come out of two aligned source words with one
        // funnel shift, the rest of the word is zero padding
        int64_t row = 0;              // code index of the word's first position
        int klo = 0, khi = 0;         // its valid positions (none: all padding)
        const bool run = (s.flat && sd == 1) || (!s.flat && per <= (uint32_t)s.owt);
        if (s.flat && sd == 1) {
            row = (int64_t)m * pl + wi * per;
            khi = min((int)per, (int)pl - (int)(wi * per));
        } else if (!s.flat && per <= (uint32_t)s.owt) {
            const uint32_t img = fast_div(m, c4d), ch = m - img * (uint32_t)c4;
            const uint32_t nn = fast_div(img, nsegd), j = img - nn * (uint32_t)s.nseg;
            const uint32_t p0 = wi * per, y = p0 >> owt_log2, kx = p0 & ((uint32_t)s.owt - 1u);
            const int col = (int)(j * s.step + kx) - s.halo;
            if (y < (uint32_t)h) {
                row = (((int64_t)nn * c4 + ch) * h + y) * w + col;
                klo = max(0, -col);
                khi = min((int)per, w - col);
            }
        }
        if (run) {
            if (khi > klo) {
                const int64_t bit = (row + klo) * bits;
                const int64_t q = bit >> 5;
                const uint32_t sh = (uint32_t)(bit & 31);
                const uint32_t lo = __ldg(src32 + q);
                uint32_t v = sh ? __funnelshift_r(lo, __ldg(src32 + q + 1), sh) : lo;
                const int nv = khi - klo;
                if (nv * bits < 32) v &= (1u << (nv * bits)) - 1u;
                acc = v << (klo * bits);
            }
            dst[o] = acc;
            continue;
        }
        if (s.flat) {
            const uint32_t nn = m / (uint32_t)c4, ch = m - nn * (uint32_t)c4;
            const uint32_t c0 = ch / sd2, uv = ch - c0 * sd2, u = uv / sd, v = uv - u * sd;
            for (uint32_t k = 0; k < per; ++k) {
                const uint32_t p = wi * per + k;
                if (p >= pl) break;
                const uint32_t Y = p / wd, X = p - Y * wd;
                const int64_t si = (((int64_t)nn * cs + c0) * h + Y * sd + u) * w + X * sd + v;
                acc |= get_code(codes, si, bits) << (k * (uint32_t)bits);
            }
        } else {   // segmented (n*nseg, c, hp, owt) layout of the 3x3 path
            const uint32_t img = m / (uint32_t)c4, ch = m - img * (uint32_t)c4;
            const uint32_t nn = img / (uint32_t)s.nseg, j = img - nn * (uint32_t)s.nseg;
            for (uint32_t k = 0; k < per; ++k) {
                const uint32_t p = wi * per + k;
                const uint32_t y = p / (uint32_t)s.owt, kx = p - y * (uint32_t)s.owt;
                const int col = (int)(j * s.step + kx) - s.halo;
                if (y < (uint32_t)h && col >= 0 && col < w)
                    acc |= get_code(codes, (((int64_t)nn * c4 + ch) * h + y) * w + col, bits)
                           << (k * (uint32_t)bits);
            }
        }
        dst[o] = acc;
    }
}

// Segmented 3x3 weight gradient from codes: the padding pixels inside the
// segmented planes (right of the image, below it) hold code 0, whose
// rectified decode z_c = relu(decode(0)) is 0 unless every code of channel c
// decodes positive.  Remove their contribution exactly:
//   dW[co][c][u][v] -= z_c * S[co][u][v],
//   S[co][u][v] = sum over outputs (y, x) whose (u, v) neighbour is such a
//   padding pixel of g[co][y][x]
// (only the last row and the first / last column of outputs have one).
// One block per co.
__global__ void seg_pad_fix_kernel(const float *g, float *grad_w, int n, int co_n, int ci, int h,
                                   int w, SegGeo s, const double *step, const int64_t *offset,
                                   int bits) {
    pdl_enter();
    __shared__ double red[9][256];
    __shared__ double S[9];
    const int co = blockIdx.x, tid = threadIdx.x;
    // only channels whose code 0 decodes positive (every code positive) see
    // the padding pixels: nothing to do for the usual tapes
    int any = 0;
    for (int c = tid; c < ci; c += blockDim.x) any |= decode(0u, step[c], offset[c], bits) > 0.f;
    if (!__syncthreads_or(any)) return;
    const int L = w + 2 * (h - 1);   // last row, last column above it, first column above it
    double acc[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) acc[q] = 0.0;
    for (int t = tid; t < n * L; t += blockDim.x) {
        const int nn = t / L, q = t - nn * L;
        const int y = q < w ? h - 1 : (q < w + h - 1 ? q - w : q - w - h + 1);
        const int x = q < w ? q : (q < w + h - 1 ? w - 1 : 0);
        const double gv = (double)g[(((int64_t)nn * co_n + co) * h + y) * w + x];
#pragma unroll
        for (int uv = 0; uv < 9; ++uv) {
            const int Y = y + uv / 3 - 1, X = x + uv % 3 - 1;
            // inside the segmented plane (row -1 and, without a halo, column
            // -1 are the kernel's own zero padding) but not an image pixel;
            // with a halo, column -1 is segment 0's first column
            const bool in_plane = Y >= 0 && Y < s.hp && X >= -s.halo && (s.halo || X < s.owt);
            const bool pad = in_plane && (Y >= h || X >= w || X < 0);
            if (pad) acc[uv] += gv;
        }
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) red[q][tid] = acc[q];
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {   // fixed-order tree
        if (tid < st)
            for (int q = 0; q < 9; ++q) red[q][tid] += red[q][tid + st];
        __syncthreads();
    }
    if (tid < 9) S[tid] = red[tid][0];
    __syncthreads();
    for (int i = tid; i < ci * 9; i += blockDim.x) {
        const int c = i / 9, uv = i - c * 9;
        const float z = decode(0u, step[c], offset[c], bits);
        if (z > 0.f && S[uv] != 0.0) {
            float *d = grad_w + ((int64_t)co * ci + c) * 9 + uv;
            *d = __fadd_rn(*d, -(float)((double)z * S[uv]));
        }
    }
}

// out (n, c, h, w) [+ shortcut res (n, cr, h*sr, w*sr), engine.py:262-269]
// from the segmented conv result (n*nseg, c, hp, owt)
// Unsegment: out (n, c, h, w) from the segmented / flattened plane (+ the
// shortcut add).  Four pixels x0..x0+3 of one output row per thread (rows
// padded to whole quads in the index space), FastDiv index math.
__global__ void seg_out4_kernel(const float *src, float *out, uint32_t quads, int c, int h, int w,
                                SegGeo s, const float *res, int cr, int sr, FastDiv gprd,
                                FastDiv hd, FastDiv cd, FastDiv stepd, FastDiv sdd) {
    pdl_enter();
    const uint32_t gpr = (uint32_t)(w + 3) >> 2;
    const size_t plane_s = (size_t)s.hp * s.owt;
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < quads; q += gridDim.x * blockDim.x) {
        const uint32_t r = fast_div(q, gprd), xq = q - r * gpr;
        const uint32_t r2 = fast_div(r, hd), y = r - r2 * (uint32_t)h;
        const uint32_t nn = fast_div(r2, cd), ch = r2 - nn * (uint32_t)c;
        const size_t obase = ((size_t)r2 * h + y) * w;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t x = 4 * xq + k;
            if (x >= (uint32_t)w) break;
            float v;
            if (s.flat) {
                const uint32_t sd = (uint32_t)s.sd;
                const uint32_t Y = fast_div(y, sdd), u = y - Y * sd, X = fast_div(x, sdd), vv = x - X * sd;
                const uint32_t cs = (ch * sd + u) * sd + vv;
                v = __ldg(src + ((size_t)nn * c * sd * sd + cs) * plane_s + Y * ((uint32_t)w / sd) + X);
            } else {
                const uint32_t j = fast_div(x, stepd), kk = x - j * s.step + s.halo;
                const uint32_t m = nn * s.nseg + j;
                v = __ldg(src + (((size_t)m * c + ch) * s.hp + y) * s.owt + kk);
            }
            if (res && (int)ch < cr)
                v = __fadd_rn(v, __ldg(res + (((size_t)nn * cr + ch) * h * sr + (size_t)y * sr) * w * sr +
                                       (size_t)x * sr));
            out[obase + x] = v;
        }
    }
}

static unsigned seg_blocks(int64_t total);

static void launch_seg_out(const float *src, float *out, int64_t n, int64_t c, int64_t h, int64_t w,
                           const SegGeo &s, const float *res, int64_t cr, int64_t sr, cudaStream_t st) {
    const int64_t gpr = (w + 3) / 4, quads = n * c * h * gpr;
    launch_pdl(seg_out4_kernel, seg_blocks(quads), 256, 0, st, src, out, (uint32_t)quads, (int)c,
               (int)h, (int)w, s, res, (int)cr, (int)sr, make_fastdiv((uint32_t)gpr),
               make_fastdiv((uint32_t)h), make_fastdiv((uint32_t)c),
               make_fastdiv((uint32_t)std::max(1, s.step)), make_fastdiv((uint32_t)std::max(1, s.sd)));
}


static int64_t seg_elems(const SegGeo &s, int64_t n, int64_t c) {
    return n * s.nseg * c * s.hp * s.owt;
}

static unsigned seg_blocks(int64_t total) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(qt_cdiv(total, 256), qt_sm_count() * 16));
}

template <int MODE>
static int seg_in(const float *src, qt_tape_t t, float *dst, int64_t n, int64_t c, int64_t h,
                  int64_t w, const SegGeo &s, cudaStream_t st) {
    const int64_t total = seg_elems(s, n, c);
    if (total % 4 == 0 && ((uintptr_t)dst & 15) == 0)   // one float4 per thread
        launch_pdl(seg_in4_kernel<MODE>, seg_blocks(total / 4), 256, 0, st, src, t, dst,
                   (uint32_t)total, (int)c, (int)h, (int)w, s, seg_div(s, c, w));
    else
        launch_pdl(seg_in_kernel<MODE>, seg_blocks(total), 256, 0, st, src, t, dst, (uint32_t)total,
                   (int)c, (int)h, (int)w, s, seg_div(s, c, w));
    QT_CHECK_LAUNCH();
    return QT_OK;
}

static bool seg_fits(const SegGeo &s, int64_t n, int64_t c, int64_t h, int64_t w) {
    return s.ok && seg_elems(s, n, c) < (1ll << 31) && n * c * h * w < (1ll << 31);
}

static int64_t seg_wbytes(int64_t ci, int64_t co) {
    return (qt_conv_workspace(ci, co, 3, 3) + 255) / 256 * 256;
}

// stride-1 3x3 "same" conv (forward: flip 0; data gradient: flip 1, ci/co
// swapped by the caller) through the segmented plane
static int seg_conv(const float *x, const float *w, float *out, int64_t n, int64_t ci, int64_t h,
                    int64_t wd, int64_t co, int flip, const float *res, int64_t cr, int64_t sr,
                    void *ws, cudaStream_t st) {
    const SegGeo s = seg_geo(n, h, wd, 3, 3, 1);
    if (!w || !ws || !seg_fits(s, n, ci, h, wd) || !seg_fits(s, n, co, h, wd) || ci % 16 || co % 16)
        return QT_EUNSUPPORTED;
    float *xs = (float *)((char *)ws + seg_wbytes(ci, co));
    float *os = xs + seg_elems(s, n, ci);
    int rc = seg_in<0>(x, qt_tape_t{}, xs, n, ci, h, wd, s, st);
    if (rc) return rc;
    rc = tc_conv_s1(xs, w, os, (int)(n * s.nseg), (int)ci, s.hp, s.owt, (int)co, 3, 3, 1, flip,
                    nullptr, 0, 1, ws, st);
    if (rc) return rc;
    launch_seg_out(os, out, n, co, h, wd, s, res, cr, sr, st);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

// kernel == stride conv (1x1 included) on a plane the flat tensor-core path
// cannot address (e.g. 7x7 = 49 px: rows not 16-byte aligned): the
// (space-to-depth) plane zero-padded to 64-px multiples, the tensor-core 1x1,
// then back.  Forward: x (n, ci, h, w) -> out (n, co, h/sd, w/sd); data
// gradient (flip 1): g (n, co, h/sd, w/sd) -> gx (n, ci, h, w).
static int seg_conv_flat(const float *src, const float *w, float *dst, int64_t n, int64_t ci,
                         int64_t h, int64_t wd, int64_t co, int sd, int flip, const float *res,
                         int64_t cr, int64_t sr, void *ws, cudaStream_t st) {
    const SegGeo s = seg_geo_flat(h, wd, sd, sd, sd, 0);
    const int64_t c4 = ci * sd * sd, oh = h / sd, ow = wd / sd;
    if (!w || !ws || !s.ok || c4 % 16 || co % 16) return QT_EUNSUPPORTED;
    if (seg_elems(s, n, c4 + co) >= (1ll << 31) || n * c4 * oh * ow >= (1ll << 31) ||
        n * co * oh * ow >= (1ll << 31))
        return QT_EUNSUPPORTED;
    float *xs = (float *)((char *)ws + (qt_conv_workspace(c4, co, 1, 1) + 255) / 256 * 256);
    float *os = xs + seg_elems(s, n, flip ? co : c4);
    SegGeo s1 = s;
    s1.sd = 1;
    int rc;
    if (!flip) {
        rc = seg_in<0>(src, qt_tape_t{}, xs, n, c4, h, wd, s, st);
        if (rc) return rc;
        rc = tc_conv_s1(xs, w, os, (int)n, (int)c4, s.hp, s.owt, (int)co, 1, 1, 0, 0, nullptr, 0, 1, ws, st);
        if (rc) return rc;
        launch_seg_out(os, dst, n, co, oh, ow, s1, res, cr, sr, st);
    } else {
        rc = seg_in<0>(src, qt_tape_t{}, xs, n, co, oh, ow, s1, st);
        if (rc) return rc;
        rc = tc_conv_s1(xs, w, os, (int)n, (int)co, s.hp, s.owt, (int)c4, 1, 1, 0, 1, nullptr, 0, 1, ws, st);
        if (rc) return rc;
        launch_seg_out(os, dst, n, ci, h, wd, s, nullptr, 0, 1, st);
    }
    QT_CHECK_LAUNCH();
    return QT_OK;
}

}  // namespace qt

// scratch of the segmented forward / data gradient (0: shape not taken)
int64_t qt_tc_seg_workspace(const qt::ConvGeo &g) {
    const SegGeo f = seg_geo_flat(g.h, g.w, g.kh, g.kw, g.s, g.pad);
    if (f.ok) {
        const int64_t c4 = g.ci * g.kh * g.kw;
        return (qt_conv_workspace(c4, g.co, 1, 1) + 255) / 256 * 256 + 4 * seg_elems(f, g.n, c4 + g.co) + 256;
    }
    if (g.s != 1) return 0;
    const SegGeo s = seg_geo(g.n, g.h, g.w, g.kh, g.kw, g.pad);
    if (!s.ok) return 0;
    return seg_wbytes(g.ci, g.co) + 4 * seg_elems(s, g.n, g.ci + g.co) + 256;
}

int qt_tc_conv_seg_forward(const float *x, const float *w, float *out, const qt::ConvGeo &g,
                           const float *res, int64_t cr, int64_t sr, void *ws, cudaStream_t st) {
    if (tc_disabled()) return QT_EUNSUPPORTED;
    if (seg_geo_flat(g.h, g.w, g.kh, g.kw, g.s, g.pad).ok)
        return seg_conv_flat(x, w, out, g.n, g.ci, g.h, g.w, g.co, (int)g.s, 0, res, cr, sr, ws, st);
    if (g.s != 1 || g.kh != 3 || g.kw != 3 || g.pad != 1) return QT_EUNSUPPORTED;
    return seg_conv(x, w, out, g.n, g.ci, g.h, g.w, g.co, 0, res, cr, sr, ws, st);
}

int qt_tc_conv_seg_dgrad(const float *gr, const float *w, float *gx, const qt::ConvGeo &g,
                         void *ws, cudaStream_t st) {
    if (tc_disabled()) return QT_EUNSUPPORTED;
    if (seg_geo_flat(g.h, g.w, g.kh, g.kw, g.s, g.pad).ok)
        return seg_conv_flat(gr, w, gx, g.n, g.ci, g.h, g.w, g.co, (int)g.s, 1, nullptr, 0, 1, ws, st);
    if (g.s != 1 || g.kh != 3 || g.kw != 3 || g.pad != 1) return QT_EUNSUPPORTED;
    return seg_conv(gr, w, gx, g.n, g.co, g.oh, g.ow, g.ci, 1, nullptr, 0, 1, ws, st);
}

int qt_tc_conv_wgrad(const float *gr, qt_tape_t act, const float *x_plain, float *grad_w,
                     const qt::ConvGeo &g, void *ws, cudaStream_t st);
int qt_tc_conv_wgrad_pre(const void *pieces, qt_tape_t act, float *grad_w, const qt::ConvGeo &g,
                         void *ws, cudaStream_t st);
bool qt_tc_wgrad_pre_ok(const qt::ConvGeo &g, int bits);
int qt_tc_conv_wgrad_fp32(const float *gr, qt_tape_t act, const float *x_plain, float *grad_w,
                          const qt::ConvGeo &g, void *ws, cudaStream_t st);
int64_t qt_tc_wgrad_workspace(const qt::ConvGeo &g);
int64_t qt_tc_wgrad_partial_workspace(const qt::ConvGeo &g);

// g_out (n, co, h, w) of an unsegmented plane (h * w % 32 == 0) into the
// weight gradient's bf16 pieces (seg_pieces_kernel on a flat geometry)
int qt_tc_wgrad_pieces(const float *g, void *dst, int64_t n, int64_t co, int64_t h, int64_t w,
                       cudaStream_t st) {
    if ((h * w) % 32 || ((uintptr_t)dst & 15) || n * co * h * w >= (1ll << 31)) return QT_EUNSUPPORTED;
    SegGeo s{};
    s.ok = 1; s.flat = 1; s.sd = 1; s.owt = 32; s.halo = 0; s.nseg = 1; s.step = 32;
    s.hp = (int)(h * w / 32);
    const uint32_t groups = (uint32_t)(n * co * h * w / 8);
    launch_pdl(seg_pieces_kernel, seg_blocks(groups), 256, 0, st, g, (uint4 *)dst, groups, (int)co,
               (int)h, (int)w, s, seg_div(s, co, w), make_fastdiv((uint32_t)co),
               make_fastdiv((uint32_t)(h * w / 32)));
    QT_CHECK_LAUNCH();
    return QT_OK;
}

static qt::ConvGeo seg_wgrad_geo(const qt::ConvGeo &g, const SegGeo &s) {
    qt::ConvGeo d = g;
    d.n = g.n * s.nseg;
    d.h = d.oh = s.hp;
    d.w = d.ow = s.owt;
    if (s.flat) {   // 1x1, stride 1 over the (space-to-depth) channels
        d.ci = g.ci * s.sd * s.sd;
        d.kh = d.kw = 1;
        d.s = 1;
        d.pad = 0;
    }
    return d;
}

static SegGeo seg_geo_wgrad(const qt::ConvGeo &g) {
    const SegGeo f = seg_geo_flat(g.h, g.w, g.kh, g.kw, g.s, g.pad);
    if (f.ok) return f;
    return g.s == 1 ? seg_geo(g.n, g.h, g.w, g.kh, g.kw, g.pad) : SegGeo{};
}

int64_t qt_tc_seg_wgrad_workspace(const qt::ConvGeo &g) {
    const SegGeo s = seg_geo_wgrad(g);
    if (!s.ok) return 0;
    const int64_t part = (qt_tc_wgrad_partial_workspace(seg_wgrad_geo(g, s)) + 255) / 256 * 256;
    // g_out region: fp32 (4 B) or bf16 pieces (6 B per element)
    const int64_t gbytes = (6 * seg_elems(s, g.n, g.co) + 255) / 256 * 256;
    return part + gbytes + 4 * seg_elems(s, g.n, g.ci * s.sd * s.sd) + g.ci * s.sd * s.sd * 16 + 1024;
}

// weight gradient: segmented g_out (zero outside each segment's own columns)
// against the segmented rectified activation, on the fp32-operand path
int qt_tc_conv_seg_wgrad(const float *gr, qt_tape_t act, const float *x_plain, float *grad_w,
                         const qt::ConvGeo &g, void *ws, cudaStream_t st) {
    if (tc_disabled() || !ws) return QT_EUNSUPPORTED;
    if (!x_plain && !act.a2 && !act.codes) return QT_EUNSUPPORTED;
    const SegGeo s = seg_geo_wgrad(g);
    const int64_t cin = g.ci * (s.flat ? s.sd * s.sd : 1);
    if (!seg_fits(s, g.n, cin, g.h, g.w) || !seg_fits(s, g.n, g.co, g.h, g.w)) return QT_EUNSUPPORTED;
    const qt::ConvGeo d = seg_wgrad_geo(g, s);
    const int64_t part = (qt_tc_wgrad_partial_workspace(d) + 255) / 256 * 256;
    if (part <= 0) return QT_EUNSUPPORTED;
    float *gs = (float *)((char *)ws + part);
    float *as = (float *)((char *)gs + (6 * seg_elems(s, g.n, g.co) + 255) / 256 * 256);
    // g_out is already the flat plane in the flat case: a 1x1 view of (oh, ow)
    SegGeo sg = s;
    if (s.flat) sg.sd = 1;
    const int64_t gh = s.flat ? g.oh : g.h, gw = s.flat ? g.ow : g.w;
    const bool codes = !x_plain && !act.a2 && act.codes && qt_bits_ok(act.bits);
    bool pre = codes && qt_tc_wgrad_pre_ok(d, act.bits);
    int rc;
    if (pre) {   // g_out straight into the bf16 pieces the weight gradient's TMA reads
        const uint32_t groups = (uint32_t)(seg_elems(s, g.n, g.co) / 8);
        const uint32_t cpi = (uint32_t)(s.hp * s.owt / 32);
        launch_pdl(seg_pieces_kernel, seg_blocks(groups), 256, 0, st, gr, (uint4 *)gs, groups,
                   (int)g.co, (int)gh, (int)gw, sg, seg_div(sg, g.co, gw), make_fastdiv((uint32_t)g.co),
                   make_fastdiv(cpi));
        QT_CHECK_LAUNCH();
    } else {
        rc = seg_in<1>(gr, qt_tape_t{}, gs, g.n, g.co, gh, gw, sg, st);
        if (rc) return rc;
    }
    if (codes) {
        // packed operand: the tensor-core path decodes it in its operand staging
        const int64_t words = seg_elems(s, g.n, cin) * act.bits / 32;
        uint32_t *cw = (uint32_t *)as;
        double *step4 = (double *)((char *)as + (words * 4 + 255) / 256 * 256);
        int64_t *off4 = (int64_t *)(step4 + cin);
        launch_pdl(seg_codes_kernel, seg_blocks(std::max(words, cin)), 256, 0, st, act.codes, cw,
                   (uint32_t)words, act.bits, (int)cin, (int)g.h, (int)g.w, s, act.step, act.offset,
                   step4, off4, make_fastdiv((uint32_t)(s.hp * s.owt * act.bits / 32)),
                   make_fastdiv((uint32_t)cin), make_fastdiv((uint32_t)s.nseg));
        QT_CHECK_LAUNCH();
        qt_tape_t t2{nullptr, (const uint8_t *)cw, step4, off4, act.bits};
        rc = pre ? qt_tc_conv_wgrad_pre(gs, t2, grad_w, d, ws, st)
                 : qt_tc_conv_wgrad_fp32(gs, t2, nullptr, grad_w, d, ws, st);
        if (rc == QT_EUNSUPPORTED && pre) {   // the fp32 plane for the paths below
            pre = false;
            rc = seg_in<1>(gr, qt_tape_t{}, gs, g.n, g.co, gh, gw, sg, st);
            if (rc) return rc;
            rc = qt_tc_conv_wgrad_fp32(gs, t2, nullptr, grad_w, d, ws, st);
        }
        if (rc != QT_EUNSUPPORTED) {
            if (rc || s.flat) return rc;
            if (s.hp == g.h && !s.halo && s.owt == g.w) return rc;   // no padding pixels
            launch_pdl(seg_pad_fix_kernel, (unsigned)g.co, 256, 0, st, gr, grad_w, (int)g.n,
                       (int)g.co, (int)g.ci, (int)g.h, (int)g.w, s, act.step, act.offset, act.bits);
            QT_CHECK_LAUNCH();
            return QT_OK;
        }
    }
    rc = seg_in<2>(x_plain, act, as, g.n, cin, g.h, g.w, s, st);
    if (rc) return rc;
    return qt_tc_conv_wgrad_fp32(gs, qt_tape_t{}, as, grad_w, d, ws, st);
}
