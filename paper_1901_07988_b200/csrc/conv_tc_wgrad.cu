// Weight gradient on the tensor cores: host planning, tensor maps, the
// fixed-order split-K reduction and the C-ABI entry points.  The kernel and
// its launch templates live in conv_tc_wgrad.cuh; each output-channel tile
// width BN is instantiated in its own unit (conv_tc_wgrad_bn*.cu).
#include "conv_tc_wgrad.cuh"

namespace qt {

// per-BN launchers (conv_tc_wgrad_bn*.cu)
int wg_launch_bn16(const CUtensorMap &, const CUtensorMap &, const WgParams &, const WgPlan &, cudaStream_t);
int wg_launch_bn32(const CUtensorMap &, const CUtensorMap &, const WgParams &, const WgPlan &, cudaStream_t);
int wg_launch_bn64(const CUtensorMap &, const CUtensorMap &, const WgParams &, const WgPlan &, cudaStream_t);
int wg_launch_bn128(const CUtensorMap &, const CUtensorMap &, const WgParams &, const WgPlan &, cudaStream_t);
int wg_launch_bn256(const CUtensorMap &, const CUtensorMap &, const WgParams &, const WgPlan &, cudaStream_t);

// grad_w[i] = fp32(grad_w[i] + fp32(sum_z partial[z][i])) -- 32 warps of a
// block sum interleaved split subsets for 32 consecutive outputs, then
// combine in warp order: fixed order, deterministic (layer.py:167).
__global__ void __launch_bounds__(1024) wgrad_reduce_kernel(const float *partial, int64_t splits,
                                                           int64_t count, float *grad_w) {
    pdl_enter();
    __shared__ double red[32][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * 32 + lane;
    double s = 0.0;
    if (i < count) {
        int64_t z = warp;
        for (; z + 96 < splits; z += 128) {
            const float a = partial[z * count + i], b = partial[(z + 32) * count + i];
            const float c = partial[(z + 64) * count + i], d = partial[(z + 96) * count + i];
            s += (double)a;
            s += (double)b;
            s += (double)c;
            s += (double)d;
        }
        for (; z < splits; z += 32) s += (double)partial[z * count + i];
    }
    red[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && i < count) {
        double t = 0.0;
        for (int w = 0; w < 32; ++w) t += red[w][lane];
        grad_w[i] = __fadd_rn(grad_w[i], __double2float_rn(t));
    }
}

// Few splits: one thread per output sums its splits in order (z = 0, 1, ...)
// in float64 -- fixed order, deterministic, coalesced across threads.
__global__ void __launch_bounds__(256) wgrad_reduce_few_kernel(const float *partial, int splits,
                                                              int64_t count, float *grad_w) {
    pdl_enter();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int z = 0; z < splits; ++z) s += (double)__ldg(partial + z * count + i);
        grad_w[i] = __fadd_rn(grad_w[i], __double2float_rn(s));
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn_wg() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *q = nullptr;
        cudaDriverEntryPointQueryResult r;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r) ==
                cudaSuccess &&
            r == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)q;
    });
    return fn;
}

// bits > 0: the activation is a packed code tape of that width; tap: 3x3
// with the column taps moved into N (4-bit codes, BN <= 32)
// pre: g_out arrives as bf16 pieces (FAST-capable codes, stacked, no taps)
static WgPlan wg_plan(const ConvGeo &g, int bits, bool tap = false, bool fbox = false,
                      bool pre = false) {
    WgPlan pl;
    if (pre && (tap || fbox || !(bits == 1 || bits == 2 || bits == 4))) return pl;
    if (g.s != 1) return pl;
    const int64_t ow = g.ow, oh = g.oh;
    if (ow != 8 && ow != 16 && ow != 32) return pl;
    if (g.w != ow) return pl;                    // same-width rows (stride 1, "same" padding)
    if ((oh * ow) % 32 || oh % (32 / ow)) return pl;
    if ((oh * ow / 32) % kWgSub) return pl;           // SUB chunks per stage within one image
    if (g.co % 16 || (g.co > 256 && g.co % 64) || !(g.kw == 1 || g.kw == 3) || g.pad > 1) return pl;
    if (g.kw == 1 && g.pad != 0) return pl;
    if (g.kh != g.kw) return pl;
    if (g.n * oh * ow / 32 > INT32_MAX) return pl;
    int bn = g.co <= 16 ? 16 : g.co <= 32 ? 32 : g.co <= 64 ? 64 : g.co <= 128 ? 128 : 256;
    // wide outputs in blocks of 64 channels (grid z): three stacked bf16
    // pieces and a four-deep operand ring fit only up to 64 -- the A decode
    // is repeated per block, cheap for the narrow-input expand layers
    if (bn > 64 && g.co % 64 == 0 && !tap) bn = 64;
    // pre-split pieces: the B tile is TMA traffic, not operand work -- wide
    // outputs take 128-channel blocks (three N = 128 MMAs per K step, one
    // accumulator) and both m-tiles of a pair, so each byte of B read from
    // L2 feeds twice the MMA work (the L2 -> SM rate bounds the stacked form)
    const int64_t mt0 = (g.ci * g.kh * g.kw + 127) / 128;
    if (pre && g.co % 128 == 0 && mt0 >= 2) bn = 128;
    if (pre) {
        static const int bn_env = [] {
            const char *e = getenv("QTAPE_WG_PRE_BN");
            return e ? atoi(e) : 0;
        }();
        if (bn_env >= 16 && bn_env <= 128 && g.co % bn_env == 0) bn = bn_env;   // tuning
    }
    if (g.co % bn) return pl;
    pl.bn = bn;
    pl.nblk = (int)(g.co / bn);
    if (tap && !(g.kh == 3 && g.pad == 1 && bn <= 32 && bits == 4)) return WgPlan{};
    pl.tap = tap ? 1 : 0;
    pl.rpc = (int)(tap ? g.kh : g.kh * g.kw);
    const int nt = tap ? 3 : 1;
    const int64_t R = g.ci * pl.rpc;                     // A rows
    const int64_t Rout = g.ci * g.kh * g.kw;             // dW rows
    const int64_t mt = (R + 127) / 128;
    const bool stack = tap ? 9 * bn <= 256 : 3 * bn <= 192;
    const int facc = stack ? 3 * nt * bn : nt * bn;      // FAST accumulator columns per tile
    const int gacc = nt * bn;                            // GENERIC accumulator columns per tile
    // operand bytes per chunk: FAST 3 bf16 pieces (only 2/4-bit codes take
    // FAST), GENERIC TF32 (hi, lo); the two modes share one smem region
    const int opb_g = 2 * nt * bn * 128;
    const int opb_f = (bits == 1 || bits == 2 || bits == 4 || bits == 8) ? 3 * nt * bn * 64 : opb_g;
    // TMEM (512 columns): FAST needs mtg*facc + ops*mtg*SUB*16, GENERIC
    // mtg*BN + ops_g*mtg*SUB*64; ring depths are powers of two (see kWgGroups)
    constexpr int SUB = kWgSub;
    // two m-tiles per CTA share one g split, but only pay when the pair
    // still leaves four operand stages in TMEM and the tiles are not one of
    // three or more (measured: mtg 1 wins for mt >= 3 and for ops < 4)
    int mtg = (int)std::min<int64_t>(mt, 2);
    if (mtg == 2 && ((!pre && mt >= 3) || 2 * facc + 4 * 2 * SUB * 16 > 512)) mtg = 1;
    if (const char *e = getenv("QTAPE_WG_MTG")) mtg = std::max(1, std::min(mtg, atoi(e)));   // tuning
    while (mtg > 1 && (mtg * gacc + mtg * SUB * 64 > 512 || mtg * facc + 2 * mtg * SUB * 16 > 512))
        --mtg;
    if (mtg * gacc + mtg * SUB * 64 > 512 || mtg * facc + 2 * mtg * SUB * 16 > 512) return WgPlan{};
    // GENERIC-PRE keeps three bf16 A pieces (48 columns per chunk) in TMEM
    while (pre && mtg > 1 && mtg * facc + mtg * SUB * 48 > 512) --mtg;
    if (pre && mtg * facc + mtg * SUB * 48 > 512) return WgPlan{};
    pl.mtg = mtg;
    pl.mgroups = (int)((mt + mtg - 1) / mtg);
    pl.ops = 4;
    while (pl.ops > 2 && mtg * facc + pl.ops * mtg * SUB * 16 > 512) pl.ops /= 2;
    const int gbytes0 = bn * 128;
    int gbytes = gbytes0;
    if (bits > 0) {   // TMA code box per stage: 16-byte aligned window of the chunk's input rows
        const int64_t plane = g.h * g.w * bits;
        if (plane % 128) return WgPlan{};               // plane stride: 16-byte multiple
        const int kk = pl.rpc;
        pl.nch = (int)std::min<int64_t>(g.ci, (mtg * 128 + kk - 1) / kk + (kk > 1 ? 1 : 0));
        pl.rb = (int)(ow * bits / 8);
        pl.cb = (((int)(32 / ow) * SUB + 2 * (int)g.pad) * pl.rb + 15 + 15) & ~15;
        if (pl.cb > 256 || pl.nch > kWgMaxCh) return WgPlan{};
        pl.cbytes = pl.cb * pl.nch;
        // padded channel stride: (hi, lo) pairs, or (pre) the value itself;
        // a table past kWgLutEntries (8-bit codes over wide channel blocks)
        // is computed inline by the GENERIC operand instead
        if (pl.nch * (1 << bits) > kWgLutEntries) {
            if (pre) return WgPlan{};
            pl.nolut = 1;
        } else {
            pl.lut_floats = pl.nch * (pre ? (1 << bits) + 1 : (2 << bits) + 2);
        }
    } else if (fbox) {   // fp32 box per stage: the chunk rows plus the pad rows of each channel
        const int kk = pl.rpc;
        pl.nch = (int)std::min<int64_t>(g.ci, (mtg * 128 + kk - 1) / kk + (kk > 1 ? 1 : 0));
        pl.rb = (int)(ow * 4);
        pl.cb = ((int)(32 / ow) * SUB + 2 * (int)g.pad) * pl.rb;
        if (pl.cb / 4 > 256 || pl.nch > kWgMaxCh) return WgPlan{};
        pl.cbytes = pl.cb * pl.nch;
        pl.fbox = 1;
    }
    gbytes = ((pre ? 0 : SUB * gbytes0) + pl.cbytes + 1023) & ~1023;    // one raw stage
    pl.slot = gbytes;
    const int fixed = pl.lut_floats * 4 + kWgMaxCh * 4 + 1024 + 512;
    const int budget = 227 * 1024 - fixed;
    if (pre) {
        // raw ring = code boxes only (owned by the FAST groups: a multiple of
        // ops), B ring = the pieces (MMA warp only, any depth >= 2); no smem
        // operand region (A lives in TMEM in both modes)
        pl.pre = 1;
        // A stages live only in TMEM: up to two per operand group
        pl.ops = 8;
        while (pl.ops > 2 && mtg * facc + pl.ops * mtg * SUB * 16 > 512) pl.ops /= 2;
        pl.ops_g = std::min(pl.ops, 4);
        while (pl.ops_g > 1 && mtg * facc + pl.ops_g * mtg * SUB * 48 > 512) pl.ops_g /= 2;
        const int bstage = SUB * 3 * bn * 64;
        const int G = std::min(pl.ops, 4);                // active FAST groups
        pl.rg = std::max(pl.ops, std::min(8, budget / 3 / gbytes) / G * G);
        pl.bring = std::min(8, (budget - pl.rg * gbytes) / bstage);
        if (pl.bring < 2) return WgPlan{};
        pl.opreg = pl.bring * bstage;
        pl.smem = pl.rg * gbytes + pl.opreg + fixed;
    } else {
    const int sraw = gbytes;                                  // bytes per raw stage
    pl.ops_g = pl.ops;
    while (pl.ops_g > 1 && mtg * gacc + pl.ops_g * mtg * SUB * 64 > 512) pl.ops_g /= 2;
    // operand region: ops FAST stages or ops_g GENERIC stages (a CTA takes
    // one mode), at least one raw stage per FAST operand stage beside it
    auto region = [&] { return std::max(pl.ops * SUB * opb_f, pl.ops_g * SUB * opb_g); };
    while (pl.ops > 1 && region() + pl.ops * sraw > budget) {
        pl.ops /= 2;
        pl.ops_g = std::min(pl.ops_g, pl.ops);
    }
    if (region() + pl.ops * sraw > budget) return WgPlan{};
    // raw ring: the largest multiple of ops up to 8 stages that fits
    pl.rg = std::min(8, (budget - region()) / sraw) / pl.ops * pl.ops;
    if (pl.rg < pl.ops) return WgPlan{};
    pl.opreg = region();
    pl.smem = pl.rg * sraw + pl.opreg + fixed;
    // FAST2 (two A pieces, 32 TMEM columns per chunk): the deepest ring
    // within the FAST one that fits beside the accumulators
    if (bits > 0 && !tap)
        for (int o2 = pl.ops; o2 >= 1 && !pl.ops2; o2 /= 2)
            if (mtg * facc + o2 * mtg * SUB * 32 <= 512) pl.ops2 = o2;
    }
    pl.total = (int)(g.n * oh * ow / 32);
    // split-K count: one CTA per SM (one is resident per SM: a second wave
    // would pay setup, pipeline fill and epilogue again), at least one
    // pipeline stage (SUB chunks) per CTA, and the fp32
    // partials (splits x R x co x 4 B, written once and read back by the
    // fixed-order reduction) at most max(4x the g_out bytes, 32 MiB)
    // With the data gradients running beside (qt_set_concurrent_backward),
    // small (CIFAR-sized, < 2^30 MAC) layers take half the SMs and the data
    // gradient the other half (measured on C2: wgrad alone on 74 CTAs 9.72 ->
    // 9.50 ms/step, both halved 8.97; any split summing past 148 is worse).
    // ImageNet-sized layers use every SM (C4 53 ms at 148 CTAs, 62 at 74).
    static const int ctas_env = [] {
        const char *e = getenv("QTAPE_WG_CTAS");
        return e && atoi(e) > 0 ? atoi(e) : 0;
    }();
    const double macs = (double)g.n * (double)oh * (double)ow * (double)g.co * (double)Rout;
    const int ctas = ctas_env > 0 ? ctas_env : ((g_concurrent_bwd && macs < kSmallLayerMacs) ? qt_sm_count() / 2 : qt_sm_count());
    int want = std::max(1, ctas / (pl.mgroups * pl.nblk));   // one wave: fixed costs once per SM
    want = std::min(want, std::max(1, pl.total / SUB));
    // a CTA's stages run concurrently on its operand groups, so give each
    // CTA at least one stage per group: the kernel takes about as long on
    // fewer SMs (latency-bound), leaves the rest to the input-gradient chain
    // running beside it, and writes fewer partials
    want = std::min(want, std::max(1, pl.total / (SUB * std::min(pl.ops, 4))));
    const double gbytes_all = 128.0 * g.co * pl.total;
    const double part_cap = std::max(4.0 * gbytes_all, 32.0 * 1024 * 1024);
    want = std::min(want, std::max(1, (int)(part_cap / (4.0 * (double)Rout * g.co))));
    pl.cps = std::max(1, (pl.total + want - 1) / want);
    pl.cps = (pl.cps + SUB - 1) / SUB * SUB;          // stages never straddle splits or images
    pl.splits = (pl.total + pl.cps - 1) / pl.cps;
    pl.ok = true;
    return pl;
}

}  // namespace qt

using namespace qt;

static bool tcw_disabled() {
    const char *e = getenv("QTAPE_NO_TC");
    return e && *e && *e != '0';
}

// ------------------------------------------------------------------------
// Kernel == stride 2 (the 2x2/s2 transitions) on a packed code tape: the
// weight gradient is the 1x1 weight gradient of the space-to-depth input
//   x'[n][(c*2 + u)*2 + v][y][x] = x[n][c][2y + u][2x + v]
// with dW viewed as (co, 4 ci) -- the same memory.  Codes move, not values:
// one 32-bit word of x' codes takes every other code of two words of an input
// row, and step'/offset' repeat each channel's constants 4x.  The tensor-core
// path then runs its FAST / GENERIC modes on the rearranged tape unchanged.
namespace qt {

__global__ void codes_s2d_kernel(const uint8_t *codes, uint32_t *out, uint32_t words,
                                 uint32_t h, uint32_t w, int bits, FastDiv wrd, FastDiv hd,
                                 const double *step, const int64_t *offset, double *step4,
                                 int64_t *offset4, uint32_t c4) {
    pdl_enter();
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    if (tid < c4) {
        step4[tid] = step[tid >> 2];
        offset4[tid] = offset[tid >> 2];
    }
    const uint32_t per = 32u / (uint32_t)bits;           // codes per output word
    const uint32_t wr = (w / 2) / per;                   // output words per x' row
    const uint32_t h2 = h >> 1;
    const uint32_t mask = (1u << bits) - 1u;
    const uint32_t rowb = w * (uint32_t)bits / 8;        // bytes per input row
    for (uint32_t o = tid; o < words; o += gridDim.x * blockDim.x) {
        const uint32_t r = fast_div(o, wrd), wi = o - r * wr;   // r = dplane * h2 + y
        const uint32_t dp = fast_div(r, hd), y = r - dp * h2;    // dp = plane * 4 + u * 2 + v
        const uint32_t pl = dp >> 2, u = (dp >> 1) & 1u, v = dp & 1u;
        const uint32_t *src = reinterpret_cast<const uint32_t *>(
            codes + ((size_t)pl * h + 2 * y + u) * rowb) + 2 * wi;
        const uint64_t both = (uint64_t)__ldg(src) | ((uint64_t)__ldg(src + 1) << 32);
        uint32_t acc = 0;
        for (uint32_t k = 0; k < per; ++k)
            acc |= ((uint32_t)(both >> ((2 * k + v) * (uint32_t)bits)) & mask) << (k * (uint32_t)bits);
        out[o] = acc;
    }
}

static bool wg_s2d_shape(const ConvGeo &g, int bits) {
    if (g.s != 2 || g.kh != 2 || g.kw != 2 || g.pad != 0 || g.h % 2 || g.w % 2) return false;
    if (bits != 1 && bits != 2 && bits != 4 && bits != 8) return false;
    if ((g.w / 2) * bits % 32 || (g.w * bits) % 8) return false;   // whole words per x' row
    return g.n * g.ci * g.h * g.w * bits / 32 < (1ll << 31);
}

// A 1x1 / stride 1 / pad 0 weight gradient only sees pixels, so a plane of
// hw % 64 == 0 pixels (e.g. 56x56) can be read as rows of 32 -- the same
// bytes in memory, codes and g alike -- when its own width is not 8/16/32.
static bool wg_flat_shape(const ConvGeo &g) {
    if (g.kh != 1 || g.kw != 1 || g.s != 1 || g.pad != 0) return false;
    if (g.w == 8 || g.w == 16 || g.w == 32) return false;
    return (g.h * g.w) % 64 == 0;
}

static ConvGeo wg_flat_geo(const ConvGeo &g) {
    ConvGeo d = g;
    d.w = d.ow = 32;
    d.h = d.oh = g.h * g.w / 32;
    return d;
}

static ConvGeo wg_s2d_geo(const ConvGeo &g) {
    ConvGeo d = g;
    d.ci = g.ci * 4;
    d.h = g.h / 2;
    d.w = g.w / 2;
    d.kh = d.kw = 1;
    d.s = 1;
    d.pad = 0;
    d.oh = d.h;
    d.ow = d.w;
    return d;
}

static int64_t wg_s2d_bytes(const ConvGeo &g, int bits) {   // codes' + step' + offset'
    return (g.n * g.ci * g.h * g.w * bits / 8 + 255) / 256 * 256 + g.ci * 4 * 16 + 256;
}

}  // namespace qt

// fp32 split-K partials of every plan this geometry may take
static int64_t wg_partial_bytes(const ConvGeo &g) {
    WgPlan a = wg_plan(g, 4), b = wg_plan(g, 0), c = wg_plan(g, 4, true), e = wg_plan(g, 0, false, true);
    int64_t sp = std::max(a.ok ? a.splits : 0, b.ok ? b.splits : 0);
    sp = std::max(sp, (int64_t)(c.ok ? c.splits : 0));
    sp = std::max(sp, (int64_t)(e.ok ? e.splits : 0));
    for (int bits : {1, 2, 8}) {   // other code widths plan their own splits
        WgPlan q = wg_plan(g, bits);
        sp = std::max(sp, (int64_t)(q.ok ? q.splits : 0));
    }
    for (int bits : {2, 4}) {      // the pre-split pieces path
        WgPlan q = wg_plan(g, bits, false, false, true);
        sp = std::max(sp, (int64_t)(q.ok ? q.splits : 0));
    }
    return sp * g.co * g.ci * g.kh * g.kw * (int64_t)sizeof(float);
}

// direct (unsegmented) planes: the in-kernel split stays the default -- an
// extra pieces pass measured slower on every C2 layer (e.g. 64->16 1x1 at
// 32x32: 13.9 -> 18.9 us) and on the C4 56x56 layers; QTAPE_WG_PRE_DIRECT=1
// opts in
static bool wg_direct_pre_on() {
    static const bool on = [] {
        const char *e = getenv("QTAPE_WG_PRE_DIRECT");
        return e && *e && *e != '0';
    }();
    return on;
}

static bool wg_direct_pre(const ConvGeo &g, int bits) {
    if (!wg_direct_pre_on() || (g.oh * g.ow) % 32) return false;
    return wg_plan(g, bits, false, false, true).ok;
}

static int64_t wg_pieces_bytes(const ConvGeo &g) { return 6 * g.n * g.co * g.oh * g.ow; }

// 1-bit tapes whose planes are not 16-byte multiples (8x8: 8 bytes) cannot
// be boxed by TMA, but their 2-bit widening can: code c stays c and the
// offset becomes offset + 1, so m = 2c + 1 - 2^K + 2 offset and the fp64
// decode (c + 0.5 - 2^(K-1)) + offset are unchanged (codec.py:146-156).
static bool wg_widen1(const ConvGeo &g0, int bits) {
    const ConvGeo g = wg_flat_shape(g0) ? wg_flat_geo(g0) : g0;
    return bits == 1 && !wg_plan(g, 1).ok && wg_plan(g, 2).ok && g.n * g.ci * g.h * g.w / 16 < (1ll << 31);
}
static int64_t wg_widen1_bytes(const ConvGeo &g) {   // 2-bit codes + offset'
    return (g.n * g.ci * g.h * g.w / 4 + 255) / 256 * 256 + (g.ci * 8 + 255) / 256 * 256;
}

__global__ void widen_1to2_kernel(const uint16_t *codes1, uint32_t *codes2, uint32_t words,
                                  const int64_t *offset, int64_t *offset2, uint32_t c) {
    pdl_enter();
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    if (tid < c) offset2[tid] = offset[tid] + 1;
    for (uint32_t o = tid; o < words; o += gridDim.x * blockDim.x) {
        uint32_t x = __ldg(codes1 + o);       // 16 one-bit codes -> 16 two-bit codes
        x = (x | (x << 8)) & 0x00FF00FFu;
        x = (x | (x << 4)) & 0x0F0F0F0Fu;
        x = (x | (x << 2)) & 0x33333333u;
        x = (x | (x << 1)) & 0x55555555u;
        codes2[o] = x;
    }
}

int64_t qt_tc_wgrad_workspace(const qt::ConvGeo &g) {
    if (wg_flat_shape(g)) return qt_tc_wgrad_workspace(wg_flat_geo(g));
    if (wg_s2d_shape(g, 8)) {   // the 2x2/s2 rearranged-codes path (widest code width)
        const ConvGeo d = wg_s2d_geo(g);
        return wg_s2d_bytes(g, 8) + qt_tc_wgrad_workspace(d);
    }
    int64_t b = wg_partial_bytes(g);
    if (wg_direct_pre(g, 4) || wg_direct_pre(g, 2)) b = (b + 255) / 256 * 256 + wg_pieces_bytes(g);
    if (wg_widen1(g, 1)) b = std::max(b, (wg_partial_bytes(g) + 255) / 256 * 256 + wg_widen1_bytes(g));
    return b;
}

// partials only: the segmented path keeps its own planes behind them
int64_t qt_tc_wgrad_partial_workspace(const qt::ConvGeo &g) {
    return wg_partial_bytes(wg_flat_shape(g) ? wg_flat_geo(g) : g);
}

// debug hook (not part of the public ABI): buf = 600 + 3*1024 int64 stamps or NULL
static long long *g_wg_trace_host = nullptr;
static int g_wg_trace_cta_host = 0;
extern "C" int qt_debug_wgrad_trace(void *buf, int cta) {
    g_wg_trace_host = (long long *)buf;
    g_wg_trace_cta_host = cta;
    return QT_OK;
}

int qt_tc_wgrad_reduce(const float *partial, int64_t splits, int64_t count, float *grad_w,
                       cudaStream_t st) {
    if (splits <= 48) {
        launch_pdl(wgrad_reduce_few_kernel, (unsigned)std::min<int64_t>(qt_cdiv(count, 256), qt_sm_count() * 8),
                   256, 0, st, partial, (int)splits, count, grad_w);
        QT_CHECK_LAUNCH();
        return QT_OK;
    }
    launch_pdl(wgrad_reduce_kernel, (unsigned)qt_cdiv(count, 32), 1024, 0, st, partial, splits, count,
                                                                      grad_w);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

// gr: fp32 g_out, or (pieces != NULL) its bf16 pieces in the wg_pieces layout
static int wgrad_tc(const float *gr, const void *pieces, qt_tape_t act, const float *x_plain,
                    float *grad_w, const qt::ConvGeo &g0, void *ws, cudaStream_t st) {
    if (tcw_disabled()) return QT_EUNSUPPORTED;
    const ConvGeo g = wg_flat_shape(g0) ? wg_flat_geo(g0) : g0;
    const bool codes = !x_plain && !act.a2;
    if (pieces && (!codes || ((uintptr_t)pieces & 15))) return QT_EUNSUPPORTED;
    // 3x3 on 4-bit codes with the column taps in N: correct (tested) but not
    // yet faster than the (ci, u, v)-row form -- its g split triples -- so
    // opt-in with QTAPE_WG_TAP=1
    static const bool use_tap = [] {
        const char *e = getenv("QTAPE_WG_TAP");
        return e && *e && *e != '0';
    }();
    WgPlan pl{};
    if (pieces) {
        pl = wg_plan(g, act.bits, false, false, true);
        if (!pl.ok) return QT_EUNSUPPORTED;
    }
    if (!pl.ok && codes && use_tap) pl = wg_plan(g, act.bits, true);
    if (!pl.ok && !codes) pl = wg_plan(g, 0, false, true);   // fp32 rows staged by TMA
    if (!pl.ok) pl = wg_plan(g, codes ? act.bits : 0);
    if (!pl.ok) return QT_EUNSUPPORTED;
    if (codes && ((uintptr_t)act.codes & 15)) return QT_EUNSUPPORTED;
    auto enc = encode_fn_wg();
    if (!enc) return QT_EUNSUPPORTED;
    // g_out (n, co, oh*ow) as 3D (pixel, c, n) -- the (h, w) plane is contiguous
    // in NCHW; box = 32 consecutive pixels (one dense 128-byte SW128 row) x BN
    // channels.  (A box whose inner extent is shorter than the 128-byte
    // swizzle span is padded per row by TMA, so rows of 8/16 px cannot be
    // stacked into one swizzle row.)
    CUtensorMap m;
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    if (pieces) {
        // 5D (32 px, co, piece, chunk, n) bf16: one box = SUB chunks x 3
        // pieces x BN channels of 64-byte rows, SW64 -- the FAST B layout
        const cuuint64_t cpi = (cuuint64_t)(g.oh * g.ow / 32), row = 64;
        cuuint64_t dims[5] = {32, (cuuint64_t)g.co, 3, cpi, (cuuint64_t)g.n};
        cuuint64_t strides[4] = {row, row * g.co, row * g.co * 3, row * g.co * 3 * cpi};
        cuuint32_t box[5] = {32, (cuuint32_t)pl.bn, 3, (cuuint32_t)kWgSub, 1};
        if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void *>(pieces), dims, strides,
                box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return QT_EUNSUPPORTED;
    } else {
    // 4D (32 px, chunk, c, n): one box = SUB consecutive chunks x BN channels
    cuuint64_t dims[4] = {32, (cuuint64_t)(g.oh * g.ow / 32), (cuuint64_t)g.co, (cuuint64_t)g.n};
    cuuint64_t strides[3] = {128, (cuuint64_t)g.oh * g.ow * 4, (cuuint64_t)g.co * g.oh * g.ow * 4};
    cuuint32_t box[4] = {32, (cuuint32_t)kWgSub, (cuuint32_t)pl.bn, 1};
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void *)gr, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return QT_EUNSUPPORTED;
    }
    CUtensorMap mc = m;   // codes (n, ci, plane bytes) as 3D (byte, c, n)
    if (codes) {
        const int64_t plane = g.h * g.w * act.bits / 8;
        cuuint64_t cd[3] = {(cuuint64_t)plane, (cuuint64_t)g.ci, (cuuint64_t)g.n};
        cuuint64_t cs[2] = {(cuuint64_t)plane, (cuuint64_t)(plane * g.ci)};
        cuuint32_t cbx[3] = {(cuuint32_t)pl.cb, (cuuint32_t)pl.nch, 1};
        if (enc(&mc, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void *)act.codes, cd, cs, cbx, es + 1,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return QT_EUNSUPPORTED;
    } else if (pl.fbox) {   // fp32 source (n, ci, h*w) as 3D (pixel, c, n)
        const float *src = x_plain ? x_plain : act.a2;
        if ((uintptr_t)src & 15) return QT_EUNSUPPORTED;
        const int64_t plane = g.h * g.w;
        cuuint64_t cd[3] = {(cuuint64_t)plane, (cuuint64_t)g.ci, (cuuint64_t)g.n};
        cuuint64_t cs[2] = {(cuuint64_t)plane * 4, (cuuint64_t)(plane * g.ci * 4)};
        cuuint32_t cbx[3] = {(cuuint32_t)(pl.cb / 4), (cuuint32_t)pl.nch, 1};
        if (plane * 4 % 16 ||
            enc(&mc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void *)src, cd, cs, cbx, es + 1,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return QT_EUNSUPPORTED;
    }
    WgParams p{};
    p.tape = act;
    p.plain = x_plain;
    p.partial = (float *)ws;
    p.n = (int)g.n; p.ci = (int)g.ci; p.h = (int)g.h; p.w = (int)g.w; p.co = (int)g.co;
    p.kh = (int)g.kh; p.kw = (int)g.kw; p.pad = (int)g.pad; p.oh = (int)g.oh; p.ow = (int)g.ow;
    p.rpc = pl.rpc;
    p.trace = g_wg_trace_host;
    p.trace_cta = g_wg_trace_cta_host;
    p.R = (int)(g.ci * pl.rpc);
    p.Rout = (int)(g.ci * g.kh * g.kw);
    p.mtg = pl.mtg;
    p.rows_per_chunk = (int)(32 / g.ow);
    p.chunks_per_img = (int)(g.oh * g.ow / 32);
    p.cpid = make_fastdiv((uint32_t)p.chunks_per_img);
    p.total_chunks = pl.total;
    p.chunks_per_split = pl.cps;
    p.splits = pl.splits;
    p.RG = pl.rg;
    p.OPS = pl.ops;
    p.OPS_G = pl.ops_g;
    static const int fast2_env = [] {   // 0: m < 2048 channels take INT (tests)
        const char *e = getenv("QTAPE_WG_FAST2");
        return e ? atoi(e) : 1;
    }();
    p.OPS2 = fast2_env ? pl.ops2 : 0;
    p.opreg = pl.opreg;
    p.pre = pl.pre;
    p.RB = pl.bring;
    p.lut_floats = pl.lut_floats;
    p.nolut = pl.nolut;
    static const int int_env = [] {   // 0: wide channels take the table GENERIC (tests)
        const char *e = getenv("QTAPE_WG_INT");
        return e ? atoi(e) : 1;
    }();
    p.intok = int_env;
    p.slot = pl.slot;
    p.cb = pl.cb;
    p.cbytes = pl.cbytes;
    p.rb = pl.rb;
    p.lut = codes ? 1 : 0;
    p.fbox = pl.fbox;
    int rc;
    switch (pl.bn) {
        case 16: rc = wg_launch_bn16(m, mc, p, pl, st); break;
        case 32: rc = wg_launch_bn32(m, mc, p, pl, st); break;
        case 64: rc = wg_launch_bn64(m, mc, p, pl, st); break;
        case 128: rc = wg_launch_bn128(m, mc, p, pl, st); break;
        case 256: rc = wg_launch_bn256(m, mc, p, pl, st); break;
        default: return QT_EUNSUPPORTED;
    }
    if (rc) return rc;
    return qt_tc_wgrad_reduce((const float *)ws, pl.splits, g.co * p.Rout, grad_w, st);
}

int qt_tc_wgrad_pieces(const float *g, void *dst, int64_t n, int64_t co, int64_t h, int64_t w,
                       cudaStream_t st);

int qt_tc_conv_wgrad(const float *gr, qt_tape_t act, const float *x_plain, float *grad_w,
                     const qt::ConvGeo &g0, void *ws, cudaStream_t st) {
    const ConvGeo g = wg_flat_shape(g0) ? wg_flat_geo(g0) : g0;
    if (!x_plain && !act.a2 && act.codes && ws && wg_direct_pre(g, act.bits)) {
        void *pieces = (char *)ws + (wg_partial_bytes(g) + 255) / 256 * 256;
        int rc = qt_tc_wgrad_pieces(gr, pieces, g.n, g.co, g.oh, g.ow, st);
        if (rc) return rc;
        rc = wgrad_tc(nullptr, pieces, act, nullptr, grad_w, g, ws, st);
        if (rc != QT_EUNSUPPORTED) return rc;
    }
    if (!x_plain && !act.a2 && act.codes && ws && wg_widen1(g0, act.bits) &&
        ((g.n * g.ci * g.h * g.w) & 15) == 0 && ((uintptr_t)act.codes & 1) == 0) {
        char *base = (char *)ws + (wg_partial_bytes(g) + 255) / 256 * 256;
        uint32_t *codes2 = (uint32_t *)base;
        int64_t *offset2 = (int64_t *)(base + (g.n * g.ci * g.h * g.w / 4 + 255) / 256 * 256);
        const uint32_t words = (uint32_t)(g.n * g.ci * g.h * g.w / 16);
        const uint32_t need = std::max(words, (uint32_t)g.ci);
        const unsigned blocks = (unsigned)std::min<int64_t>(qt_cdiv(need, 256), qt_sm_count() * 8);
        launch_pdl(widen_1to2_kernel, blocks, 256, 0, st, (const uint16_t *)act.codes, codes2, words,
                   act.offset, offset2, (uint32_t)g.ci);
        QT_CHECK_LAUNCH();
        qt_tape_t t2 = act;
        t2.codes = (const uint8_t *)codes2;
        t2.offset = offset2;
        t2.bits = 2;
        return wgrad_tc(gr, nullptr, t2, nullptr, grad_w, g0, ws, st);
    }
    return wgrad_tc(gr, nullptr, act, x_plain, grad_w, g0, ws, st);
}

// the fp32 g_out path only (the segmented path's planes follow the partials)
int qt_tc_conv_wgrad_fp32(const float *gr, qt_tape_t act, const float *x_plain, float *grad_w,
                          const qt::ConvGeo &g, void *ws, cudaStream_t st) {
    return wgrad_tc(gr, nullptr, act, x_plain, grad_w, g, ws, st);
}

// weight gradient with g_out already split into bf16 pieces (wg_pieces layout)
int qt_tc_conv_wgrad_pre(const void *pieces, qt_tape_t act, float *grad_w, const qt::ConvGeo &g,
                         void *ws, cudaStream_t st) {
    return wgrad_tc(nullptr, pieces, act, nullptr, grad_w, g, ws, st);
}

// the pieces path is planned for this (32-px-row) geometry and code width
bool qt_tc_wgrad_pre_ok(const qt::ConvGeo &g, int bits) {
    if (tcw_disabled()) return false;
    static const bool off = [] {
        const char *e = getenv("QTAPE_WG_PRE");
        return e && *e == '0';
    }();
    return !off && wg_plan(wg_flat_shape(g) ? wg_flat_geo(g) : g, bits, false, false, true).ok;
}

// 2x2/s2 weight gradient from a packed code tape through the rearranged tape
int qt_tc_conv_wgrad_s2d(const float *gr, qt_tape_t act, float *grad_w, const qt::ConvGeo &g,
                         void *ws, cudaStream_t st) {
    if (tcw_disabled() || !act.codes || act.a2 || !wg_s2d_shape(g, act.bits)) return QT_EUNSUPPORTED;
    const ConvGeo d = wg_s2d_geo(g);
    if (!wg_plan(d, act.bits).ok) return QT_EUNSUPPORTED;
    if (((uintptr_t)act.codes & 3) || ((uintptr_t)ws & 255)) return QT_EUNSUPPORTED;
    uint8_t *base = (uint8_t *)ws;
    const int64_t cbytes = (g.n * g.ci * g.h * g.w * act.bits / 8 + 255) / 256 * 256;
    uint32_t *codes4 = (uint32_t *)base;
    double *step4 = (double *)(base + cbytes);
    int64_t *offset4 = (int64_t *)(base + cbytes + g.ci * 4 * 8);
    const uint32_t words = (uint32_t)(g.n * g.ci * g.h * g.w * act.bits / 32);
    const uint32_t per = 32u / (uint32_t)act.bits;
    const FastDiv wrd = make_fastdiv((uint32_t)(g.w / 2) / per), hd = make_fastdiv((uint32_t)(g.h / 2));
    const uint32_t c4 = (uint32_t)(g.ci * 4);
    const uint32_t need = std::max(words, c4);
    const unsigned blocks = (unsigned)std::min<int64_t>(qt_cdiv(need, 256), qt_sm_count() * 8);
    launch_pdl(codes_s2d_kernel, blocks, 256, 0, st, act.codes, codes4, words, (uint32_t)g.h,
               (uint32_t)g.w, act.bits, wrd, hd, act.step, act.offset, step4, offset4, c4);
    QT_CHECK_LAUNCH();
    qt_tape_t t4 = act;
    t4.codes = (const uint8_t *)codes4;
    t4.step = step4;
    t4.offset = offset4;
    return qt_tc_conv_wgrad(gr, t4, nullptr, grad_w, d, base + wg_s2d_bytes(g, act.bits), st);
}
