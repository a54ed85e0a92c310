// Weight gradient on the tensor cores with the activation operand decoded
// from the packed K-bit tape inside the operand staging.
//
//   dW[co][r = (ci,u,v)] += sum_{pixels p} act[ci][p shifted by (u,v)] * g[co][p]
//
// GEMM view: M = r (ci*kh*kw rows, 128-row tiles), N = co, K = output
// pixels (32 per stage = one 128-byte K-major SW128 row).  Per stage:
//   * TMA loads the g_out box (32 pixels x BN channels) straight from NCHW;
//     transform warps split it in place into TF32 (hi, lo) halves;
//   * transform warps build the activation tile: for each (ci, u) and pixel
//     quad they fetch 4 + 2*pad codes of the input row, decode them with the
//     frozen per-channel (step, offset) to the reference's fp32 interval
//     medians, apply the ReLU, split (hi, lo), and write the kw column-
//     shifted copies (the 3x3 halo / zero padding happens here) -- the fp32
//     activation never exists in HBM;
//   * one thread issues A_hi*G_hi + A_hi*G_lo + A_lo*G_hi (3xTF32).
// Split-K over CTAs (contiguous pixel ranges), fp32 partials, then a
// deterministic fixed-order float64 reduction into grad_w (layer.py:167).
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "tc_common.cuh"

namespace qt {

using namespace tc;

constexpr int kWgThreads = 320;   // w0 TMA, w1 MMA/TMEM, w2..w9 transform + epilogue

template <int BN>
struct WgCfg {
    static constexpr int G_BYTES = BN * 128;          // BN rows x 32 px fp32
    static constexpr int MT_BYTES = 128 * 128;        // one 128-row x 32-px tile
};

struct WgParams {
    qt_tape_t tape;          // codes (+step/offset) or a2 (relu) ...
    const float *plain;      // ... or the plain input (no relu)
    float *partial;          // [split][co][R]
    int n, ci, h, w, co, kh, kw, pad, oh, ow;
    int R;                   // ci*kh*kw
    int mtg;                 // 128-row M tiles per CTA (group)
    int rows_per_chunk;      // 32 / ow
    int chunks_per_img;      // oh*ow/32
    int total_chunks, chunks_per_split, splits;
    int stages;
    uint32_t tmem_cols;
    int lut_ch;              // >0: channels per CTA covered by the smem code table
};

constexpr int kWgLutEntries = 4096;   // (channels x 2^K) entries of (hi, lo) = 32 KiB

__device__ __forceinline__ float act_value(const WgParams &p, int nn, int c, int y, int x) {
    if (y < 0 || y >= p.h || x < 0 || x >= p.w) return 0.f;  // conv zero padding
    const int64_t i = (((int64_t)nn * p.ci + c) * p.h + y) * p.w + x;
    if (p.plain) return __ldg(p.plain + i);
    float a = p.tape.a2 ? __ldg(p.tape.a2 + i)
                        : decode(get_code(p.tape.codes, i, p.tape.bits), p.tape.step[c],
                                 p.tape.offset[c], p.tape.bits);
    return (a >= 0.f || isnan(a)) ? a : 0.f;  // ReLU as np.maximum (layer.py:356)
}

template <int BN, int KW>
__global__ void __launch_bounds__(kWgThreads, 1)
    conv_wgrad_tc_kernel(const __grid_constant__ CUtensorMap tmG, WgParams p) {
    using C = WgCfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int S = p.stages;
    const int stage_bytes = 2 * C::G_BYTES + 2 * p.mtg * C::MT_BYTES;
    uint64_t *full = (uint64_t *)(smem + S * stage_bytes);
    uint64_t *ready = full + S;
    uint64_t *empty = ready + S;
    uint64_t *done = empty + S;
    uint32_t *tmem_slot = (uint32_t *)(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int split = blockIdx.x;
    const int row0 = blockIdx.y * p.mtg * 128;        // first M row of this group
    const int nrows = min(p.mtg * 128, p.R - row0);
    const int mt_here = (nrows + 127) / 128;
    const int c_begin = row0 / (p.kh * p.kw);
    const int c_end = min(p.ci, (row0 + nrows + p.kh * p.kw - 1) / (p.kh * p.kw));
    const int k0 = split * p.chunks_per_split;
    const int k1 = min(p.total_chunks, k0 + p.chunks_per_split);
    const int nk = k1 - k0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&ready[s], 256);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(p.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (warp == 0 && lane == 0) tma_prefetch(&tmG);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    auto sGh = [&](int s) { return smem + s * stage_bytes; };
    auto sGl = [&](int s) { return smem + s * stage_bytes + C::G_BYTES; };
    auto sAh = [&](int s, int t) { return smem + s * stage_bytes + 2 * C::G_BYTES + t * C::MT_BYTES; };
    auto sAl = [&](int s, int t) {
        return smem + s * stage_bytes + 2 * C::G_BYTES + (p.mtg + t) * C::MT_BYTES;
    };

    if (warp == 0) {
        if (lane == 0) {  // ----------------------------- TMA producer (g_out)
            for (int i = 0; i < nk; ++i) {
                const int s = i % S;
                const uint32_t ph = (uint32_t)(i / S) & 1u;
                mbar_wait(&empty[s], ph ^ 1u);
                const int kc = k0 + i;
                const int nn = kc / p.chunks_per_img;
                const int y0 = (kc % p.chunks_per_img) * p.rows_per_chunk;
                mbar_expect_tx(&full[s], C::G_BYTES);
                tma_load_3d(sGh(s), &tmG, &full[s], y0 * p.ow, 0, nn);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // --------------------------------------- MMA issuer
            constexpr uint32_t idesc = instr_desc(128, BN, 2, 0, 0);
            for (int i = 0; i < nk; ++i) {
                const int s = i % S;
                const uint32_t ph = (uint32_t)(i / S) & 1u;
                mbar_wait(&ready[s], ph);
                tc_fence_after();
                const uint32_t gh = smem_u32(sGh(s)), gl = smem_u32(sGl(s));
                for (int t = 0; t < mt_here; ++t) {
                    const uint32_t ah = smem_u32(sAh(s, t)), al = smem_u32(sAl(s, t));
                    const uint32_t d = tmem + (uint32_t)(t * BN);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint64_t dah = smem_desc(ah + j * 32, 16, 1024, 2);
                        const uint64_t dal = smem_desc(al + j * 32, 16, 1024, 2);
                        const uint64_t dgh = smem_desc(gh + j * 32, 16, 1024, 2);
                        const uint64_t dgl = smem_desc(gl + j * 32, 16, 1024, 2);
                        mma_tf32(d, dah, dgh, idesc, (i | j) ? 1u : 0u);
                        mma_tf32(d, dah, dgl, idesc, 1u);
                        mma_tf32(d, dal, dgh, idesc, 1u);
                    }
                }
                mma_commit(&empty[s]);
            }
            mma_commit(done);
        }
    } else {  // ------------------------------ warps 2..9: transform + epilogue
        const int t = threadIdx.x - 64;  // 0..255
        const int kk = p.kh * p.kw;
        const int quads_per_chunk = 8;    // 32 px / 4
        const int tasks = (c_end - c_begin) * p.kh * quads_per_chunk;
        // per-CTA code table: relu(decode(code)) of every channel in range,
        // pre-split into TF32 (hi, lo) -- exactly the reference's fp32 a3
        float *s_lut = reinterpret_cast<float *>(smem + S * stage_bytes + 1024);
        const bool use_lut = p.lut_ch > 0;
        if (use_lut) {
            const int nc = c_end - c_begin, ncode = 1 << p.tape.bits;
            for (int e = t; e < nc * ncode; e += 256) {
                const int c = c_begin + e / ncode, code = e % ncode;
                float a = decode((uint32_t)code, p.tape.step[c], p.tape.offset[c], p.tape.bits);
                a = (a >= 0.f || isnan(a)) ? a : 0.f;
                split_tf32(a, s_lut[2 * e], s_lut[2 * e + 1]);
            }
            // the 8 transform warps sync among themselves (named barrier 1)
            asm volatile("bar.sync 1, 256;" ::: "memory");
        }
        for (int i = 0; i < nk; ++i) {
            const int s = i % S;
            const uint32_t ph = (uint32_t)(i / S) & 1u;
            mbar_wait(&full[s], ph);
            const int kc = k0 + i;
            const int nn = kc / p.chunks_per_img;
            const int y0 = (kc % p.chunks_per_img) * p.rows_per_chunk;
            // g tile: in-place TF32 split (layout preserving)
            {
                float4 *gh = reinterpret_cast<float4 *>(sGh(s));
                float4 *gl = reinterpret_cast<float4 *>(sGl(s));
                for (int q = t; q < C::G_BYTES / 16; q += 256) {
                    float4 x = gh[q], hi, lo;
                    split_tf32(x.x, hi.x, lo.x);
                    split_tf32(x.y, hi.y, lo.y);
                    split_tf32(x.z, hi.z, lo.z);
                    split_tf32(x.w, hi.w, lo.w);
                    gh[q] = hi;
                    gl[q] = lo;
                }
            }
            // activation tile rows (ci,u,v) x 32 output pixels of this chunk
            for (int task = t; task < tasks; task += 256) {
                const int q = task % quads_per_chunk;
                const int cu = task / quads_per_chunk;
                const int c = c_begin + cu / p.kh, u = cu % p.kh;
                const int pix = q * 4;                           // pixel within chunk
                const int oy = y0 + pix / p.ow, ox0 = pix % p.ow;
                const int iy = oy + u - p.pad;
                constexpr int span = 4 + KW - 1;                 // 4 px + halo
                float vh[span], vl[span];
                if (iy < 0 || iy >= p.h) {
#pragma unroll
                    for (int e = 0; e < span; ++e) vh[e] = vl[e] = 0.f;
                } else if (use_lut) {
                    // codes of the 4 core pixels in one aligned load, halo codes apart
                    const int64_t rowi = (((int64_t)nn * p.ci + c) * p.h + iy) * p.w;
                    const int64_t i0 = rowi + ox0;               // multiple of 4
                    const int bits = p.tape.bits;
                    uint32_t w4;
                    if (bits == 4) w4 = *reinterpret_cast<const uint16_t *>(p.tape.codes + (i0 >> 1));
                    else if (bits == 2) w4 = p.tape.codes[i0 >> 2];
                    else w4 = (uint32_t)(p.tape.codes[i0 >> 3] >> (i0 & 7));
                    const float *lh = s_lut + (c - c_begin) * (2 << bits);
                    const uint32_t cm = (1u << bits) - 1u;
#pragma unroll
                    for (int e = 0; e < span; ++e) {
                        const int x = ox0 + e - p.pad;
                        uint32_t code;
                        bool inb = x >= 0 && x < p.w;
                        if (e >= p.pad && e < p.pad + 4) code = (w4 >> ((e - p.pad) * bits)) & cm;
                        else code = inb ? get_code(p.tape.codes, rowi + x, bits) : 0u;
                        vh[e] = inb ? lh[2 * code] : 0.f;
                        vl[e] = inb ? lh[2 * code + 1] : 0.f;
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < span; ++e)
                        split_tf32(act_value(p, nn, c, iy, ox0 + e - p.pad), vh[e], vl[e]);
                }
#pragma unroll
                for (int v = 0; v < KW; ++v) {
                    const int r = (c * p.kh + u) * KW + v - row0;  // local row
                    if (r < 0 || r >= nrows) continue;
                    const int tt = r >> 7, rr = r & 127;
                    const uint32_t off = swz_off<128>((uint32_t)(rr >> 3) * 1024 +
                                                      (uint32_t)(rr & 7) * 128 + (uint32_t)q * 16);
                    *reinterpret_cast<float4 *>(sAh(s, tt) + off) =
                        make_float4(vh[v], vh[v + 1], vh[v + 2], vh[v + 3]);
                    *reinterpret_cast<float4 *>(sAl(s, tt) + off) =
                        make_float4(vl[v], vl[v + 1], vl[v + 2], vl[v + 3]);
                }
            }
            (void)kk;
            fence_async_smem();
            mbar_arrive(&ready[s]);
        }
        // epilogue: warps 2..5 -> M tile 0, 6..9 -> M tile 1, ... (lanes 32*(warp%4))
        mbar_wait(done, 0);
        tc_fence_after();
        const int quarter = warp & 3;
        const int tgrp = (warp - 2) >> 2;      // 0 or 1
        for (int tl = tgrp; tl < mt_here; tl += 2) {
            const int r = tl * 128 + 32 * quarter + lane;    // local row
            const int rg = row0 + r;
            const uint32_t tbase = tmem + ((uint32_t)(32 * quarter) << 16) + (uint32_t)(tl * BN);
            for (int cb = 0; cb < BN; cb += 16) {
                uint32_t rv[16];
                tmem_ld16(tbase + cb, rv);
                tmem_wait_ld();
                if (r < nrows && nk > 0) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int co = cb + j;
                        if (co < p.co)
                            p.partial[((int64_t)split * p.co + co) * p.R + rg] = __uint_as_float(rv[j]);
                    }
                }
            }
            if (nk == 0 && r < nrows)
                for (int co = 0; co < p.co; ++co) p.partial[((int64_t)split * p.co + co) * p.R + rg] = 0.f;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(p.tmem_cols)
                     : "memory");
    }
}

// grad_w[i] = fp32(grad_w[i] + fp32(sum_z partial[z][i])) -- the 8 warps of
// a block sum interleaved split subsets for 32 consecutive outputs, then
// combine in warp order: fixed order, deterministic (layer.py:167).
__global__ void __launch_bounds__(1024) wgrad_reduce_kernel(const float *partial, int64_t splits,
                                                           int64_t count, float *grad_w) {
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

struct WgPlan {
    bool ok = false;
    int bn = 0, mtg = 0, mgroups = 0, splits = 0, cps = 0, total = 0, stages = 0, smem = 0;
    uint32_t cols = 0;
};

static WgPlan wg_plan(const ConvGeo &g) {
    WgPlan pl;
    if (g.s != 1) return pl;
    const int64_t ow = g.ow, oh = g.oh;
    if (ow != 8 && ow != 16 && ow != 32) return pl;
    if ((oh * ow) % 32 || oh % (32 / ow)) return pl;
    if (g.co % 16 || g.co > 256 || !(g.kw == 1 || g.kw == 3) || g.pad > 1) return pl;
    if (g.kw == 1 && g.pad != 0) return pl;
    if (g.n * oh * ow / 32 > INT32_MAX) return pl;
    pl.bn = g.co <= 16 ? 16 : g.co <= 32 ? 32 : g.co <= 64 ? 64 : g.co <= 128 ? 128 : 256;
    if (g.co % pl.bn) return pl;
    const int64_t R = g.ci * g.kh * g.kw;
    const int64_t mt = (R + 127) / 128;
    int mtg = (int)std::min<int64_t>(mt, pl.bn >= 256 ? 2 : 3);
    while (mtg > 1 && mtg * pl.bn > 512) --mtg;
    // smem: stages x (g hi/lo + mtg x (a hi/lo) x 16 KiB)
    int stage = 2 * pl.bn * 128 + 2 * mtg * 128 * 128;
    while (mtg > 1 && 2 * stage > 200 * 1024) {
        --mtg;
        stage = 2 * pl.bn * 128 + 2 * mtg * 128 * 128;
    }
    pl.mtg = mtg;
    pl.mgroups = (int)((mt + mtg - 1) / mtg);
    pl.stages = std::max(1, std::min(4, (190 * 1024) / stage));
    pl.smem = pl.stages * stage + 1024 + 1024 + kWgLutEntries * 8;
    uint32_t cols = 32;
    while (cols < (uint32_t)(mtg * pl.bn)) cols <<= 1;
    pl.cols = cols;
    pl.total = (int)(g.n * oh * ow / 32);
    // split-K count: enough CTAs to cover the SMs twice, but the fp32
    // partials (splits x R x co x 4 B) must stay well below the operand
    // bytes the split reads (g: 128*co B and codes per 32-pixel chunk).
    int want = std::max(1, (2 * 148) / pl.mgroups);
    const double chunk_bytes = 128.0 * g.co + 32.0 * g.ci * 1.0;
    const double part_bytes = 4.0 * R * g.co;
    const int cap = std::max(48, (int)(4.0 * pl.total * chunk_bytes / part_bytes));
    want = std::min(want, cap);
    pl.cps = std::max(1, (pl.total + want - 1) / want);
    pl.splits = (pl.total + pl.cps - 1) / pl.cps;
    pl.ok = true;
    return pl;
}

template <int BN, int KW>
static int launch_wg(const CUtensorMap &m, const WgParams &p, const WgPlan &pl, cudaStream_t st) {
    auto kern = conv_wgrad_tc_kernel<BN, KW>;
    static int attr = 0;
    if (attr < pl.smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = 227 * 1024;
    }
    kern<<<dim3(pl.splits, pl.mgroups), kWgThreads, pl.smem, st>>>(m, p);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

}  // namespace qt

using namespace qt;

static bool tcw_disabled() {
    const char *e = getenv("QTAPE_NO_TC");
    return e && *e && *e != '0';
}

int64_t qt_tc_wgrad_workspace(const qt::ConvGeo &g) {
    WgPlan pl = wg_plan(g);
    if (!pl.ok) return 0;
    return (int64_t)pl.splits * g.co * g.ci * g.kh * g.kw * (int64_t)sizeof(float);
}

int qt_tc_wgrad_reduce(const float *partial, int64_t splits, int64_t count, float *grad_w,
                       cudaStream_t st) {
    wgrad_reduce_kernel<<<(unsigned)qt_cdiv(count, 32), 1024, 0, st>>>(partial, splits, count,
                                                                      grad_w);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

int qt_tc_conv_wgrad(const float *gr, qt_tape_t act, const float *x_plain, float *grad_w,
                     const qt::ConvGeo &g, void *ws, cudaStream_t st) {
    if (tcw_disabled()) return QT_EUNSUPPORTED;
    WgPlan pl = wg_plan(g);
    if (!pl.ok) return QT_EUNSUPPORTED;
    auto enc = encode_fn_wg();
    if (!enc) return QT_EUNSUPPORTED;
    // g_out (n, co, oh*ow) as 3D (pixel, c, n) -- the (h, w) plane is contiguous
    // in NCHW; box = 32 consecutive pixels (one dense 128-byte SW128 row) x BN
    // channels.  (A box whose inner extent is shorter than the 128-byte
    // swizzle span is padded per row by TMA, so rows of 8/16 px cannot be
    // stacked into one swizzle row.)
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)(g.oh * g.ow), (cuuint64_t)g.co, (cuuint64_t)g.n};
    cuuint64_t strides[2] = {(cuuint64_t)g.oh * g.ow * 4, (cuuint64_t)g.co * g.oh * g.ow * 4};
    cuuint32_t box[3] = {32, (cuuint32_t)pl.bn, 1};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void *)gr, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return QT_EUNSUPPORTED;
    WgParams p{};
    p.tape = act;
    p.plain = x_plain;
    p.partial = (float *)ws;
    p.n = (int)g.n; p.ci = (int)g.ci; p.h = (int)g.h; p.w = (int)g.w; p.co = (int)g.co;
    p.kh = (int)g.kh; p.kw = (int)g.kw; p.pad = (int)g.pad; p.oh = (int)g.oh; p.ow = (int)g.ow;
    p.R = (int)(g.ci * g.kh * g.kw);
    p.mtg = pl.mtg;
    p.rows_per_chunk = (int)(32 / g.ow);
    p.chunks_per_img = (int)(g.oh * g.ow / 32);
    p.total_chunks = pl.total;
    p.chunks_per_split = pl.cps;
    p.splits = pl.splits;
    p.stages = pl.stages;
    p.tmem_cols = pl.cols;
    {
        // smem code table when every CTA's channel range fits (K <= 4)
        const int kk = (int)(g.kh * g.kw);
        const int max_ch = (pl.mtg * 128 + kk - 1) / kk + (kk > 1 ? 1 : 0);
        p.lut_ch = (!x_plain && !act.a2 && act.bits <= 4 && max_ch * (1 << act.bits) <= kWgLutEntries)
                       ? max_ch : 0;
    }
    int rc;
#define QT_WG_CASES(KW)                                          \
    switch (pl.bn) {                                             \
        case 16: rc = launch_wg<16, KW>(m, p, pl, st); break;    \
        case 32: rc = launch_wg<32, KW>(m, p, pl, st); break;    \
        case 64: rc = launch_wg<64, KW>(m, p, pl, st); break;    \
        case 128: rc = launch_wg<128, KW>(m, p, pl, st); break;  \
        case 256: rc = launch_wg<256, KW>(m, p, pl, st); break;  \
        default: return QT_EUNSUPPORTED;                         \
    }
    if (g.kw == 1) {
        QT_WG_CASES(1)
    } else {
        QT_WG_CASES(3)
    }
#undef QT_WG_CASES
    if (rc) return rc;
    return qt_tc_wgrad_reduce((const float *)ws, pl.splits, g.co * p.R, grad_w, st);
}
