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

constexpr int kTcThreads = 192;

template <int BN, int OWT, int KC, int KW>
struct FwdCfg {
    static constexpr int BM = 128;
    static constexpr int A_BYTES = BM * KC * 4;                     // one tap's K-chunk
    static constexpr int B_BYTES = BN * KC * 4;
    static constexpr int B_SLOT = (B_BYTES + 1023) / 1024 * 1024;   // keep every tile 1 KiB aligned
    // raw activation box (TMA, MN-major) + KW taps x (hi, lo) K-major + KW x weights (hi, lo)
    static constexpr int STAGE_BYTES = A_BYTES * (1 + 2 * KW) + 2 * KW * B_SLOT;
    static constexpr int S0 = (200 * 1024) / STAGE_BYTES;
    static constexpr int S_MAX = S0 > 4 ? 4 : (S0 < 1 ? 1 : S0);
    static constexpr int OUT_BYTES = BM * BN * 4;                   // output staging tile
    static int smem_bytes(int stages) { return stages * STAGE_BYTES + OUT_BYTES + 1024 + 256; }
    static constexpr uint32_t TMEM_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
    static constexpr int A_SW = OWT * 4;     // swizzle bytes of the raw activation box
    static constexpr int K_SW = KC * 4;      // swizzle bytes of the K-major operand tiles
};

struct FwdGeo {
    int n, ci, h, w, co, kh, kw, pad, oh, ow;
    int rows, nimg, tiles_per_img;  // tile = nimg images x rows x OW pixels
    int stages;                     // smem ring depth (<= the K loop length)
};

struct EpiParams {
    float *out;
    const float *res;
    int cr, sr;
    int res_tma;   // 1: residual tile TMA-loaded into the output staging buffer
};

// One CTA = one 128-pixel x BN-channel output tile.  K loop: for each kernel
// row u and channel chunk: ONE TMA box of KC channels x (rows of the tile
// shifted by u) whole image rows; the KW column taps v are produced from it
// by the transform warps (TMA cannot start a tile at an unaligned innermost
// coordinate, so the +-1 column shift and its zero padding happen in smem).
template <int BN, int OWT, int KC, int KW>
__global__ void __launch_bounds__(kTcThreads, 2)
    conv_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmA,
                       const __grid_constant__ CUtensorMap tmBh,
                       const __grid_constant__ CUtensorMap tmBl,
                       const __grid_constant__ CUtensorMap tmOut,
                       const __grid_constant__ CUtensorMap tmRes, FwdGeo g, EpiParams ep) {
    using C = FwdCfg<BN, OWT, KC, KW>;
    const int S = g.stages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    // output staging tile [nimg][BN][rows][OWT] fp32 (TMA-store box layout)
    float *s_out = (float *)(smem + S * C::STAGE_BYTES);
    uint64_t *full = (uint64_t *)(smem + S * C::STAGE_BYTES + C::OUT_BYTES);
    uint64_t *ready = full + S;
    uint64_t *empty = ready + S;
    uint64_t *done = empty + S;
    uint64_t *resbar = done + 1;
    uint32_t *tmem_slot = (uint32_t *)(resbar + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile = blockIdx.x;
    const int co0 = blockIdx.y * BN;
    const int n0 = (g.nimg > 1) ? tile * g.nimg : tile / g.tiles_per_img;
    const int h0 = (g.nimg > 1) ? 0 : (tile % g.tiles_per_img) * g.rows;
    const int kchunks = g.ci / KC;
    const int nstages = g.kh * kchunks;     // (u, channel chunk) pairs

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&ready[s], 128);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        mbar_init(resbar, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<C::TMEM_COLS>(tmem_slot);
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmBh);
        tma_prefetch(&tmBl);
        tma_prefetch(&tmOut);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    auto sRaw = [&](int s) { return smem + s * C::STAGE_BYTES; };
    auto sAh = [&](int s, int v) { return smem + s * C::STAGE_BYTES + (1 + v) * C::A_BYTES; };
    auto sAl = [&](int s, int v) { return smem + s * C::STAGE_BYTES + (1 + KW + v) * C::A_BYTES; };
    auto sBh = [&](int s, int v) {
        return smem + s * C::STAGE_BYTES + (1 + 2 * KW) * C::A_BYTES + v * C::B_SLOT;
    };
    auto sBl = [&](int s, int v) {
        return smem + s * C::STAGE_BYTES + (1 + 2 * KW) * C::A_BYTES + (KW + v) * C::B_SLOT;
    };

    if (warp == 0) {
        if (lane == 0) {  // ---------------------------------- TMA producer
            if (ep.res_tma) {  // shortcut tile straight into the output staging buffer
                mbar_expect_tx(resbar, C::OUT_BYTES);
                tma_load_4d(s_out, &tmRes, resbar, 0, h0, co0, n0);
            }
            for (int i = 0; i < nstages; ++i) {
                const int s = i % S;
                const uint32_t ph = (uint32_t)(i / S) & 1u;
                mbar_wait(&empty[s], ph ^ 1u);
                const int u = i / kchunks, c0 = (i % kchunks) * KC;
                mbar_expect_tx(&full[s], C::A_BYTES + 2 * KW * C::B_BYTES);
                tma_load_4d(sRaw(s), &tmA, &full[s], 0, c0, h0 + u - g.pad, n0);
#pragma unroll
                for (int v = 0; v < KW; ++v) {
                    const int kcol = (u * g.kw + v) * g.ci + c0;
                    tma_load_2d(sBh(s, v), &tmBh, &full[s], kcol, co0);
                    tma_load_2d(sBl(s, v), &tmBl, &full[s], kcol, co0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ----------------------------------- MMA issuer
            constexpr uint32_t idesc = instr_desc(128, BN, 2, 0, 0);   // both K-major
            constexpr uint32_t k_sbo = 8 * KC * 4;        // stride between 8-row groups
            constexpr uint32_t lay = swizzle_layout(C::K_SW);
            for (int i = 0; i < nstages; ++i) {
                const int s = i % S;
                const uint32_t ph = (uint32_t)(i / S) & 1u;
                mbar_wait(&ready[s], ph);
                tc_fence_after();
#pragma unroll
                for (int v = 0; v < KW; ++v) {
                    const uint32_t ah = smem_u32(sAh(s, v)), al = smem_u32(sAl(s, v));
                    const uint32_t bh = smem_u32(sBh(s, v)), bl = smem_u32(sBl(s, v));
#pragma unroll
                    for (int j = 0; j < KC / 8; ++j) {
                        const uint64_t dah = smem_desc(ah + j * 32, 16, k_sbo, lay);
                        const uint64_t dal = smem_desc(al + j * 32, 16, k_sbo, lay);
                        const uint64_t dbh = smem_desc(bh + j * 32, 16, k_sbo, lay);
                        const uint64_t dbl = smem_desc(bl + j * 32, 16, k_sbo, lay);
                        mma_tf32(tmem, dah, dbh, idesc, (i | v | j) ? 1u : 0u);
                        mma_tf32(tmem, dah, dbl, idesc, 1u);
                        mma_tf32(tmem, dal, dbh, idesc, 1u);
                    }
                }
                mma_commit(&empty[s]);
            }
            mma_commit(done);
        }
    } else {  // ---------------------------- warps 2..5: split, then epilogue
        const int t = threadIdx.x - 64;  // 0..127 = tile row (output pixel)
        const uint32_t atom = (uint32_t)(t / OWT);
        const int px = t % OWT;
        const int kw_pad = (KW > 1) ? g.pad : 0;
        for (int i = 0; i < nstages; ++i) {
            const int s = i % S;
            const uint32_t ph = (uint32_t)(i / S) & 1u;
            mbar_wait(&full[s], ph);
            const uint8_t *raw = sRaw(s);
#pragma unroll
            for (int v = 0; v < KW; ++v) {
                // column tap v reads pixel px + v - pad of the same image row
                const int sx = px + v - kw_pad;
                const bool inb = sx >= 0 && sx < OWT;
                uint8_t *ah = sAh(s, v), *al = sAl(s, v);
#pragma unroll
                for (int q = 0; q < KC / 4; ++q) {
                    float xv[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t c = 4 * q + j;
                        const uint32_t off = (atom * KC + c) * (OWT * 4) + (uint32_t)sx * 4;
                        xv[j] = inb ? *reinterpret_cast<const float *>(raw + swz_off<C::A_SW>(off))
                                    : 0.f;
                    }
                    float4 hi, lo;
                    split_tf32(xv[0], hi.x, lo.x);
                    split_tf32(xv[1], hi.y, lo.y);
                    split_tf32(xv[2], hi.z, lo.z);
                    split_tf32(xv[3], hi.w, lo.w);
                    const uint32_t koff = swz_off<C::K_SW>((uint32_t)(t / 8) * (8 * KC * 4) +
                                                           (uint32_t)(t % 8) * (KC * 4) + q * 16);
                    *reinterpret_cast<float4 *>(ah + koff) = hi;
                    *reinterpret_cast<float4 *>(al + koff) = lo;
                }
            }
            fence_async_smem();
            mbar_arrive(&ready[s]);
        }
        // epilogue: this warp owns TMEM lanes 32*(warp%4) .. +31 = tile rows
        mbar_wait(done, 0);
        tc_fence_after();
        const int row = 32 * (warp & 3) + lane;
        const int ratom = row / OWT, wcol = row % OWT;
        const int img = ratom / g.rows, rr = ratom % g.rows;
        const int nn = n0 + img, y = h0 + rr;
        const uint32_t tbase = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
        // staging index of (channel j, this pixel): [img][BN][rows][OWT]
        float *so = s_out + ((size_t)img * BN * g.rows + rr) * OWT + wcol;
        const size_t cstride = (size_t)g.rows * OWT;
        if (ep.res_tma) mbar_wait(resbar, 0);
        const bool res_ldg = ep.res && !ep.res_tma;
#pragma unroll 1
        for (int cb = 0; cb < BN; cb += 16) {
            float rv[16];
            if (res_ldg) {  // strided shortcut (sr > 1): gather, all loads in flight
                const int64_t hr = (int64_t)g.oh * ep.sr, wr = (int64_t)g.ow * ep.sr;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int co = co0 + cb + j;
                    rv[j] = co < ep.cr ? __ldg(ep.res + (((int64_t)nn * ep.cr + co) * hr +
                                                         (int64_t)y * ep.sr) * wr +
                                                (int64_t)wcol * ep.sr)
                                       : 0.f;
                }
            }
            uint32_t r[16];
            tmem_ld16(tbase + cb, r);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                float v = __uint_as_float(r[j]);
                float *dst = so + (size_t)(cb + j) * cstride;
                // out = fp32(conv); cur += shortcut(res)  (engine.py:262-269)
                if (ep.res_tma) {
                    if (co0 + cb + j < ep.cr) v = __fadd_rn(v, *dst);
                } else if (res_ldg && co0 + cb + j < ep.cr) {
                    v = __fadd_rn(v, rv[j]);
                }
                *dst = v;
            }
        }
        fence_async_smem();
        asm volatile("bar.sync 1, 128;" ::: "memory");   // the 4 epilogue warps
        if (threadIdx.x == 64) {
            tma_store_4d(&tmOut, s_out, 0, h0, co0, n0);
            bulk_commit();
            bulk_wait_read0();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<C::TMEM_COLS>(tmem);
    }
}

// Weight prep: B[co'][(u,v)*ci' + c] = hi/lo of W[co'][c][u][v] (forward) or of
// W[c][co'][kh-1-u][kw-1-v] (data gradient: transposed + flipped kernel).
__global__ void weight_prep_kernel(const float *w, int co_n, int ci_n, int kh, int kw, int flip,
                                   float *bhi, float *blo) {
    // output rows co' (co_n of them), K' = kh*kw*ci_n
    const int kk = kh * kw;
    const int64_t total = (int64_t)co_n * kk * ci_n;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(idx % ci_n);
        const int uv = (int)((idx / ci_n) % kk);
        const int o = (int)(idx / ((int64_t)ci_n * kk));
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

static bool make_map_act(CUtensorMap *m, const float *x, const FwdGeo &g, int owt, int kc) {
    auto enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[4] = {(cuuint64_t)g.w, (cuuint64_t)g.ci, (cuuint64_t)g.h, (cuuint64_t)g.n};
    cuuint64_t strides[3] = {(cuuint64_t)g.h * g.w * 4, (cuuint64_t)g.w * 4,
                             (cuuint64_t)g.ci * g.h * g.w * 4};
    cuuint32_t box[4] = {(cuuint32_t)owt, (cuuint32_t)kc, (cuuint32_t)g.rows, (cuuint32_t)g.nimg};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void *)x, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, swz(owt * 4), CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool make_map_w(CUtensorMap *m, const float *b, int rows, int kdim, int bn, int kc) {
    auto enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)kdim, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)kdim * 4};
    cuuint32_t box[2] = {(cuuint32_t)kc, (cuuint32_t)bn};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)b, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, swz(kc * 4), CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct Maps {
    CUtensorMap a, bh, bl, out, res;
};

template <int BN, int OWT, int KC, int KW>
static int launch_fwd(const Maps &m, const FwdGeo &g, const EpiParams &ep, int tiles, int ntiles,
                      cudaStream_t st) {
    using C = FwdCfg<BN, OWT, KC, KW>;
    auto kern = conv_fwd_tc_kernel<BN, OWT, KC, KW>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = true;
    }
    // ring depth: no deeper than the K loop, and small enough that 2+ CTAs
    // share an SM (one CTA's epilogue / prologue overlaps another's mainloop)
    FwdGeo gg = g;
    const int nst = g.kh * (g.ci / KC);
    int S = std::min(nst, C::S_MAX);
    while (S > 1 && C::smem_bytes(S) > 112 * 1024) --S;
    gg.stages = S;
    kern<<<dim3(tiles, ntiles), kTcThreads, C::smem_bytes(S), st>>>(m.a, m.bh, m.bl, m.out, m.res,
                                                                   gg, ep);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

template <int OWT, int KC, int KW>
static int dispatch_bn(int bn, const Maps &m, const FwdGeo &g, const EpiParams &ep, int tiles,
                       int ntiles, cudaStream_t st) {
    switch (bn) {
        case 16: return launch_fwd<16, OWT, KC, KW>(m, g, ep, tiles, ntiles, st);
        case 32: return launch_fwd<32, OWT, KC, KW>(m, g, ep, tiles, ntiles, st);
        case 64: return launch_fwd<64, OWT, KC, KW>(m, g, ep, tiles, ntiles, st);
        case 128: return launch_fwd<128, OWT, KC, KW>(m, g, ep, tiles, ntiles, st);
        default: return QT_EUNSUPPORTED;
    }
}

template <int OWT>
static int dispatch_kc(int kc, int kw, int bn, const Maps &m, const FwdGeo &g,
                       const EpiParams &ep, int tiles, int ntiles, cudaStream_t st) {
    if (kw == 1) {
        switch (kc) {
            case 8: return dispatch_bn<OWT, 8, 1>(bn, m, g, ep, tiles, ntiles, st);
            case 16: return dispatch_bn<OWT, 16, 1>(bn, m, g, ep, tiles, ntiles, st);
            case 32: return dispatch_bn<OWT, 32, 1>(bn, m, g, ep, tiles, ntiles, st);
        }
    } else if (kw == 3) {
        switch (kc) {
            case 8: return dispatch_bn<OWT, 8, 3>(bn, m, g, ep, tiles, ntiles, st);
            case 16: return dispatch_bn<OWT, 16, 3>(bn, m, g, ep, tiles, ntiles, st);
        }
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

// Shape predicate of the tensor-core path (also used by qt_conv_uses_tc).
static bool tc_shape_ok(int n, int ci, int h, int wd, int co, int kh, int kw, int pad) {
    const int oh = h + 2 * pad - kh + 1, ow = wd + 2 * pad - kw + 1;
    if (kw != 1 && kw != 3) return false;
    if (kw == 1 && pad != 0) return false;
    if (ow != 8 && ow != 16 && ow != 32) return false;
    if (ow != wd || ci % 8 || co % 16 || ci < 8) return false;
    const int per = 128 / ow;
    if (oh >= per) return oh % per == 0;
    return per % oh == 0 && n % (per / oh) == 0;
}

// Runs out = conv_s1(x, W') with W' the (possibly transposed+flipped) kernel.
// x: (n, ci, h, w); out: (n, co, oh, ow); weights w in the ORIGINAL layout.
static int tc_conv_s1(const float *x, const float *w, float *out, int n, int ci, int h, int wd,
                      int co, int kh, int kw, int pad, int flip, const float *res, int cr, int sr,
                      void *ws, cudaStream_t st) {
    FwdGeo g{};
    g.n = n; g.ci = ci; g.h = h; g.w = wd; g.co = co; g.kh = kh; g.kw = kw; g.pad = pad;
    g.oh = h + 2 * pad - kh + 1;
    g.ow = wd + 2 * pad - kw + 1;
    if (!tc_shape_ok(n, ci, h, wd, co, kh, kw, pad)) return QT_EUNSUPPORTED;
    const int per = 128 / g.ow;                         // rows per 128-pixel tile
    if (g.oh >= per) {
        if (g.oh % per) return QT_EUNSUPPORTED;
        g.rows = per; g.nimg = 1; g.tiles_per_img = g.oh / per;
    } else {
        if (per % g.oh || n % (per / g.oh)) return QT_EUNSUPPORTED;
        g.rows = g.oh; g.nimg = per / g.oh; g.tiles_per_img = 1;
    }
    const int kcmax = kw == 1 ? 32 : 16;
    const int kc = ci % kcmax == 0 ? kcmax : (ci % 16 == 0 ? 16 : 8);
    int bn = co <= 16 ? 16 : (co <= 32 ? 32 : (co <= 64 ? 64 : 128));
    if (co % bn) return QT_EUNSUPPORTED;
    const int kdim = kh * kw * ci;
    float *bhi = (float *)ws;
    float *blo = bhi + (int64_t)co * kdim;
    if (!ws) return QT_EINVAL;
    weight_prep_kernel<<<(unsigned)std::min<int64_t>(qt_cdiv((int64_t)co * kdim, 256), 1024), 256, 0,
                         st>>>(w, co, ci, kh, kw, flip, bhi, blo);
    QT_CHECK_LAUNCH();
    Maps mp;
    if (!make_map_act(&mp.a, x, g, g.ow, kc) || !make_map_w(&mp.bh, bhi, co, kdim, bn, kc) ||
        !make_map_w(&mp.bl, blo, co, kdim, bn, kc) ||
        !make_map_nchw(&mp.out, out, n, co, g.oh, g.ow, g.rows, bn, g.nimg))
        return QT_EUNSUPPORTED;
    EpiParams ep{out, res, cr, sr, 0};
    if (res && sr == 1) {  // same-resolution shortcut: one TMA box per tile (OOB channels -> 0)
        if (!make_map_nchw(&mp.res, res, n, cr, g.oh, g.ow, g.rows, bn, g.nimg))
            return QT_EUNSUPPORTED;
        ep.res_tma = 1;
    } else {
        mp.res = mp.out;   // unused
    }
    const int tiles = (n / g.nimg) * g.tiles_per_img;
    const int ntiles = co / bn;
    switch (g.ow) {
        case 8: return dispatch_kc<8>(kc, kw, bn, mp, g, ep, tiles, ntiles, st);
        case 16: return dispatch_kc<16>(kc, kw, bn, mp, g, ep, tiles, ntiles, st);
        case 32: return dispatch_kc<32>(kc, kw, bn, mp, g, ep, tiles, ntiles, st);
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
