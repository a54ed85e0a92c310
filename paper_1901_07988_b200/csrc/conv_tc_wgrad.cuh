// Shared by conv_tc_wgrad.cu (host side) and the per-BN instantiation units
// conv_tc_wgrad_bn*.cu (compiled in parallel).
#pragma once
// Weight gradient on the tensor cores with the activation operand decoded
// from the packed K-bit tape straight into tensor memory.
//
//   dW[co][r = (ci,u,v)] += sum_{pixels p} act[ci][p shifted by (u,v)] * g[co][p]
//
// GEMM view: M = r (ci*kh*kw rows, 128-row tiles, A operand in TMEM), N = co
// (B operand = g_out, K-major in smem), K = output pixels, 32 per stage.
//   * TMA streams the g_out box (32 pixels x BN channels) from NCHW into a raw
//     ring; the same stage carries the packed codes the chunk needs: a box of
//     the input rows y-pad .. y+rows-1+pad (16-byte aligned byte window of
//     each channel plane) for every channel of the CTA's row group, so the
//     operand warps never wait on a global load.
//   * A rows are produced by their owning TMEM lane: the thread for row
//     (ci, u, v) reads the codes of input row y+u-pad from the stage, applies
//     the column shift v-pad with zero padding (a funnel shift of the row's
//     words) and writes the row with tcgen05.st -- the fp32 activation never
//     exists in HBM or shared memory.
//
// Two arithmetic modes, chosen per CTA from the frozen offsets of its
// channels (uniform branch, the tape's constants are on the device):
//   FAST (4-bit codes, every channel with 2^K-1+2*offset <= 127):
//     relu(decode(c)) = step/2 * m, m = max(0, 2c + 1 - 2^K + 2*offset), an
//     integer below 128, exact in bf16.  Two codes -> one bf16x2 A word with
//     three integer ops: (nibble pair)*2 + (0x4300 + b) per 16-bit lane is the
//     bf16 bit pattern of 128 + (2c + b), and fma.rn.relu(x, 1, -128) leaves
//     m exactly (negative lanes clamp to 0, the ReLU).  g_out is split into
//     three bf16 pieces (hi + mid + lo == g to fp32 precision), stacked along
//     N when 3*BN <= 192 so one kind::f16 MMA (K = 16 pixels) covers all
//     three; the epilogue sums the pieces in float64 and scales by step/2.
//     The pixel order inside a K step is permuted identically in A and B
//     (A word j of an 8-pixel group holds pixels j and j+4).
//   GENERIC (any width / offset, exact fp32 tapes, the plain stem input):
//     the reference's fp32 relu(decode) (or the fp32 value) is split into
//     TF32 (hi, lo) and three kind::tf32 passes hi*hi + hi*lo + lo*hi.
// Each MMA issues in ~46 cycles for N <= 64 (kind::f16 K=16 and kind::tf32
// K=8 alike), so pixels per instruction is the throughput lever.
// PRE-SPLIT (p.pre, FAST-capable codes, stacked pieces): g_out comes as the
//   three bf16 pieces already, in the FAST B layout (wg_pieces: per image,
//   chunk: [piece][co][32 px, pair-permuted]); one TMA box per stage lands
//   in a B ring read only by the MMA warp, so the operand warps only decode
//   A.  A CTA whose offsets leave the FAST range (GENERIC-PRE) splits the
//   reference's fp32 relu(decode) into three bf16 pieces in TMEM as well and
//   issues A_hi*[hi mid lo] + A_mid*[hi mid] + A_lo*[hi] (the six products
//   above 2^-24 relative), summed by the same three-group epilogue.
// Split-K over CTAs (contiguous pixel ranges), fp32 partials, then a
// deterministic fixed-order float64 reduction into grad_w (layer.py:167).
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "tc_common.cuh"

namespace qt {

using namespace tc;

constexpr int kWgThreads = 576;   // w0 TMA, w1 MMA/TMEM, w2..w17 operands + epilogue
constexpr int kWgLutEntries = 4096;
constexpr int kWgMaxCh = 256;     // channels per CTA row group (code box / FAST constants)

// debug timeline (qt_debug_wgrad_trace): per-chunk clock64 stamps of CTA
// (trace_cta, 0): [0] start, [1] setup done, then 5 per chunk: producer
// issue, operand raw_full ok, operand op_empty ok, operand done, MMA issue.
#define WG_TRACE(idx)                      \
    do {                                   \
        if (tr_) tr_[idx] = clock64();     \
    } while (0)

// FAST operand pair word from x = codes (pixel k | pixel k + 4 << 16):
// FAST: relu(m) for m = 2x + b (bc = 0x4300 + b; 8-bit: bf16x2_relu_m8);
// FAST2 (m < 2048): bc = (b + 2048) x 0x10001, v = max(2x + bc, 2048) per
// half, m = v & 0x7FF as the exact bf16 pieces (m & 0x7F0) + (m & 0xF) --
// 0x4500 + t is the bf16 pattern of 2048 + 16 t, 0x4300 + t of 128 + t
template <int BITS, bool TWO>
__device__ __forceinline__ void fast_pair(uint32_t x, uint32_t bc, uint32_t &a1, uint32_t &a2) {
    uint32_t v = x * 2u + bc;
    if constexpr (!TWO) {
        a1 = BITS == 8 ? bf16x2_relu_m8(v) : bf16x2_relu_sub128(v);
        return;
    } else {
    asm("max.u16x2 %0, %1, %2;" : "=r"(v) : "r"(v), "r"(0x08000800u));
    const uint32_t p1 = ((v >> 4) & 0x007F007Fu) | 0x45004500u, p2 = (v & 0x000F000Fu) | 0x43004300u;
    asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(a1) : "r"(p1), "r"(0x3F803F80u), "r"(0xC500C500u));
    asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(a2) : "r"(p2), "r"(0x3F803F80u), "r"(0xC300C300u));
    }
}

struct WgParams {
    qt_tape_t tape;          // codes (+step/offset) or a2 (relu) ...
    const float *plain;      // ... or the plain input (no relu)
    float *partial;          // [split][co][R]
    int n, ci, h, w, co, kh, kw, pad, oh, ow;
    int R;                   // ci*kh*kw
    int mtg;                 // 128-row M tiles per CTA (1 or 2)
    int rows_per_chunk;      // 32 / ow
    int chunks_per_img;      // oh*ow/32
    int total_chunks, chunks_per_split, splits;
    int RG, OPS, OPS_G;      // raw ring, operand ring (FAST), operand ring (GENERIC)
    int OPS2;                // operand ring (FAST2: two bf16 A pieces per chunk), 0: none
    int lut;                 // codes: smem code table in use
    int fbox;                // fp32 source (plain input / exact tape) staged per stage by TMA
    int lut_floats;          // smem table size (floats)
    int nolut;               // codes without the table (8-bit, wide channel blocks): decode inline
    int intok;               // INT mode allowed (QTAPE_WG_INT, default on)
    int slot;                // raw ring slot stride: g tile + code box (bytes)
    int cb;                  // code box bytes per channel (16-byte multiple)
    int cbytes;              // code box bytes per stage (cb x channels)
    int rb;                  // packed bytes per input row (ow*bits/8)
    int rpc;                 // A rows per input channel (kh*kw, or kh with column taps in N)
    long long *trace;        // debug timeline buffer (qt_debug_wgrad_trace) or NULL
    int trace_cta;
    int Rout;                // rows of dW = ci*kh*kw (partial row stride)
    int opreg;               // operand ring bytes (FAST and GENERIC strides share it)
    int pre;                 // g_out arrives pre-split: tmG maps the bf16 pieces
    int RB;                  // pre: B-piece ring depth (stages of SUB * 3 * BN rows of 64 B)
    FastDiv cpid;            // / chunks_per_img
};

// value of act at (nn, c, y, x) for fp32 sources (zero padding outside)
__device__ __forceinline__ float act_f32(const WgParams &p, int nn, int c, int y, int x) {
    if (y < 0 || y >= p.h || x < 0 || x >= p.w) return 0.f;
    const int64_t i = (((int64_t)nn * p.ci + c) * p.h + y) * p.w + x;
    if (p.plain) return __ldg(p.plain + i);
    const float a = __ldg(p.tape.a2 + i);
    return (a >= 0.f || isnan(a)) ? a : 0.f;  // ReLU as np.maximum (layer.py:356)
}

// GENERIC operand: 16 consecutive chunk pixels [P0, P0+16) of act row
// (c, u, v) as TF32 (hi, lo) -- the reference's fp32 relu(decode) from the
// smem code box through the per-channel table, or the fp32 source value.
// GENERIC operand: pixel i of the chunk for act row (c, u, v), as TF32 (hi,
// lo) of the reference's fp32 relu(decode(code)) (smem code box through the
// per-channel table), of the staged fp32 source, or of a global fp32 read.
// Branch-free: every smem read stays inside the stage's box (the pad rows are
// in the box; a column one past either edge reads a neighbouring word of the
// same stage) and out-of-image pixels are zeroed by a select.
__device__ __forceinline__ void generic_px(const WgParams &p, const uint8_t *cst, int cbox,
                                           int wbase, int nn, int c, int iy, int sx, int ow,
                                           const float *lut, uint32_t &hv, uint32_t &lv) {
    const bool ok = iy >= 0 && iy < p.h && sx >= 0 && sx < ow;
    float hh, ll;
    if (p.lut) {
        const uint32_t *cw = reinterpret_cast<const uint32_t *>(cst);
        const int bits = p.tape.bits;
        const int bp = (cbox + iy * p.rb - wbase) * 8 + sx * bits;
        const uint32_t code =
            __funnelshift_r(cw[bp >> 5], cw[(bp >> 5) + 1], bp & 31) & ((1u << bits) - 1u);
        if (p.nolut) {   // the table entry, computed: relu(decode(code)) as (hi, lo)
            float a = decode(code, __ldg(p.tape.step + c), __ldg(p.tape.offset + c), bits);
            a = (a >= 0.f || isnan(a)) ? a : 0.f;
            split_tf32(a, hh, ll);
        } else {
            const float2 e = *reinterpret_cast<const float2 *>(lut + 2 * code);
            hh = e.x;
            ll = e.y;
        }
    } else if (p.fbox) {
        float a = *reinterpret_cast<const float *>(cst + cbox + iy * p.rb - wbase + sx * 4);
        if (!p.plain) a = (a >= 0.f || isnan(a)) ? a : 0.f;   // exact tape: ReLU
        split_tf32(a, hh, ll);
    } else {
        split_tf32(act_f32(p, nn, c, iy, sx), hh, ll);
    }
    hv = ok ? __float_as_uint(hh) : 0u;
    lv = ok ? __float_as_uint(ll) : 0u;
}

// x -> three bf16 pieces hi + mid + lo (== x to fp32 precision), packed with
// a second value y in the high halves (pair words of the FAST layouts)
__device__ __forceinline__ void split3_bf16x2(float x, float y, uint32_t &H, uint32_t &M,
                                             uint32_t &L) {
    H = pack_bf16x2(x, y);
    const float rx = __fsub_rn(x, bf16_lo(H)), ry = __fsub_rn(y, bf16_hi(H));
    M = pack_bf16x2(rx, ry);
    L = pack_bf16x2(__fsub_rn(rx, bf16_lo(M)), __fsub_rn(ry, bf16_hi(M)));
}

// Operand warps form up to 4 warpgroups (one warp per TMEM lane quarter).
// With an operand ring of `ops` stages (a power of two <= 4), groups
// 0..ops-1 are active and group g owns chunks g, g+ops, ... -- so each ring
// stage (and each raw stage, RG being a multiple of ops) is only ever waited
// on by one group, in phase order (no mbarrier parity aliasing), and ops
// chunks are decoded concurrently.
constexpr int kWgGroups = 4;
constexpr int kWgSub = 2;          // 32-pixel chunks per ring stage (one MMA batch + commit)

// TAP (3x3, pad 1): A rows are (ci, u) only and the three column taps v move
// into N -- B_v[co][y][x] = g[co][y][x - v + 1] (zero outside the image row)
// -- so a 3x3 layer decodes 3x fewer A rows and issues fewer, wider MMAs.
template <int BN, int OW, int BITS, bool TAP>
__global__ void __launch_bounds__(kWgThreads, 1)
    conv_wgrad_tc_kernel(const __grid_constant__ CUtensorMap tmG,
                         const __grid_constant__ CUtensorMap tmC, WgParams p) {
    constexpr int ROWS = 32 / OW;                           // image rows per 32-pixel chunk
    constexpr int G_BYTES = BN * 128;                       // raw g tile: BN rows x 32 px fp32
    constexpr bool FAST_OK = (BITS == 4 || BITS == 2 || BITS == 1 || BITS == 8);
    // FAST2 is compiled for 8-bit codes only, where positive offsets are the
    // common case; narrower codes reach m >= 128 only past offset ~56 and take
    // INT there (the extra decode variant cost the FAST kernels ~3 %)
    constexpr bool kFast2 = BITS == 8;
    constexpr int NT = TAP ? 3 : 1;                         // column taps stacked in N
    constexpr bool STACK = TAP ? (9 * BN <= 256) : (3 * BN <= 192);   // pieces stacked in N
    constexpr int FACC = STACK ? 3 * NT * BN : NT * BN;     // FAST accumulator columns per tile
    constexpr int GACC = NT * BN;                           // GENERIC accumulator columns per tile
    // operand bytes per 32-px chunk: FAST 3 pieces x NT*BN rows x 64 B,
    // GENERIC (hi, lo) x NT*BN rows x 128 B (one shared region, p.opreg)
    constexpr int OPB_F = 3 * NT * BN * 64;
    constexpr int OPB_G = 2 * NT * BN * 128;
    constexpr int SUB = kWgSub;                             // 32-px chunks per pipeline stage
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1 KiB alignment by pointer arithmetic on the __shared__ array (keeps
    // every access in the shared window: LDS/STS, not generic LD/ST)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int RG = p.RG;
    // raw ring stage: g box [co][sub][32 px] (SW128 rows of 128 B), then the
    // code box [channel][cb bytes] covering the stage's SUB chunks
    uint8_t *graw = smem;                                   // RG x slot
    uint8_t *gop = graw + RG * p.slot;                      // operand ring (p.opreg bytes)
    float *s_lut = (float *)(gop + p.opreg);                // GENERIC code table (hi, lo)
    uint32_t *s_bc = (uint32_t *)(s_lut + p.lut_floats);    // FAST: 0x4300 + b per channel
    uint64_t *bars = (uint64_t *)(s_bc + kWgMaxCh);
    uint64_t *raw_full = bars, *raw_empty = bars + RG;
    uint64_t *op_full = raw_empty + RG, *op_empty = op_full + p.OPS;
    uint64_t *b_full = op_empty + p.OPS, *b_empty = b_full + p.RB;   // pre: B-piece ring
    uint64_t *done = b_empty + p.RB;
    uint32_t *tmem_slot = (uint32_t *)(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int split = blockIdx.x;
    const int co0 = blockIdx.z * BN;                        // this CTA's output-channel block
    const int row0 = blockIdx.y * p.mtg * 128;              // first M row of this group
    const int nrows = min(p.mtg * 128, p.R - row0);
    const int mt_here = (nrows + 127) / 128;
    const int kk = p.rpc;                                   // A rows per input channel
    const int c_begin = row0 / kk;
    const int c_end = min(p.ci, (row0 + nrows + kk - 1) / kk);
    const int k0 = split * p.chunks_per_split;
    const int k1 = min(p.total_chunks, k0 + p.chunks_per_split);
    const int nk = k1 - k0;                                 // chunks of this split
    const int nst = (nk + SUB - 1) / SUB;                   // pipeline stages
    long long *const tr_ =
        (p.trace && blockIdx.x == (unsigned)p.trace_cta && blockIdx.y == 0 && blockIdx.z == 0) ? p.trace : nullptr;
    if (threadIdx.x == 0) WG_TRACE(0);
    if (threadIdx.x == 0 && tr_)
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_[332]));
    if (threadIdx.x == 0 && p.trace && blockIdx.y == 0 && blockIdx.z == 0 && blockIdx.x < 1024) {
        uint32_t sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(p.trace[600 + 3 * blockIdx.x]));
        p.trace[602 + 3 * blockIdx.x] = sm;
    }

    if (threadIdx.x == 0) {
        for (int s = 0; s < RG; ++s) { mbar_init(&raw_full[s], 1); mbar_init(&raw_empty[s], 128); }
        for (int s = 0; s < p.OPS; ++s) { mbar_init(&op_full[s], 128); mbar_init(&op_empty[s], 1); }
        for (int s = 0; s < p.RB; ++s) { mbar_init(&b_full[s], 1); mbar_init(&b_empty[s], 1); }
        mbar_init(done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmG);
        if (p.lut || p.fbox) tma_prefetch(&tmC);
    }
    // per-CTA code tables: the reference's fp32 relu(decode(code)) split
    // (hi, lo) for GENERIC, and the FAST lane constant 0x4300 + b with
    // b = 1 - 2^K + 2*offset (clamped below at -64: all-zero channel)
    // The producer starts streaming right after this barrier; the other warps
    // build the per-CTA tables meanwhile (named barriers among warps 1..17).
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // setup above touched only smem / TMEM / the tensor maps: overlap it with
    // the previous kernel, then wait for that kernel's results
    pdl_wait();
    pdl_trigger();
    int fast = 0, fast2 = 0, intm = 0;
    if (warp != 0) {
        constexpr int kRest = kWgThreads - 32;     // warps 1..17
        int narrow = 1, inarrow = 1;
        const int nc = c_end - c_begin;
        if (FAST_OK && p.lut && threadIdx.x >= 64) {
            const int bits = p.tape.bits;
            for (int e = threadIdx.x - 64; e < nc; e += kWgThreads - 64) {
                const int64_t off = p.tape.offset[c_begin + e];
                const int64_t top = (1 << bits) - 1;            // m at the largest code
                if (off > (2047 - top) / 2) inarrow = 0;        // INT: m < 2048, exact in TF32
                if (BITS == 8) {
                    // m = 2c + b up to 255 + 2 off: exact in bf16 for off <= 0
                    // (decode bf16x2_relu_m8); off < -128 leaves every m < 0
                    if (off > 0) narrow = 0;
                    const int64_t b = 1 - (1 << bits) + 2 * max(off, (int64_t)-128);
                    s_bc[e] = (uint32_t)(0x4300 + b) * 0x10001u;
                    continue;
                }
                if (off > (127 - top) / 2) narrow = 0;          // m could reach 128
                const int64_t b = 1 - (1 << bits) + 2 * max(off, (int64_t)-64);
                s_bc[e] = (uint32_t)(0x4300 + max(b, (int64_t)-64)) * 0x10001u;
            }
        }
        uint32_t all;
        asm volatile(
            "{\n\t.reg .pred p, q;\n\t"
            "setp.ne.u32 q, %1, 0;\n\t"
            "bar.red.and.pred p, 1, %2, q;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(all)
            : "r"((uint32_t)narrow), "n"(kRest)
            : "memory");
        fast = (all != 0) && FAST_OK && p.lut;
        if (!fast && FAST_OK && p.lut && p.intok && p.pre == 0 && !TAP) {
            asm volatile(
                "{\n\t.reg .pred p, q;\n\t"
                "setp.ne.u32 q, %1, 0;\n\t"
                "bar.red.and.pred p, 1, %2, q;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(all)
                : "r"((uint32_t)inarrow), "n"(kRest)
                : "memory");
            // m < 2048: FAST2 (two bf16 A pieces) when its ring fits TMEM,
            // else INT (TF32 A)
            fast2 = (all != 0) && p.OPS2 > 0 && kFast2;
            intm = (all != 0) && !fast2;
        }
        // INT: s_bc holds b = 1 - 2^K + 2 off; FAST2: (max(b, -2048) + 2048) x 0x10001
        if ((intm || fast2) && threadIdx.x >= 64) {
            const int bits = p.tape.bits;
            for (int e = threadIdx.x - 64; e < nc; e += kWgThreads - 64) {
                const int64_t off = max(p.tape.offset[c_begin + e], (int64_t)-4096);
                const int32_t b = (int32_t)(1 - (1 << bits) + 2 * off);
                s_bc[e] = fast2 ? (uint32_t)(max(b, -2048) + 2048) * 0x10001u : (uint32_t)b;
            }
        }
        // the GENERIC table only when this CTA takes the GENERIC path
        if (!fast && !fast2 && !intm && p.lut && !p.nolut && threadIdx.x >= 64) {
            const int bits = p.tape.bits, ncode = 1 << bits;
            for (int e = threadIdx.x - 64; e < nc * ncode; e += kWgThreads - 64) {
                const int cc = c_begin + e / ncode, code = e % ncode;
                float a = decode((uint32_t)code, p.tape.step[cc], p.tape.offset[cc], bits);
                a = (a >= 0.f || isnan(a)) ? a : 0.f;
                if (p.pre) {   // GENERIC-PRE: the value itself, channel stride 2^K + 1
                    s_lut[(e / ncode) * (ncode + 1) + code] = a;
                    continue;
                }
                // channel stride 2^(K+1) + 2 floats: lanes on different
                // channels reading the same code hit different banks
                float *q = s_lut + (e / ncode) * ((2 << bits) + 2) + 2 * code;
                split_tf32(a, q[0], q[1]);
            }
        }
        if (threadIdx.x >= 64)   // operand warps: tables complete before use
            asm volatile("bar.sync 2, %0;" ::"n"(kWgThreads - 64) : "memory");
    }
    if (threadIdx.x == 0) WG_TRACE(1);
    if (threadIdx.x == 64 && tr_)   // an operand thread (warp 0 does not take part in the vote)
        tr_[525] = fast, tr_[526] = intm, tr_[527] = fast2;
    const bool fastb = fast || fast2;                       // bf16 integer A, g pieces in smem
    const int ops = fast ? p.OPS : fast2 ? p.OPS2 : p.OPS_G;
    const bool pre = p.pre != 0;                            // B pieces by TMA (STACK, !TAP)
    const bool pieces = fastb || pre;                       // three-piece accumulator groups
    const int OPB = pieces ? OPB_F : OPB_G;                 // operand stride per chunk
    const uint32_t acc_cols = (uint32_t)(p.mtg * (pieces ? FACC : GACC));
    const uint32_t acols = fast ? 16u : fast2 ? 32u : (pre ? 48u : 64u);  // A columns per tile per stage

    if (warp == 0) {
        if (lane == 1 && pre) {  // ------------- TMA producer of the B pieces (pre-split)
            // its own lane: the code boxes run ahead of the B ring's depth
            int nn = k0 / p.chunks_per_img, yc = k0 % p.chunks_per_img;
            int sb = 0;
            uint32_t phb = 0;
            for (int st = 0; st < nst; ++st) {
                mbar_wait(&b_empty[sb], phb ^ 1u);
                mbar_expect_tx(&b_full[sb], SUB * OPB_F);
                tma_load_5d(gop + sb * (SUB * OPB_F), &tmG, &b_full[sb], 0, co0, 0, yc, nn);
                if (++sb == p.RB) { sb = 0; phb ^= 1u; }
                yc += SUB;
                if (yc >= p.chunks_per_img) { yc -= p.chunks_per_img; ++nn; }
            }
        }
        if (lane == 0) {  // ----------------------------- TMA producer (g_out + codes)
            // one g box and one code box per stage: its SUB chunks are
            // consecutive pixel runs of one image (cps, cpi multiples of SUB)
            int nn = k0 / p.chunks_per_img, yc = k0 % p.chunks_per_img;
            int s = 0;
            uint32_t ph = 0;
            for (int st = 0; st < nst; ++st) {
                mbar_wait(&raw_empty[s], ph ^ 1u);
                if (st < 64) WG_TRACE(2 + 5 * st);
                const int y0 = yc * p.rows_per_chunk;
                uint8_t *slot = graw + s * p.slot;
                if (pre) {   // codes -> raw ring (the B pieces: lane 1)
                    mbar_expect_tx(&raw_full[s], p.cbytes);
                    tma_load_3d(slot, &tmC, &raw_full[s], ((y0 - p.pad) * p.rb) & ~15, c_begin, nn);
                } else {
                mbar_expect_tx(&raw_full[s], SUB * G_BYTES + p.cbytes);
                tma_load_4d(slot, &tmG, &raw_full[s], 0, yc, co0, nn);
                if (p.lut)   // 16-byte aligned window of input rows y0-pad ..
                    tma_load_3d(slot + SUB * G_BYTES, &tmC, &raw_full[s],
                                ((y0 - p.pad) * p.rb) & ~15, c_begin, nn);
                else if (p.fbox)               // fp32 rows y0-pad .. (OOB rows zero-filled)
                    tma_load_3d(slot + SUB * G_BYTES, &tmC, &raw_full[s], (y0 - p.pad) * p.ow,
                                c_begin, nn);
                }
                yc += SUB;
                if (yc >= p.chunks_per_img) { yc -= p.chunks_per_img; ++nn; }
                if (st < 64) WG_TRACE(336 + 3 * st);
                if (++s == RG) { s = 0; ph ^= 1u; }
            }
        }
    } else if (warp == 1) {  // ---------------- MMA issuer (whole warp, one lane issues)
        // descriptors are a fixed base plus (byte offset >> 4) in the start
        // address field (all operand tiles lie below 256 KiB); the loops are
        // unrolled over the compile-time maxima with predicates, so an MMA
        // costs a couple of uniform adds
        int o = 0, sb = 0;
        uint32_t ph = 0, phb = 0;
        const uint32_t gop_base = smem_u32(gop);
        const uint64_t dfast = smem_desc(gop_base, 16, 512, 4);    // bf16 SW64 K-major
        const uint64_t dgen = smem_desc(gop_base, 16, 1024, 2);    // tf32 SW128 K-major
        const uint32_t mtg = (uint32_t)p.mtg;
        for (int st = 0; st < nst; ++st) {
            mbar_wait(&op_full[o], ph);
            if (pre) mbar_wait(&b_full[sb], phb);
            if (lane == 0 && st < 64) WG_TRACE(6 + 5 * st);
            tc_fence_after();
            const int nsub = min(SUB, nk - st * SUB);
            if (elect_one()) {
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    if (t >= mt_here) break;
#pragma unroll
                    for (int sub = 0; sub < SUB; ++sub) {
                        if (sub >= nsub) break;
                        const uint32_t off16 =
                            (uint32_t)((((pre ? sb : o) * SUB + sub) * OPB) >> 4);
                        const uint32_t a =
                            tmem + acc_cols + (((uint32_t)o * mtg + t) * SUB + sub) * acols;
                        const uint32_t first = (st | sub) ? 1u : 0u;   // 0: zero-init D
                        if (fastb) {
                            // FAST2: the second A piece (16 columns on) against the same B
                            constexpr uint32_t idesc = instr_desc(128, FACC, 1, 0, 0);
                            const uint32_t d = tmem + (uint32_t)(t * FACC);
#pragma unroll
                            for (int j = 0; j < 2; ++j) {
#pragma unroll
                                for (int ap = 0; ap < 2; ++ap) {
                                    if (ap && (!kFast2 || !fast2)) break;
                                    if (STACK) {
                                        mma_bf16_ts(d, a + 16 * ap + j * 8, dfast + off16 + j * 2, idesc,
                                                    (first | j | ap) ? 1u : 0u);
                                    } else {
#pragma unroll
                                        for (int pc = 0; pc < 3; ++pc)
                                            mma_bf16_ts(d, a + 16 * ap + j * 8,
                                                        dfast + off16 + ((pc * NT * BN * 64) >> 4) + j * 2,
                                                        idesc, (first | j | pc | ap) ? 1u : 0u);
                                    }
                                }
                            }
                        } else if (!STACK && !TAP && pre) {
                            // GENERIC-PRE, one accumulator: the six products above
                            // 2^-24 relative, each N = BN
                            constexpr uint32_t id1 = instr_desc(128, BN, 1, 0, 0);
                            const uint32_t d = tmem + (uint32_t)(t * FACC);
                            constexpr uint32_t pb = (BN * 64) >> 4;   // piece block (desc units)
#pragma unroll
                            for (int j = 0; j < 2; ++j) {
                                const uint64_t bh = dfast + off16 + j * 2;
                                mma_bf16_ts(d, a + j * 8, bh, id1, (first | j) ? 1u : 0u);
                                mma_bf16_ts(d, a + j * 8, bh + pb, id1, 1u);
                                mma_bf16_ts(d, a + 16 + j * 8, bh, id1, 1u);
                                mma_bf16_ts(d, a + 16 + j * 8, bh + pb, id1, 1u);
                                mma_bf16_ts(d, a + j * 8, bh + 2 * pb, id1, 1u);
                                mma_bf16_ts(d, a + 32 + j * 8, bh, id1, 1u);
                            }
                        } else if (STACK && !TAP && pre) {
                            // GENERIC-PRE: A pieces (hi, mid, lo) at +0/16/32 columns
                            // against the stacked B rows [hi | mid | lo]
                            constexpr uint32_t id3 = instr_desc(128, 3 * BN, 1, 0, 0);
                            constexpr uint32_t id2 = instr_desc(128, 2 * BN, 1, 0, 0);
                            constexpr uint32_t id1 = instr_desc(128, BN, 1, 0, 0);
                            const uint32_t d = tmem + (uint32_t)(t * FACC);
#pragma unroll
                            for (int j = 0; j < 2; ++j) {
                                mma_bf16_ts(d, a + j * 8, dfast + off16 + j * 2, id3,
                                            (first | j) ? 1u : 0u);
                                mma_bf16_ts(d, a + 16 + j * 8, dfast + off16 + j * 2, id2, 1u);
                                mma_bf16_ts(d, a + 32 + j * 8, dfast + off16 + j * 2, id1, 1u);
                            }
                        } else {
                            constexpr uint32_t idesc = instr_desc(128, GACC, 2, 0, 0);
                            const uint32_t d = tmem + (uint32_t)(t * GACC);
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const uint64_t dgh = dgen + off16 + j * 2;
                                const uint64_t dgl = dgh + ((NT * BN * 128) >> 4);
                                mma_tf32_ts(d, a + j * 8, dgh, idesc, (first | j) ? 1u : 0u);
                                mma_tf32_ts(d, a + j * 8, dgl, idesc, 1u);
                                if (!intm) mma_tf32_ts(d, a + 32 + j * 8, dgh, idesc, 1u);
                            }
                        }
                    }
                }
                mma_commit(&op_empty[o]);
                if (pre) mma_commit(&b_empty[sb]);
                if (st == nst - 1) mma_commit(done);
            }
            __syncwarp();
            if (lane == 0 && st < 64) WG_TRACE(401 + 2 * st);
            if (++o == ops) { o = 0; ph ^= 1u; }
            if (pre && ++sb == p.RB) { sb = 0; phb ^= 1u; }
        }
        if (nst == 0 && lane == 0) mbar_arrive(done);
    } else {  // ---------------------- operand warpgroups + epilogue
        const int grp = (warp - 2) >> 2;     // warpgroup 0..kWgGroups-1
        const int quarter = warp & 3;        // TMEM lanes 32*quarter .. +31
        const int tg = threadIdx.x - 64 - 128 * grp;        // 0..127 within the group
        const uint32_t lane_base = tmem + ((uint32_t)(32 * quarter) << 16);
        const int lut_stride = !p.lut ? 0 : (p.pre ? (1 << p.tape.bits) + 1 : (2 << p.tape.bits) + 2);
        // this thread's act rows: tile t -> local row t*128 + 32*quarter + lane
        int rc[2], ru[2], rsh[2];
        bool rok[2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int rl = t * 128 + 32 * quarter + lane;
            rok[t] = rl < nrows && t < mt_here;
            const int r = row0 + rl;
            const int c = r / kk, uv = r - c * kk;
            const int u = TAP ? uv : uv / p.kw, v = TAP ? p.pad : uv - u * p.kw;
            rc[t] = rok[t] ? c : c_begin;
            ru[t] = u;
            rsh[t] = v - p.pad;   // TAP: 0 (the column shift is in B)
        }
        // FAST: group g owns ring stage g (stages g, g+ops, ...).  GENERIC
        // (coop): the TF32 A operand limits the ring to 1-2 stages, so all
        // four groups share every stage -- pixel quads and g items dealt
        // round-robin -- and meet at a named barrier before group 0 arrives.
        const bool coop = !fastb;
        // FAST: group g takes stages g, g + G, ... (G = active groups); with
        // an operand ring deeper than G (pre-split: A only in TMEM, up to 8)
        // it alternates between op stages g and g + G -- raw slots and op
        // stages of one group never alias another's (RG, ops multiples of G)
        const int sstep = coop ? 1 : min(ops, kWgGroups);
        const int gsplit = coop ? grp : 0, gstride = coop ? kWgGroups : 1;
        int st = coop ? 0 : (grp < ops ? grp : nst);   // FAST groups beyond the ring idle
        int s = st % RG;
        int o = coop ? 0 : st % ops;          // operand ring stage
        uint32_t phr = (uint32_t)(st / RG) & 1u, pho = (uint32_t)(st / ops) & 1u;
        for (; st < nst; st += sstep) {
            mbar_wait(&raw_full[s], phr);
            if (tg == 0 && st < 64) WG_TRACE(3 + 5 * st);
            mbar_wait(&op_empty[o], pho ^ 1u);
            if (tg == 0 && st < 64) WG_TRACE(4 + 5 * st);
            tc_fence_after();
            const int nsub = min(SUB, nk - st * SUB);
            const int kc0 = k0 + st * SUB;                            // first chunk of the stage
            const int nn = (int)fast_div((uint32_t)kc0, p.cpid);
            const int ys = (kc0 - nn * p.chunks_per_img) * p.rows_per_chunk;
            const uint8_t *graws = graw + s * p.slot;
            const uint8_t *cst = graws + (pre ? 0 : SUB * G_BYTES);   // code box
            const int wbase = p.fbox ? (ys - p.pad) * p.rb                // its first byte
                                     : ((ys - p.pad) * p.rb) & ~15;
            for (int sub = 0; sub < nsub; ++sub) {
            const int y0 = ys + sub * p.rows_per_chunk;
            uint8_t *opb = gop + (o * SUB + sub) * OPB;
            if (pre) {
                // B pieces arrive by TMA (B ring)
            } else if (TAP) {
                // g -> the three column-shifted copies B_v[x] = g[x - v + 1]
                // (zero outside the image row); FAST: bf16 pieces, rows
                // (piece, v, co), pair-permuted K; GENERIC: TF32 (hi, lo),
                // rows (v, co), natural pixel order
                // items (v, co, 8-px group): three per (co, group), spread over
                // all 128 threads of the group
                for (int q = tg + 128 * gsplit; q < 3 * BN * 4; q += 128 * gstride) {
                    const int v = q / (BN * 4), qr = q - v * (BN * 4);
                    const int co = qr >> 2, qq = qr & 3, px0 = 8 * qq;
                    const uint32_t rrow = (uint32_t)((co * SUB + sub) * 128);
                    const float4 x0 = *reinterpret_cast<const float4 *>(
                        graws + swz_off<128>(rrow + px0 * 4));
                    const float4 x1 = *reinterpret_cast<const float4 *>(
                        graws + swz_off<128>(rrow + px0 * 4 + 16));
                    const float left = (px0 % OW) ? *reinterpret_cast<const float *>(
                                                        graws + swz_off<128>(rrow + px0 * 4 - 4))
                                                  : 0.f;
                    const float right = ((px0 + 8) % OW) ? *reinterpret_cast<const float *>(
                                                               graws + swz_off<128>(rrow + px0 * 4 + 32))
                                                         : 0.f;
                    const float vals[10] = {left, x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w, right};
                    // this tap's window: wv[k] = g[px0 + k - v + 1] = vals[k + 2 - v]
                    float wv[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        wv[k] = v == 0 ? vals[k + 2] : (v == 1 ? vals[k + 1] : vals[k]);
                    {
                        if (fast) {
                            uint32_t H[4], M[4], L[4];
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const float xa = wv[k], xb = wv[k + 4];
                                H[k] = pack_bf16x2(xa, xb);
                                const float ra = __fsub_rn(xa, bf16_lo(H[k]));
                                const float rb = __fsub_rn(xb, bf16_hi(H[k]));
                                M[k] = pack_bf16x2(ra, rb);
                                L[k] = pack_bf16x2(__fsub_rn(ra, bf16_lo(M[k])),
                                                   __fsub_rn(rb, bf16_hi(M[k])));
                            }
#pragma unroll
                            for (int pc = 0; pc < 3; ++pc) {
                                const int row = (pc * 3 + v) * BN + co;
                                const uint32_t off =
                                    swz_off<64>((uint32_t)((row >> 3) * 512 + (row & 7) * 64 + qq * 16));
                                *reinterpret_cast<uint4 *>(opb + off) =
                                    pc == 0 ? make_uint4(H[0], H[1], H[2], H[3])
                                            : (pc == 1 ? make_uint4(M[0], M[1], M[2], M[3])
                                                       : make_uint4(L[0], L[1], L[2], L[3]));
                            }
                        } else {
                            float hi[8], lo[8];
#pragma unroll
                            for (int k = 0; k < 8; ++k) split_tf32(wv[k], hi[k], lo[k]);
                            const int row = v * BN + co;
                            const uint32_t o0 = swz_off<128>((uint32_t)(row * 128 + px0 * 4));
                            const uint32_t o1 = swz_off<128>((uint32_t)(row * 128 + px0 * 4 + 16));
                            *reinterpret_cast<float4 *>(opb + o0) = make_float4(hi[0], hi[1], hi[2], hi[3]);
                            *reinterpret_cast<float4 *>(opb + o1) = make_float4(hi[4], hi[5], hi[6], hi[7]);
                            *reinterpret_cast<float4 *>(opb + NT * BN * 128 + o0) =
                                make_float4(lo[0], lo[1], lo[2], lo[3]);
                            *reinterpret_cast<float4 *>(opb + NT * BN * 128 + o1) =
                                make_float4(lo[4], lo[5], lo[6], lo[7]);
                        }
                    }
                }
            } else if (fastb) {
                // g -> bf16 (hi, mid, lo), K-major SW64, 8-pixel groups
                // permuted (pair word k = pixels k and k+4)
                for (int q = tg; q < BN * 4; q += 128) {
                    const int co = q >> 2, qq = q & 3;
                    const uint32_t rrow = (uint32_t)((co * SUB + sub) * 128);
                    // odd channels read their two 16-byte halves in the other
                    // order: the 8 lanes of a quarter warp (2 channels x 4
                    // groups) then hit 8 distinct swizzled chunks (no conflict)
                    const uint32_t fl = (uint32_t)(co & 1) * 16u;
                    const float4 y0 = *reinterpret_cast<const float4 *>(
                        graws + swz_off<128>(rrow + qq * 32 + fl));
                    const float4 y1 = *reinterpret_cast<const float4 *>(
                        graws + swz_off<128>(rrow + qq * 32 + (16u - fl)));
                    const float4 x0 = fl ? y1 : y0, x1 = fl ? y0 : y1;
                    const float xa[4] = {x0.x, x0.y, x0.z, x0.w}, xb[4] = {x1.x, x1.y, x1.z, x1.w};
                    uint32_t H[4], M[4], L[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        H[k] = pack_bf16x2(xa[k], xb[k]);
                        const float ra = __fsub_rn(xa[k], bf16_lo(H[k]));
                        const float rb = __fsub_rn(xb[k], bf16_hi(H[k]));
                        M[k] = pack_bf16x2(ra, rb);
                        L[k] = pack_bf16x2(__fsub_rn(ra, bf16_lo(M[k])), __fsub_rn(rb, bf16_hi(M[k])));
                    }
                    const uint32_t off = swz_off<64>((uint32_t)((co >> 3) * 512 + (co & 7) * 64 + qq * 16));
                    *reinterpret_cast<uint4 *>(opb + off) = make_uint4(H[0], H[1], H[2], H[3]);
                    *reinterpret_cast<uint4 *>(opb + BN * 64 + off) = make_uint4(M[0], M[1], M[2], M[3]);
                    *reinterpret_cast<uint4 *>(opb + 2 * BN * 64 + off) = make_uint4(L[0], L[1], L[2], L[3]);
                }
                if (tg == 0 && st < 64) WG_TRACE(3700 + 4 * st + 2 * sub);
            } else {   // g tile: TF32 (hi, lo) split into a K-major SW128 tile
                for (int q = tg + 128 * gsplit; q < G_BYTES / 16; q += 128 * gstride) {
                    const int co = q >> 3, ch16 = q & 7;
                    const float4 x = *reinterpret_cast<const float4 *>(
                        graws + swz_off<128>((uint32_t)((co * SUB + sub) * 128 + ch16 * 16)));
                    float4 *gh = reinterpret_cast<float4 *>(opb + swz_off<128>((uint32_t)(co * 128 + ch16 * 16)));
                    float4 *gl = reinterpret_cast<float4 *>(reinterpret_cast<uint8_t *>(gh) + G_BYTES);
                    float4 hi, lo;
                    split_tf32(x.x, hi.x, lo.x);
                    split_tf32(x.y, hi.y, lo.y);
                    split_tf32(x.z, hi.z, lo.z);
                    split_tf32(x.w, hi.w, lo.w);
                    *gh = hi;
                    *gl = lo;
                }
            }
#pragma unroll
            for (int t = 0; t < 2; ++t) {    // A rows of tile t for this chunk's 32 pixels
                if (t >= mt_here) break;
                const uint32_t acol = acc_cols + (uint32_t)((o * p.mtg + t) * SUB + sub) * acols;
                const int c = rc[t], u = ru[t], sh = rsh[t];
                const int cbox = (c - c_begin) * p.cb;
                if (FAST_OK && fastb) {
                    // FAST / FAST2 rows; the A piece count is a compile-time
                    // branch so the FAST loops carry none of FAST2's decode
                    auto rows = [&](auto two_c) {
                    [[maybe_unused]] constexpr bool TWO = decltype(two_c)::value;
                    if constexpr (BITS == 1) {
                    // 1-bit codes: a row of OW <= 32 px is one 8/16/32-bit field
                    // (bit x = pixel x).  Per 8-pixel group (byte b):
                    // z = (b & 0xF) | (b >> 4) << 16 puts pixel k at bit k and
                    // pixel k + 4 at bit 16 + k, so (z >> k) & 0x00010001 is A
                    // word k of the (k, k + 4) pairing -- then the same
                    // *2 + (0x4300 + b) and relu(x - 128) as the 4-bit path
                    uint32_t av[16], av2[16];
#pragma unroll
                    for (int x = 0; x < 16; ++x) av[x] = av2[x] = 0u;
                    if (rok[t]) {
                        const uint32_t bc = s_bc[c - c_begin];
#pragma unroll
                        for (int seg = 0; seg < ROWS; ++seg) {
                            const int iy = y0 + seg + u - p.pad;
                            if (iy < 0 || iy >= p.h) continue;
                            const uint8_t *rowp = cst + cbox + iy * p.rb - wbase;
                            uint32_t w = OW == 32 ? *reinterpret_cast<const uint32_t *>(rowp)
                                       : OW == 16 ? (uint32_t)*reinterpret_cast<const uint16_t *>(rowp)
                                                  : (uint32_t)*rowp;
                            constexpr uint32_t rmask = OW == 32 ? 0xFFFFFFFFu : ((1u << OW) - 1u);
                            w = sh > 0 ? (w >> 1) : sh < 0 ? ((w << 1) & rmask) : w;
#pragma unroll
                            for (int gq = 0; gq < OW / 8; ++gq) {
                                const uint32_t b8 = (w >> (8 * gq)) & 0xFFu;
                                const uint32_t z = (b8 & 0xFu) | ((b8 >> 4) << 16);
#pragma unroll
                                for (int k = 0; k < 4; ++k)
                                    fast_pair<BITS, TWO>((z >> k) & 0x00010001u, bc,
                                                    av[seg * (OW / 2) + 4 * gq + k],
                                                    av2[seg * (OW / 2) + 4 * gq + k]);
                            }
                            if (sh < 0)   // x = 0 pads
                                av[seg * (OW / 2)] &= 0xFFFF0000u, av2[seg * (OW / 2)] &= TWO ? 0xFFFF0000u : 0u;
                            if (sh > 0)   // x = OW-1
                                av[seg * (OW / 2) + OW / 2 - 1] &= 0x0000FFFFu,
                                    av2[seg * (OW / 2) + OW / 2 - 1] &= TWO ? 0x0000FFFFu : 0u;
                        }
                    }
                    tmem_st16(lane_base + acol, av);
                    if (TWO) tmem_st16(lane_base + acol + 16, av2);
                    } else if constexpr (BITS == 8) {
                    // 8-bit codes: a row is OW bytes (8 px: two words lo, hi).
                    // A word k of a group pairs byte k of lo and of hi
                    // (pixels k, k + 4), then *2 + (0x4300 + b) and the
                    // 8-bit relu decode (m <= 255: exact in bf16)
                    constexpr int NW = OW / 4;                 // 32-bit words per row
                    uint32_t av[16], av2[16];
#pragma unroll
                    for (int x = 0; x < 16; ++x) av[x] = av2[x] = 0u;
                    if (rok[t]) {
                        const uint32_t bc = s_bc[c - c_begin];
#pragma unroll
                        for (int seg = 0; seg < ROWS; ++seg) {
                            const int iy = y0 + seg + u - p.pad;
                            if (iy < 0 || iy >= p.h) continue;
                            const uint8_t *rowp = cst + cbox + iy * p.rb - wbase;
                            uint32_t w[NW + 2];
                            w[0] = 0u;
                            w[NW + 1] = 0u;
                            if constexpr (NW == 2) {
                                const uint2 v2 = *reinterpret_cast<const uint2 *>(rowp);
                                w[1] = v2.x; w[2] = v2.y;
                            } else {
#pragma unroll
                                for (int q = 0; q < NW / 4; ++q) {
                                    const uint4 v4 = reinterpret_cast<const uint4 *>(rowp)[q];
                                    w[4 * q + 1] = v4.x; w[4 * q + 2] = v4.y;
                                    w[4 * q + 3] = v4.z; w[4 * q + 4] = v4.w;
                                }
                            }
                            uint32_t sw[NW];
#pragma unroll
                            for (int q = 0; q < NW; ++q)
                                sw[q] = sh > 0   ? __funnelshift_r(w[q + 1], w[q + 2], 8)
                                        : sh < 0 ? __funnelshift_l(w[q], w[q + 1], 8)
                                                 : w[q + 1];
#pragma unroll
                            for (int gq = 0; gq < OW / 8; ++gq) {
#pragma unroll
                                for (int k = 0; k < 4; ++k) {
                                    const uint32_t z =
                                        __byte_perm(sw[2 * gq], sw[2 * gq + 1], k | (4u + k) << 8);
                                    fast_pair<BITS, TWO>(z & 0x00FF00FFu, bc,
                                                    av[seg * (OW / 2) + 4 * gq + k],
                                                    av2[seg * (OW / 2) + 4 * gq + k]);
                                }
                            }
                            if (sh < 0)   // x = 0 pads
                                av[seg * (OW / 2)] &= 0xFFFF0000u, av2[seg * (OW / 2)] &= TWO ? 0xFFFF0000u : 0u;
                            if (sh > 0)   // x = OW-1
                                av[seg * (OW / 2) + OW / 2 - 1] &= 0x0000FFFFu,
                                    av2[seg * (OW / 2) + OW / 2 - 1] &= TWO ? 0x0000FFFFu : 0u;
                        }
                    }
                    tmem_st16(lane_base + acol, av);
                    if (TWO) tmem_st16(lane_base + acol + 16, av2);
                    } else if constexpr (BITS == 2) {
                    // 2-bit codes: a row is OW/4 bytes (8 px: one halfword).
                    // Per 8-pixel group (16 bits h): z = (h & 0xFF) | (h >> 8) << 16
                    // puts pixel k at bits 2k and pixel k + 4 at bits 16 + 2k,
                    // so (z >> 2k) & 0x00030003 is A word k of the group's
                    // (k, k + 4) pixel pairing -- then the same *2 + (0x4300 + b)
                    // and relu(x - 128) as the 4-bit path (m < 128, exact)
                    uint32_t av[16], av2[16];
#pragma unroll
                    for (int x = 0; x < 16; ++x) av[x] = av2[x] = 0u;
                    if (rok[t]) {
                        const uint32_t bc = s_bc[c - c_begin];
#pragma unroll
                        for (int seg = 0; seg < ROWS; ++seg) {
                            const int iy = y0 + seg + u - p.pad;
                            if (iy < 0 || iy >= p.h) continue;
                            const uint8_t *rowp = cst + cbox + iy * p.rb - wbase;
                            uint32_t hw[OW / 8];               // one 16-bit group per entry
                            if (OW == 8) {
                                uint32_t w0 = *reinterpret_cast<const uint16_t *>(rowp);
                                w0 = sh > 0 ? (w0 >> 2) : sh < 0 ? ((w0 << 2) & 0xFFFFu) : w0;
                                hw[0] = w0;
                            } else {
                                constexpr int NW = OW / 16;            // 32-bit words per row
                                const uint32_t *cw = reinterpret_cast<const uint32_t *>(rowp);
                                uint32_t w[NW + 2];
                                w[0] = 0u;
                                w[NW + 1] = 0u;
                                if constexpr (NW == 2) {
                                    const uint2 v2 = *reinterpret_cast<const uint2 *>(cw);
                                    w[1] = v2.x; w[2] = v2.y;
                                } else {
#pragma unroll
                                    for (int q = 0; q < NW; ++q) w[q + 1] = cw[q];
                                }
#pragma unroll
                                for (int q = 0; q < NW; ++q) {
                                    const uint32_t sw = sh > 0   ? __funnelshift_r(w[q + 1], w[q + 2], 2)
                                                        : sh < 0 ? __funnelshift_l(w[q], w[q + 1], 2)
                                                                 : w[q + 1];
                                    hw[2 * q] = sw & 0xFFFFu;
                                    hw[2 * q + 1] = sw >> 16;
                                }
                            }
#pragma unroll
                            for (int gq = 0; gq < OW / 8; ++gq) {
                                const uint32_t z = (hw[gq] & 0xFFu) | ((hw[gq] >> 8) << 16);
#pragma unroll
                                for (int k = 0; k < 4; ++k)
                                    fast_pair<BITS, TWO>((z >> (2 * k)) & 0x00030003u, bc,
                                                    av[seg * (OW / 2) + 4 * gq + k],
                                                    av2[seg * (OW / 2) + 4 * gq + k]);
                            }
                            if (sh < 0)   // x = 0 pads
                                av[seg * (OW / 2)] &= 0xFFFF0000u, av2[seg * (OW / 2)] &= TWO ? 0xFFFF0000u : 0u;
                            if (sh > 0)   // x = OW-1
                                av[seg * (OW / 2) + OW / 2 - 1] &= 0x0000FFFFu,
                                    av2[seg * (OW / 2) + OW / 2 - 1] &= TWO ? 0x0000FFFFu : 0u;
                        }
                    }
                    tmem_st16(lane_base + acol, av);
                    if (TWO) tmem_st16(lane_base + acol + 16, av2);
                    } else if constexpr (BITS == 4) {
                    constexpr int NW = OW / 8;                 // 32-bit words per row (4-bit)
                    uint32_t av[16], av2[16];
#pragma unroll
                    for (int x = 0; x < 16; ++x) av[x] = av2[x] = 0u;
                    if (rok[t]) {
                        const uint32_t bc = s_bc[c - c_begin];
#pragma unroll
                        for (int seg = 0; seg < ROWS; ++seg) {
                            const int iy = y0 + seg + u - p.pad;
                            if (iy < 0 || iy >= p.h) continue;
                            const uint32_t *cw = reinterpret_cast<const uint32_t *>(
                                cst + cbox + iy * p.rb - wbase);
                            uint32_t w[NW + 2];
                            w[0] = 0u;
                            w[NW + 1] = 0u;
                            // one vector load per row (rows are NW-word aligned):
                            // lanes on different channels then spread over the
                            // banks instead of queueing per word
                            if constexpr (NW == 4) {
                                const uint4 v4 = *reinterpret_cast<const uint4 *>(cw);
                                w[1] = v4.x; w[2] = v4.y; w[3] = v4.z; w[4] = v4.w;
                            } else if constexpr (NW == 2) {
                                const uint2 v2 = *reinterpret_cast<const uint2 *>(cw);
                                w[1] = v2.x; w[2] = v2.y;
                            } else {
#pragma unroll
                                for (int q = 0; q < NW; ++q) w[q + 1] = cw[q];
                            }
#pragma unroll
                            for (int q = 0; q < NW; ++q) {
                                const uint32_t sw = sh > 0   ? __funnelshift_r(w[q + 1], w[q + 2], 4)
                                                    : sh < 0 ? __funnelshift_l(w[q], w[q + 1], 4)
                                                             : w[q + 1];
#pragma unroll
                                for (int k = 0; k < 4; ++k)
                                    fast_pair<BITS, TWO>((sw >> (4 * k)) & 0x000F000Fu, bc,
                                                    av[seg * (OW / 2) + 4 * q + k],
                                                    av2[seg * (OW / 2) + 4 * q + k]);
                            }
                            if (sh < 0)   // x = 0 pads
                                av[seg * (OW / 2)] &= 0xFFFF0000u, av2[seg * (OW / 2)] &= TWO ? 0xFFFF0000u : 0u;
                            if (sh > 0)   // x = OW-1
                                av[seg * (OW / 2) + OW / 2 - 1] &= 0x0000FFFFu,
                                    av2[seg * (OW / 2) + OW / 2 - 1] &= TWO ? 0x0000FFFFu : 0u;
                        }
                    }
                    if (tg == 0 && st < 64 && t == 0) WG_TRACE(3701 + 4 * st + 2 * sub);
                    tmem_st16(lane_base + acol, av);
                    if (TWO) tmem_st16(lane_base + acol + 16, av2);
                    }
                    };
                    if constexpr (kFast2) {
                        if (fast2) rows(std::true_type{});
                        else rows(std::false_type{});
                    } else {
                        rows(std::false_type{});
                    }
                } else if (FAST_OK && !TAP && pre) {
                    // GENERIC-PRE: the reference's fp32 relu(decode) (table hi +
                    // lo, exact) as three bf16 pieces in pair words (k, k + 4)
                    // like the B rows; each group takes one 8-pixel group
                    const float *lut = s_lut + (size_t)(c - c_begin) * lut_stride;
                    const bool live = rok[t];
#pragma unroll 1
                    for (int q8 = gsplit; q8 < 4; q8 += gstride) {
                        float a8[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const int i = 8 * q8 + k;
                            const int seg = i / OW, x = i - seg * OW;
                            const int iy = y0 + seg + u - p.pad, sx = x + sh;
                            float a = 0.f;
                            if (live && iy >= 0 && iy < p.h && sx >= 0 && sx < OW) {
                                const uint32_t *cw = reinterpret_cast<const uint32_t *>(cst);
                                const int bp = (cbox + iy * p.rb - wbase) * 8 + sx * BITS;
                                const uint32_t code = __funnelshift_r(cw[bp >> 5], cw[(bp >> 5) + 1],
                                                                      bp & 31) & ((1u << BITS) - 1u);
                                a = lut[code];
                            }
                            a8[k] = a;
                        }
                        uint32_t H[4], M[4], L[4];
#pragma unroll
                        for (int k = 0; k < 4; ++k) split3_bf16x2(a8[k], a8[k + 4], H[k], M[k], L[k]);
                        tmem_st4(lane_base + acol + 4 * q8, H[0], H[1], H[2], H[3]);
                        tmem_st4(lane_base + acol + 16 + 4 * q8, M[0], M[1], M[2], M[3]);
                        tmem_st4(lane_base + acol + 32 + 4 * q8, L[0], L[1], L[2], L[3]);
                    }
                } else {
                    // a compact loop of 4-pixel quads (x4 TMEM stores): the
                    // fully unrolled form overflows the instruction cache
                    const float *lut = s_lut + (size_t)(c - c_begin) * lut_stride;
                    const bool live = rok[t];
#pragma unroll 1
                    for (int q4 = gsplit; q4 < 8; q4 += gstride) {
                        uint32_t h[4] = {0u, 0u, 0u, 0u}, l[4] = {0u, 0u, 0u, 0u};
                        if (live && intm) {
                            // INT: relu(m) = max(2 code + b, 0) < 2048, exact in TF32
                            // (no lo piece, no A_lo pass); step / 2 in the epilogue
                            const int b = (int)s_bc[c - c_begin];
                            const uint32_t *cw = reinterpret_cast<const uint32_t *>(cst);
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const int i = 4 * q4 + k;
                                const int seg = i / OW, x = i - seg * OW;
                                const int iy = y0 + seg + u - p.pad, sx = x + sh;
                                const int bp = (cbox + iy * p.rb - wbase) * 8 + sx * BITS;
                                const uint32_t code = __funnelshift_r(cw[bp >> 5], cw[(bp >> 5) + 1],
                                                                      bp & 31) & ((1u << BITS) - 1u);
                                const bool in = iy >= 0 && iy < p.h && sx >= 0 && sx < OW;
                                const int m = max(2 * (int)code + b, 0);
                                h[k] = in ? __float_as_uint((float)m) : 0u;
                            }
                        } else if (live) {
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const int i = 4 * q4 + k;
                                const int seg = i / OW, x = i - seg * OW;
                                generic_px(p, cst, cbox, wbase, nn, c, y0 + seg + u - p.pad, x + sh,
                                           OW, lut, h[k], l[k]);
                            }
                        }
                        tmem_st4(lane_base + acol + 4 * q4, h[0], h[1], h[2], h[3]);
                        if (!intm) tmem_st4(lane_base + acol + 32 + 4 * q4, l[0], l[1], l[2], l[3]);
                    }
                }
            }
            }   // sub
            tmem_wait_st();
            if (coop) {
                fence_async_smem();
                tc_fence_before();
                asm volatile("bar.sync 3, %0;" ::"n"(kWgThreads - 64) : "memory");
                if (grp == 0) {
                    mbar_arrive(&raw_empty[s]);
                    mbar_arrive(&op_full[o]);
                }
            } else {
                mbar_arrive(&raw_empty[s]);      // raw slots (g tiles + codes) free for TMA
                fence_async_smem();
                tc_fence_before();
                if (tg == 0 && st < 64) WG_TRACE(5 + 5 * st);
                if (tg == 96 && st < 64) WG_TRACE(400 + 2 * st);
                mbar_arrive(&op_full[o]);
            }
            s += sstep;
            if (s >= RG) { s -= RG; phr ^= 1u; }   // RG is a multiple of sstep
            o += sstep;
            if (o >= ops) { o -= ops; pho ^= 1u; }
        }
        // epilogue: all four groups drain TMEM -- items (tile, tap, 16-column
        // chunk) dealt round-robin over the groups, each warp its lane
        // quarter (lane = act row); FAST sums the three g pieces and scales
        // by step/2.  Warps whose 32 rows are all past the tile skip.
        if (coop || grp < ops) mbar_wait(done, 0);   // groups that ran stages: short tail
        else mbar_wait_idle(done, 0);         // idle groups (ring shallower than 4)
        if (tg == 0 && grp == 0) WG_TRACE(330);
        tc_fence_after();
        constexpr int kChunks = NT * (BN / 16);              // items per tile
        const int items = mt_here * kChunks;
        // fp32 throughout: the pieces sum to within an ulp and fp64 converts
        // (16/clk/SM) would pace the drain
        float scale[2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int rl = t * 128 + 32 * quarter + lane;
            scale[t] = ((fastb || intm) && rl < nrows) ? (float)(0.5 * p.tape.step[(row0 + rl) / kk]) : 1.f;
        }
#pragma unroll 1
        for (int it = grp; it < items; it += kWgGroups) {
            const int t = it >= kChunks ? 1 : 0;
            const int ic = it - t * kChunks;
            const int v = ic / (BN / 16), cb = (ic - v * (BN / 16)) * 16;
            if (t * 128 + 32 * quarter >= nrows) continue;   // warp-uniform
            const int rl = t * 128 + 32 * quarter + lane;
            const bool ok = rl < nrows;
            const int r = row0 + rl;
            const int rout = TAP ? r * 3 + v : r;            // dW row (ci, u, v); TAP rows (ci, u)
            const uint32_t tbase = lane_base + (uint32_t)t * (pieces ? FACC : GACC);
            uint32_t r0[16], r1[16], r2[16];
            if (pieces && STACK) {
                tmem_ld16(tbase + (0 * NT + v) * BN + cb, r0);
                tmem_ld16(tbase + (1 * NT + v) * BN + cb, r1);
                tmem_ld16(tbase + (2 * NT + v) * BN + cb, r2);
            } else {
                tmem_ld16(tbase + v * BN + cb, r0);
            }
            tmem_wait_ld();
            if (ok) {
                const float sc = t ? scale[1] : scale[0];
                float *dst = p.partial + ((int64_t)split * p.co + co0 + cb) * p.Rout + rout;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    float acc = __uint_as_float(r0[j]);
                    if (pieces && STACK)   // hi + (mid + lo): the small pieces first
                        acc = __fadd_rn(acc, __fadd_rn(__uint_as_float(r1[j]), __uint_as_float(r2[j])));
                    const float val = (fastb || intm) ? __fmul_rn(acc, sc) : acc;
                    if (co0 + cb + j < p.co) dst[(int64_t)j * p.Rout] = val;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) WG_TRACE(331);
    if (threadIdx.x == 0 && tr_)
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_[333]));
    if (threadIdx.x == 0 && p.trace && blockIdx.y == 0 && blockIdx.z == 0 && blockIdx.x < 1024)
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(p.trace[601 + 3 * blockIdx.x]));
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

struct WgPlan {
    bool ok = false;
    int bn = 0, mtg = 0, mgroups = 0, splits = 0, cps = 0, total = 0, rg = 0, smem = 0;
    int ops = 0, ops_g = 0;                               // FAST / GENERIC operand stages
    int nch = 0, rb = 0, cb = 0, cbytes = 0, slot = 0;    // code box (codes tapes)
    int lut_floats = 0, nolut = 0;                        // nolut: GENERIC decodes inline
    int opreg = 0;                                        // operand region bytes
    int pre = 0, bring = 0;                               // pieces by TMA; B ring depth
    int ops2 = 0;                                         // FAST2 operand stages (0: INT)
    int tap = 0, rpc = 0;                                 // column taps in N; A rows per channel
    int fbox = 0;                                         // fp32 source boxed per stage
    int nblk = 1;                                         // output-channel blocks of BN
};

template <int BN, int OW, int BITS, bool TAP = false>
static int launch_wg2(const CUtensorMap &m, const CUtensorMap &mc, const WgParams &p,
                      const WgPlan &pl, cudaStream_t st) {
    auto kern = conv_wgrad_tc_kernel<BN, OW, BITS, TAP>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = true;
    }
    launch_pdl(kern, dim3(pl.splits, pl.mgroups, pl.nblk), kWgThreads, pl.smem, st, m, mc, p);
    QT_CHECK_LAUNCH();
    return QT_OK;
}

// specialised code widths: 4 bits (FAST-capable), 2 and 8 bits; 0 = runtime
// width or an fp32 source
template <int BN, int OW>
static int launch_wg1(const CUtensorMap &m, const CUtensorMap &mc, const WgParams &p,
                      const WgPlan &pl, cudaStream_t st) {
    if constexpr (BN <= 32) {
        if (pl.tap) return launch_wg2<BN, OW, 4, true>(m, mc, p, pl, st);
    }
    switch (p.lut ? p.tape.bits : 0) {
        case 4: return launch_wg2<BN, OW, 4>(m, mc, p, pl, st);
        case 2: return launch_wg2<BN, OW, 2>(m, mc, p, pl, st);
        case 1: return launch_wg2<BN, OW, 1>(m, mc, p, pl, st);
        case 8: return launch_wg2<BN, OW, 8>(m, mc, p, pl, st);
        default: return launch_wg2<BN, OW, 0>(m, mc, p, pl, st);
    }
}

template <int BN>
static int launch_wg(const CUtensorMap &m, const CUtensorMap &mc, const WgParams &p,
                     const WgPlan &pl, cudaStream_t st) {
    switch (p.ow) {
        case 8: return launch_wg1<BN, 8>(m, mc, p, pl, st);
        case 16: return launch_wg1<BN, 16>(m, mc, p, pl, st);
        case 32: return launch_wg1<BN, 32>(m, mc, p, pl, st);
    }
    return QT_EUNSUPPORTED;
}

}  // namespace qt
