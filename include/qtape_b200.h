/*
 * qtape_b200 -- C ABI of the B200-native approximate-activation training step
 * (arXiv 1901.07988).  Built from paper_1901_07988_b200/csrc into
 * paper_1901_07988_b200/libqtape_b200.so (sm_100a).
 *
 * Conventions
 *   - every pointer is a DEVICE pointer (cudaMalloc'd / torch.cuda storage)
 *     unless stated; tensors are C-contiguous NCHW float32 ("rank 4") or
 *     (N, C) ("rank 2", pass hw = 1);
 *   - packed codes use the reference bit layout exactly: code i of the flat
 *     NCHW tensor at bits [i*K, (i+1)*K), little-endian inside a byte, tail
 *     of the last byte zero (reference codec.py:59-78);
 *   - `stream` is a cudaStream_t (the caller's current torch stream); every
 *     call is stream-ordered, never synchronises, never allocates, and is
 *     safe inside CUDA-graph capture;
 *   - workspaces are caller-owned; their size comes from qt_*_workspace();
 *   - return value: 0 (QT_OK), a negative QT_E* code for an argument error
 *     detected before launch, or a positive cudaError_t from the launch.
 *     There is no CPU fallback anywhere.
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/qtape/<file>:<line>).
 */
#ifndef QTAPE_B200_H
#define QTAPE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QT_OK 0
#define QT_EINVAL (-1)        /* bad extents / pointer / bit width          */
#define QT_EUNSUPPORTED (-2)  /* shape outside what the kernels implement  */

typedef void *qt_stream_t;    /* cudaStream_t */

int qt_version(void);
const char *qt_error_string(int status);
int qt_num_sms(void);
/* SM partition for a backward pass that runs the data gradients and the
 * weight gradients concurrently on two streams (the engine's side-stream
 * weight gradients, engine.py Workspace): when on, layers under 2^30 MACs
 * launch their data-gradient and weight-gradient GEMMs on half the SMs each,
 * so the two chains run side by side instead of queueing for every SM.
 * Off (the default): both use every SM.  Returns the previous setting. */
int qt_set_concurrent_backward(int on);

/* ---------------------------------------------------------------- codec ---
 * Per-channel codec constants (codec.py:27-29, :101-104, :117):
 *   step[c]   = 6*max(|gamma_c|,1e-8) * 2^-K           (float64)
 *   offset[c] = floor(beta_c * 2^K/(6*max(|gamma_c|,1e-8)))  (int64, x86 cast)
 */
int qt_codec_constants(const float *gamma, const float *beta, int64_t c, int bits,
                       double *step, int64_t *offset, qt_stream_t stream);

/* Quantize + pack a pre-ReLU activation tensor a (N,C,HW).
 * Replaces codec.quantize (codec.py:123-143) incl. raw_codes (:107-120) and
 * pack_codes (:59-78).  clip_count (one int64, device) is ACCUMULATED into. */
int qt_quantize_pack(const float *a, int64_t n, int64_t c, int64_t hw,
                     const float *gamma, const float *beta, int bits,
                     uint8_t *codes, double *step, int64_t *offset,
                     int64_t *clip_count, qt_stream_t stream);

/* Decode a tape to interval medians (codec.dequantize, codec.py:146-156;
 * unpack_codes :81-98).  relu != 0 additionally applies max(.,0). */
int qt_unpack_dequant(const uint8_t *codes, int64_t n, int64_t c, int64_t hw,
                      int bits, const double *step, const int64_t *offset,
                      int relu, float *out, qt_stream_t stream);

/* Raw bit packing of uint8 codes (pack_codes / unpack_codes, codec.py:59-98).
 * qt_pack_codes writes ceil(count*K/8) bytes; out-of-range codes set
 * *bad (device int32) to 1 (caller raises CodecError). */
int qt_pack_codes(const uint8_t *codes, int64_t count, int bits, uint8_t *packed,
                  int32_t *bad, qt_stream_t stream);
int qt_unpack_codes(const uint8_t *packed, int64_t count, int bits, uint8_t *codes,
                    qt_stream_t stream);

/* ------------------------------------------------------------------- BN ---
 * Per-channel population mean/var over (N,HW), float64 (ops.channel_moments,
 * ops.py:186-196).  If running_mean/var are non-NULL they are updated as
 * layer.py:237-241 (r = 0.9 r; r += (1-0.9) batch).  ws: qt_bn_stats_workspace. */
int64_t qt_bn_stats_workspace(int64_t n, int64_t c, int64_t hw);
int qt_bn_stats(const float *x, int64_t n, int64_t c, int64_t hw,
                double *mean, double *var, double *running_mean, double *running_var,
                void *ws, qt_stream_t stream);

/* Per-channel float64 sum over (N,HW) (ops.channel_sum, ops.py:199-201);
 * ws: qt_bn_stats_workspace. */
int qt_channel_sum(const float *x, int64_t n, int64_t c, int64_t hw, double *out,
                   void *ws, qt_stream_t stream);

/* Fused forward K1: BN apply (4 rounded fp32 ops, layer.py:245-249) ->
 * tape -> ReLU (layer.py:264).  mode: 0 exact, 1 approx, 2 naive
 * (layer.py:32); bits 0 = identity bypass (layer.py:256-258).
 *   a3_out      : ReLU'd activations for the linear transform (the `work` slot)
 *   a2_tape     : fp32 pre-ReLU copy (exact / bypass tapes), else NULL
 *   codes/step/offset/clip_count : K-bit tape (approx / naive), else NULL
 * training == 0 uses mean/var as given (running stats) and writes no tape. */
int qt_bn_relu_forward(const float *x, int64_t n, int64_t c, int64_t hw,
                       const double *mean, const double *var, double eps,
                       const float *gamma, const float *beta, int mode, int bits,
                       float *a3_out, float *a2_tape, uint8_t *codes, double *step,
                       int64_t *offset, int64_t *clip_count, const void *consts,
                       qt_stream_t stream);

/* Training-mode fusion of the layer's per-channel work in ONE launch:
 * qt_bn_stats + the constants of qt_bn_relu_forward (pass the same `consts`
 * buffer, 48 bytes per channel, to it) + the frozen gamma/beta tape copies
 * + the tape's step/offset + zeroing the clip counter (layer.py:236-255). */
int qt_bn_stats_prep(const float *x, int64_t n, int64_t c, int64_t hw, double eps,
                     const float *gamma, const float *beta, int bits, double *mean,
                     double *var, double *running_mean, double *running_var,
                     float *gamma_copy, float *beta_copy, double *step, int64_t *offset,
                     int64_t *clip_count, void *consts, void *ws, qt_stream_t stream);

/* qt_bn_stats_prep + qt_bn_relu_forward in ONE launch (layer.py:236-264):
 * the same cluster partition and arithmetic as the two-launch path (mean /
 * var bit-identical), then each block applies BN -> tape -> ReLU to its own
 * planes from a shared-memory copy of x staged during the statistics pass.
 * clip_count is ACCUMULATED (the caller zeroes it).  hw % 8 == 0
 * (qt_bn_forward_fused_ok); QT_EUNSUPPORTED otherwise. */
int qt_bn_forward_fused_ok(int64_t n, int64_t c, int64_t hw);
int qt_bn_forward_fused(const float *x, int64_t n, int64_t c, int64_t hw, double eps,
                        const float *gamma, const float *beta, int mode, int bits,
                        double *mean, double *var, double *running_mean, double *running_var,
                        float *gamma_copy, float *beta_copy, double *step, int64_t *offset,
                        int64_t *clip_count, void *consts, float *a3_out, float *a2_tape,
                        uint8_t *codes, qt_stream_t stream);

/* Tape source descriptor used by the backward kernels: either a fp32 pre-ReLU
 * tape (a2 != NULL) or packed codes + frozen constants. */
typedef struct {
    const float *a2;        /* exact tape, or NULL                     */
    const uint8_t *codes;   /* packed codes, or NULL                   */
    const double *step;     /* [C] frozen decode step                  */
    const int64_t *offset;  /* [C] frozen decode offset                */
    int bits;
} qt_tape_t;

/* Rebuild (a1, a2, a3) from a tape (layer.reconstruct_from_tape,
 * layer.py:269-283).  Any output may be NULL. */
int qt_reconstruct(qt_tape_t tape, int64_t n, int64_t c, int64_t hw,
                   const float *gamma_tape, const float *beta_tape,
                   float *a1, float *a2, float *a3, qt_stream_t stream);

/* Backward of mask + scale/bias + normalization (layer.py:353-381 and
 * bn_input_gradient :286-308), in two launches.
 *   g3  : gradient w.r.t. the rectified activations (dgrad output), (N,C,HW)
 *   reduce: accumulates grad_beta += sum(g3*mask), grad_gamma += sum(a1*g3*mask)
 *           and writes stats[3*C] = {t2[C], t3[C], inv[C]} (float32)
 *   apply : g_in = ((g1 - t2) - a1v*t3) * inv, g1 = g3*mask*gamma, in place
 *           (ws = the workspace the reduce wrote its per-code tables into)
 *           allowed (g_in == g3); if res_g != NULL also adds the shortcut
 *           adjoint (engine.py:272-279): res_g has shape (N,CR,HR,WR) with
 *           HR = H/sc, CR >= C.
 * variance_a1 (nullable) replaces a1 in the variance term (diagnostics). */
int64_t qt_bn_backward_workspace(int64_t n, int64_t c, int64_t hw);
int qt_bn_backward_reduce(const float *g3, qt_tape_t tape, int64_t n, int64_t c,
                          int64_t hw, const float *gamma_tape, const float *beta_tape,
                          const double *sigma2, double eps, const float *variance_a1,
                          float *grad_gamma, float *grad_beta, float *stats, void *ws,
                          qt_stream_t stream);
int qt_bn_backward_apply(const float *g3, qt_tape_t tape, int64_t n, int64_t c,
                         int64_t h, int64_t w, const float *gamma_tape,
                         const float *beta_tape, const float *variance_a1,
                         const float *stats, const float *res_g, int64_t cr,
                         int64_t sc, const void *ws, float *g_in, qt_stream_t stream);

/* ----------------------------------------------------------------- conv ---
 * Cross-correlation with zero padding; integral extents are validated by the
 * caller (ops.conv2d_out_shape, ops.py:80-94).
 * Forward (ops.conv2d_forward ops.py:106-138; _kernels.c:10-52):
 *   out = conv(x, w) (+ shortcut(res) if res != NULL, engine.py:262-269;
 *   res is (N, CR, HR, WR) with CR <= Co and HR = OH*sr). */
int qt_conv_forward(const float *x, const float *w, float *out,
                    int64_t n, int64_t ci, int64_t h, int64_t wd, int64_t co,
                    int64_t kh, int64_t kw, int64_t stride, int64_t pad,
                    const float *res, int64_t cr, int64_t sr, void *ws,
                    qt_stream_t stream);

/* Fused forward of one pre-activation layer around the forward GEMM.
 * Replaces, for shapes qt_conv_fused_support accepts, the reference's
 * layer_forward sequence channel_moments -> BN apply -> codec.quantize ->
 * ReLU -> conv2d_forward (layer.py:236-266, codec.py:123-143, ops.py:106-138):
 *   pro != NULL: x is the layer's PRE-BN input; the operand staging applies
 *     ((x - mean32) * inv32) * gamma + beta (4 rounded fp32 ops) from the
 *     layer's BnConst table `consts` (written by qt_bn_stats_prep or by the
 *     previous conv's statistics epilogue), ReLU, zero padding AFTER the
 *     apply, and writes the K-bit packed tape of A2 (bit-identical to
 *     qt_bn_relu_forward's) and ACCUMULATES its clip count.  The rectified
 *     activation never exists in memory.
 *   epi != NULL: the output (after the fused shortcut add) gets the NEXT
 *     layer's batch statistics and all of qt_bn_stats_prep's outputs for it
 *     (mean, var, running stats, BnConst, frozen gamma/beta, step/offset,
 *     clip counter zeroed); epi->ws holds qt_conv_stats_workspace(co) bytes,
 *     zeroed once by the caller (the kernel leaves its counters at zero).
 * Both NULL: exactly qt_conv_forward. */
typedef struct {
    const void *consts;     /* BnConst[ci] (48 B each) of this layer           */
    uint8_t *codes;         /* packed K-bit tape of this layer (4-byte aligned) */
    int64_t *clip_count;    /* accumulated                                      */
    int bits;               /* 1, 2, 4, 8                                       */
} qt_bn_prologue_t;
typedef struct {
    double eps;
    const float *gamma, *beta;   /* next layer's parameters                    */
    int bits;                    /* next layer's tape width (0: exact tape)     */
    double *mean, *var, *running_mean, *running_var;
    float *gamma_copy, *beta_copy;
    double *step;
    int64_t *offset;
    int64_t *clip_count;
    void *consts;
    void *ws;
} qt_bn_stats_epilogue_t;
int64_t qt_conv_stats_workspace(int64_t co);
/* Bit 0: the BN prologue is available for this shape at `bits`; bit 1: the
 * statistics epilogue is (sr = the fused shortcut's stride, 1 if none). */
int qt_conv_fused_support(int64_t n, int64_t ci, int64_t h, int64_t wd, int64_t co,
                          int64_t kh, int64_t kw, int64_t stride, int64_t pad, int64_t sr,
                          int bits);
int qt_conv_forward_fused(const float *x, const float *w, float *out,
                          int64_t n, int64_t ci, int64_t h, int64_t wd, int64_t co,
                          int64_t kh, int64_t kw, int64_t stride, int64_t pad,
                          const float *res, int64_t cr, int64_t sr,
                          const qt_bn_prologue_t *pro, const qt_bn_stats_epilogue_t *epi,
                          void *ws, qt_stream_t stream);

/* Data gradient (ops.conv2d_backward g_x path, ops.py:168-183). */
int qt_conv_dgrad(const float *g, const float *w, float *gx,
                  int64_t n, int64_t ci, int64_t h, int64_t wd, int64_t co,
                  int64_t kh, int64_t kw, int64_t stride, int64_t pad, void *ws,
                  qt_stream_t stream);

/* Prepared weight operands.  On the tensor-core path qt_conv_forward /
 * qt_conv_dgrad first re-lay the kernel into (hi, lo) TF32 halves in `ws`
 * ([kh*kw][rows][cols] each; rows = co, cols = ci for the forward, rows = ci,
 * cols = co of the 180-degree-flipped kernel for the data gradient).  Passing
 * w == NULL means `ws` already holds that operand -- prepared for many layers
 * at once by qt_conv_prepare_weights (one launch per optimizer step instead
 * of one per conv call).  `descs` is a DEVICE array of `count` descriptors;
 * max_elems = max over descriptors of rows*cols*kh*kw.  w == NULL is an error
 * for shapes that run on the CUDA cores. */
typedef struct {
    const float *w;   /* original (co, ci, kh, kw) kernel */
    float *out;       /* 2 * rows * cols * kh * kw floats: hi then lo */
    int32_t rows, cols, kh, kw, flip, pad_;
} qt_wprep_t;
int qt_conv_prepare_weights(const qt_wprep_t *descs, int64_t count, int64_t max_elems,
                            qt_stream_t stream);

/* Scratch for qt_conv_forward / qt_conv_dgrad: size it with
 * qt_conv_workspace_ex (below), which covers every path; qt_conv_workspace
 * alone covers the weight operand only.  The tensor-core path keeps the
 * (hi, lo) TF32 split of the re-laid-out kernel there (2*ci*co*kh*kw floats).
 * The tensor-core path serves stride-1 convs whose output rows are 8, 16 or
 * 32 pixels wide with ci % 8 == 0 and co % 16 == 0 (every CIFAR ResNet conv
 * except the stem and the 2x2/s2 transitions); other shapes run on the
 * CUDA-core implicit GEMM.  QTAPE_NO_TC=1 forces the CUDA-core path. */
int64_t qt_conv_workspace(int64_t ci, int64_t co, int64_t kh, int64_t kw);
/* Full scratch for qt_conv_forward / qt_conv_dgrad of one shape (>= the
 * above): non-overlapping convs (kernel == stride, pad 0, e.g. the 2x2/s2
 * transitions) run as tensor-core 1x1 convs of the space-to-depth tensor,
 * which lives in this workspace after the weight operand. */
int64_t qt_conv_workspace_ex(int64_t n, int64_t ci, int64_t h, int64_t wd, int64_t co,
                             int64_t kh, int64_t kw, int64_t stride, int64_t pad);
/* 1 if qt_conv_forward (dgrad = 0) / qt_conv_dgrad (dgrad = 1) of this shape
 * runs on the tensor cores, 0 if on the CUDA cores (host-side query). */
int qt_conv_uses_tc(int64_t n, int64_t ci, int64_t h, int64_t wd, int64_t co, int64_t kh,
                    int64_t kw, int64_t stride, int64_t pad, int dgrad);

/* Weight gradient, accumulated: grad_w += fp32(sum) (ops.py:164-167,
 * layer.py:167).  The activation operand comes from `act`:
 *   act.a2 with relu   -> exact tape
 *   act.codes          -> relu(decode(codes)) fused into operand staging
 *   x_plain != NULL    -> the plain input (stem, layer.py:340-342). */
int64_t qt_conv_wgrad_workspace(int64_t n, int64_t ci, int64_t h, int64_t wd,
                                int64_t co, int64_t kh, int64_t kw, int64_t stride,
                                int64_t pad);
int qt_conv_wgrad(const float *g, qt_tape_t act, const float *x_plain, float *grad_w,
                  int64_t n, int64_t ci, int64_t h, int64_t wd, int64_t co,
                  int64_t kh, int64_t kw, int64_t stride, int64_t pad,
                  void *ws, qt_stream_t stream);

/* ---------------------------------------------------------- dense / head ---
 * C[M,N] (=|+=) fp32( sum_k A[m,k] B[k,n] ) with float64 accumulation in
 * ascending k, one rounding per multiply and add: bit-identical to
 * ops.matmul (ops.py:54-77).  ta/tb: operand stored transposed. */
int qt_matmul(const float *a, const float *b, float *c, int64_t m, int64_t k,
              int64_t nn, int ta, int tb, int accumulate, qt_stream_t stream);
/* Global average pool (N,C,HW)->(N,C), float64 mean (layer._gap :154-157). */
int qt_gap(const float *x, int64_t n, int64_t c, int64_t hw, float *out,
           qt_stream_t stream);
/* out[n,c,:] = fp32(g[n,c] / hw) broadcast (layer.py:173-179). */
int qt_gap_backward(const float *g, int64_t n, int64_t c, int64_t hw, float *out,
                    qt_stream_t stream);
/* Mean softmax cross-entropy (training.softmax_xent, training.py:120-134).
 * loss: float64 buffer of 1 + N slots (slot 0 = loss, the rest per-row nll
 * scratch); grad (N,C) fp32; labels int64; *bad_label set to 1 if a label
 * lies outside [0, C) (caller raises DataError). */
int qt_softmax_xent(const float *logits, const int64_t *labels, int64_t n, int64_t c,
                    double *loss, float *grad, int32_t *bad_label, qt_stream_t stream);
/* Momentum SGD on a contiguous slab (training.sgd_step, training.py:98-117);
 * zeroes grad afterwards.  If lr_dev != NULL the learning rate is read from
 * device memory (so a captured CUDA graph follows a schedule). */
int qt_sgd(float *value, float *grad, float *vel, int64_t count, float lr,
           const float *lr_dev, float momentum, float weight_decay, qt_stream_t stream);

/* ------------------------------------------------------------ input data ---
 * Device-side CIFAR-10 pipeline (data.py:45-87, :182-206), bit-identical to
 * the reference's numpy arithmetic.
 * qt_cifar_decode: n binary records (3073 B: label byte + 3072 channel-major
 * pixels, data.py:20, :52-57) -> labels (int64) and images fp32 = u8 / 255;
 * *bad_label = 1 if a label byte exceeds 9 (DataError, data.py:73-74).
 * qt_standardize: images = (images - mean[c]) / std[c] in fp32 (data.py:84-85).
 * qt_gather_augment: dst[i] = src[idx[i]] (idx NULL: src[i]) horizontally
 * flipped where flip[i] != 0 (flip NULL: none), then translated to
 * padded[:, dy:dy+h, dx:dx+w] of a zero border of `pad` pixels with
 * (dy, dx) = offsets[2i], offsets[2i+1] (offsets NULL: no translation). */
int qt_cifar_decode(const uint8_t *records, int64_t n, float *images, int64_t *labels,
                    int32_t *bad_label, qt_stream_t stream);
int qt_standardize(float *images, int64_t n, int64_t c, int64_t hw, const float *mean,
                   const float *std_, qt_stream_t stream);
int qt_gather_augment(const float *src, const int64_t *idx, int64_t n, int64_t c, int64_t h,
                      int64_t w, const uint8_t *flip, const int32_t *offsets, int pad,
                      float *dst, qt_stream_t stream);

/* ------------------------------------------------------------ engine glue ---
 * res = copy(x) and shortcut add / adjoint (engine.py:262-279) as standalone
 * kernels (the fused forms live in qt_conv_forward / qt_bn_backward_apply). */
int qt_copy(const float *src, float *dst, int64_t count, qt_stream_t stream);
int qt_shortcut_add(float *cur, const float *res, int64_t n, int64_t c, int64_t h,
                    int64_t w, int64_t cr, int64_t sr, qt_stream_t stream);
int qt_shortcut_adjoint(float *g_in, const float *g_res, int64_t n, int64_t c,
                        int64_t h, int64_t w, int64_t cres, int64_t sr,
                        qt_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* QTAPE_B200_H */
