/*
 * b2dl.h — C ABI of the B200-native DeepLabv3+/FC-DenseNet training-step library
 * (libb2dl.so).  Plain C: raw device pointers, sizes, a cudaStream_t passed as
 * void*.  No torch types cross this boundary.
 *
 * Two groups of entry points:
 *
 *  (1) Reference-shaped convolution kernels.  These are the drop-in for the
 *      reference's kernel-backend protocol (pkg/src/deskdl/model/kernels.py:36-40)
 *      and its compiled core (pkg/src/deskdl/model/_convkernels.pyx:16-71):
 *      NCHW fp32 tensors, "same" padding with the TF split
 *      (_kernels_py.py:18-21), stride 1 only, any dilation.  Validation errors
 *      are returned as codes that the Python shim maps to the reference's
 *      exceptions (NotImplementedError / ValueError).
 *
 *  (2) The NHWC bf16 fast path used by the training step: tcgen05 implicit-GEMM
 *      convolution (forward + dgrad share one kernel, wgrad is split-K), the
 *      fused weighted cross-entropy, the LARC multi-tensor update and the
 *      memory-bound pool / upsample / mask / bias-gradient kernels.
 *
 * Every function returns 0 on success or a B2DL_E* code.  All launches are
 * asynchronous on the given stream; the caller owns every buffer.
 */
#ifndef B2DL_H
#define B2DL_H
#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define B2DL_API __attribute__((visibility("default")))
#else
#define B2DL_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
  B2DL_OK = 0,
  B2DL_E_NOT_IMPLEMENTED = 1, /* stride != 1            -> NotImplementedError */
  B2DL_E_VALUE = 2,           /* shape / channel errors  -> ValueError          */
  B2DL_E_CUDA = 3,            /* launch or driver error  -> RuntimeError        */
  B2DL_E_ALIGN = 4,           /* TMA alignment violated  -> ValueError          */
  B2DL_E_NONFINITE = 5        /* LARC non-finite norm    -> FloatingPointError  */
};

/* NHWC bf16 (or fp32 where stated) activation view.  `ptr` points at element
 * (0,0,0,c_off) of a buffer whose pixel pitch is `c_stride` channels; the view
 * covers `c` channels.  Concat buffers are shared by several views. */
typedef struct b2dl_act {
  void* ptr;
  int n, h, w;
  int c;
  int c_stride;
} b2dl_act;

/* ---------------------------------------------------------------- (1) reference-shaped */

/* Reference-precision core (csrc/refconv.cu): the Cython core's fused type
 * (_convkernels.pyx:11-13, float32 / float64) -- NCHW tensors of `dtype`, computed in
 * that type (fp32 FFMA / fp64 DFMA), "same" padding, stride 1, any dilation.  No
 * workspace; outputs are fully overwritten (the core zero-fills, pyx:23,42,61).
 * These are what the drop-in backend (backend.py, BACKEND_NAME "b200") calls. */
enum { B2DL_DTYPE_F32 = 0, B2DL_DTYPE_F64 = 1 };

/* Replaces conv2d_forward_core (_convkernels.pyx:16-32) + _kernels_py.conv2d_forward (:44-55). */
B2DL_API int b2dl_conv2d_forward_typed(int dtype, const void* x, const void* w, void* y, int n, int cin, int h,
                                       int wd, int cout, int kh, int kw, int stride, int dilation, void* stream);
/* Replaces conv2d_backward_input_core (_convkernels.pyx:35-51) + _kernels_cy.py:34-44. */
B2DL_API int b2dl_conv2d_backward_input_typed(int dtype, const void* dy, const void* w, void* dx, int n, int cin,
                                              int h, int wd, int cout, int kh, int kw, int stride, int dilation,
                                              void* stream);
/* Replaces conv2d_backward_weights_core (_convkernels.pyx:54-71) + _kernels_cy.py:28-31. */
B2DL_API int b2dl_conv2d_backward_weights_typed(int dtype, const void* x, const void* dy, void* dw, int n, int cin,
                                                int h, int wd, int cout, int kh, int kw, int dilation, void* stream);

/* bf16 tensor-core variants of the same three products (fp32 NCHW in / out, operands rounded
 * to bf16, fp32 accumulation): the training step's arithmetic, opt-in backend "b200-bf16".
 * Workspace bytes needed by these entry points for this shape: */
B2DL_API size_t b2dl_conv2d_workspace_size(int n, int cin, int h, int w, int cout, int kh, int kw);

/* y[n,cout,h,w] = conv(x[n,cin,h,w], w[cout,cin,kh,kw]), same padding.
 * Replaces _kernels_py.conv2d_forward (_kernels_py.py:44-55) and
 * _convkernels.conv2d_forward_core (_convkernels.pyx:16-32). */
B2DL_API int b2dl_conv2d_forward(const float* x, const float* w, float* y, int n, int cin, int h, int wd, int cout,
                        int kh, int kw, int stride, int dilation, void* workspace, size_t workspace_bytes,
                        void* stream);

/* dx[n,cin,h,w] from dy[n,cout,h,w].  Replaces _kernels_py.conv2d_backward_input
 * (_kernels_py.py:65-83) and conv2d_backward_input_core (_convkernels.pyx:35-51). */
B2DL_API int b2dl_conv2d_backward_input(const float* dy, const float* w, float* dx, int n, int cin, int h, int wd,
                               int cout, int kh, int kw, int stride, int dilation, void* workspace,
                               size_t workspace_bytes, void* stream);

/* dw[cout,cin,kh,kw] from x and dy.  Replaces _kernels_py.conv2d_backward_weights
 * (_kernels_py.py:58-62) and conv2d_backward_weights_core (_convkernels.pyx:54-71). */
B2DL_API int b2dl_conv2d_backward_weights(const float* x, const float* dy, float* dw, int n, int cin, int h, int wd,
                                 int cout, int kh, int kw, int dilation, void* workspace,
                                 size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------- (2) NHWC fast path */

/* Implicit-GEMM convolution on tcgen05 (stride 1, same padding):
 *   y = epilogue( sum_{tap,ci} x[p + off(tap), ci] * w_packed[co, tap, ci] )
 * epilogue: +bias[co], +residual, relu, y_old + (accumulate), *(mask > 0).
 * w_packed: bf16 [cout][kh*kw][cin_pad], cin_pad = b2dl_cin_pad(cin).
 * Used for the forward conv and, with dgrad-packed weights and swapped pads,
 * for the input gradient (the reference's conv2d_backward_input). */
typedef struct b2dl_conv_args {
  b2dl_act x;
  const void* w_packed;
  int cout, kh, kw, dilation, pad_top, pad_left;
  b2dl_act y;
  int y_f32;
  const float* bias;
  b2dl_act residual;
  int relu;
  int accumulate;
  b2dl_act mask;
  int block_n; /* 0 = auto */
  /* weight source: 0 = w_packed; 1 = w_master, the forward conv's bf16 HWIO
   * [kh*kw][cin][cout] copy read as an MN-major operand (forward); 2 = w_master of the
   * forward conv read tap-flipped as the input gradient's K-major operand (dgrad).
   * Modes 1/2 need the forward cout % 8 == 0; they remove all weight repacking. */
  const void* w_master;
  int w_mode;
  /* Row-window mode (window = kw' > 0, the reference conv's kernel width; pass kw = 1,
   * pad_left = 0): x is stored with its horizontal "same" padding baked in as zero columns
   * (x.w >= y.w + window - 1, x.c == x.c_stride) and the window input pixels of a kernel row
   * are folded into one K run of window * x.c channels.  Weights are those of a kh x 1 conv
   * over window * x.c input channels -- memory-identical to the kh x kw x cin HWIO tensor.
   * Used for narrow inputs (the 16-channel 7x7 stem) whose per-tap K would be tiny. */
  int window;
  /* Input stride s >= 1 (0 = 1): output pixel (y, x) reads x at (s*y + i*dilation - pad_top,
   * s*x + j*dilation - pad_left); x.h == s*y.h, x.w == s*y.w.  With the merged weights of
   * b2dl_pack_upsampled_dgrad this is the input gradient of a conv whose input was a nearest
   * upsampling by s, already summed over each s x s block (the upsample VJP): one conv at the
   * low resolution instead of a full-resolution dgrad plus a block sum. */
  int in_stride;
  /* Output phase view (out_stride f > 1): y is the full-resolution tensor and the conv writes
   * output pixel (i, j) to y pixel (f*i + out_phase_h, f*j + out_phase_w); y.h == f*x.h,
   * y.w == f*x.w.  No residual / mask / accumulate, bf16 y.  With the merged weights of
   * b2dl_pack_upsampled_fprop, the f*f phase launches are the forward of a conv over a nearest
   * upsampling by f, computed from the low-resolution input (no upsampled tensor). */
  int out_stride;
  int out_phase_h, out_phase_w;
  /* Batch-norm statistics from the epilogue (training-mode BN after this conv):
   * when non-NULL, the fprop writes rows of per-channel sums and sums of squares of its stored
   * bf16 output over the valid pixels, bn_partial[(row * 2 + k) * cout + c] (k = 0 sum, 1 sum of
   * squares): one row per CTA (its tiles, in order) when the launch has one N tile, else one row
   * per 128-pixel M tile -- b2dl_conv_fprop_bn_rows rows; reduced by b2dl_bn_forward_partials.
   * Needs the TMA epilogue (bf16 y, cout % 8 == 0, aligned views), no phase view, else
   * B2DL_E_VALUE. */
  float* bn_partial;
  /* Batch-norm backward statistics from the epilogue: when this launch writes g = d loss / d y of a
   * batch norm's output y = relu(scale z + shift) (no residual; bnb_stats = that BN's stats [4][c]:
   * mean, rstd, scale, shift), pass the BN input z as `mask`: the relu mask is recomputed from z
   * and the launch writes rows of (sum g, sum g * (z - mean) rstd) over the stored g,
   * bnb_partial[(row * 2 + k) * cout + c], 4 * b2dl_conv_fprop_bn_rows rows (one per TMEM lane
   * quarter) -- reduced by b2dl_bn_backward_partials.  Requires the TMA epilogue, no residual, no
   * accumulate, 16-byte aligned stats. */
  const float* bnb_stats;
  float* bnb_partial;
} b2dl_conv_args;

/* Number of bn_partial rows the b2dl_conv_fprop launch for these arguments writes. */
B2DL_API int b2dl_conv_fprop_bn_rows(const b2dl_conv_args* a);

B2DL_API int b2dl_cin_pad(int cin);
B2DL_API int b2dl_conv_fprop(const b2dl_conv_args* a, void* stream);

/* Weight gradient (the reference's conv2d_backward_weights), split-K over
 * pixels on tcgen05 with a deterministic reduction:
 *   dw[tap][ci][co] (+)= sum_p x[p + off(tap), ci] * dy[p, co]      (fp32, HWIO)
 * If bias_grad != NULL it also receives sum_p dy[p, co] (the bias_add VJP,
 * ops.py:172-175), accumulated when accumulate != 0. */
typedef struct b2dl_wgrad_args {
  b2dl_act x;
  b2dl_act dy;
  int kh, kw, dilation, pad_top, pad_left;
  float* dw;
  float* bias_grad;
  int accumulate;
  void* workspace;
  size_t workspace_bytes;
  int splits;       /* 0 = auto */
  int defer_reduce; /* 1: leave the split-K partials in `workspace` (layout from
                       b2dl_wgrad_partials) for a later batched b2dl_reduce_segments */
  int window;       /* row-window mode, as in b2dl_conv_args (dw is then [kh][window*cin][cout],
                       memory-identical to HWIO [kh][kw][cin][cout]) */
} b2dl_wgrad_args;

B2DL_API size_t b2dl_wgrad_workspace_size(const b2dl_wgrad_args* a);
B2DL_API int b2dl_conv_wgrad(const b2dl_wgrad_args* a, void* stream);
/* Partial-sum layout of a deferred wgrad: weight partials [w_parts][taps*cin*cout] at byte 0,
 * bias partials [b_parts][cout] at byte b_offset of the workspace. */
B2DL_API int b2dl_wgrad_partials(const b2dl_wgrad_args* a, int* w_parts, int* b_parts, size_t* b_offset);

/* Batched deterministic reduction of split-K partials: for every segment,
 * dst_base[dst_off + i] (+)= sum_k src[k * n + i], k < parts.  `segs` is device memory. */
typedef struct b2dl_segment {
  const float* src;
  int64_t dst_off;
  int64_t n;
  int32_t parts;
  int32_t accumulate;
} b2dl_segment;
B2DL_API int b2dl_reduce_segments(const b2dl_segment* segs, int nseg, int64_t max_n, float* dst_base,
                                  void* stream);

/* Pack fp32 HWIO master weights into the bf16 fprop layout [cout][taps][cin_pad]
 * and (optionally) the dgrad layout [cin][taps(flipped)][cout_pad]. */
B2DL_API int b2dl_pack_weights(const float* w_hwio, int kh, int kw, int cin, int cout, void* fprop_packed,
                      void* dgrad_packed, void* stream);

/* Merged weights for the strided input gradient above: conv k x k (HWIO fp32 [k*k][cin][cout],
 * same padding (k-1)/2) applied to a nearest upsampling by f; out is packed bf16
 * [cin][(k+f-1)^2][cin_pad(cout)] with W'(o) = sum over taps t, block offsets b with b - t = o of
 * W(t)^T (pads: pad_top = pad_left = (k-1)/2, in_stride f, kernel k+f-1, w_mode 0). */
/* Phase weights of a "same" k x k conv over a nearest x f upsampling: for output phase
 * (a, b) (row-major) a bf16 HWIO block [ka*kb][cin][cout] where ka spans the low-resolution
 * row offsets floor((a + t - (k-1)/2) / f), t = 0..k-1, and taps landing on one offset are
 * summed.  b2dl_upsampled_fprop_taps(k, f) = total taps over all phases (the buffer holds
 * taps * cin * cout bf16). */
B2DL_API int b2dl_upsampled_fprop_taps(int k, int f);
B2DL_API int b2dl_pack_upsampled_fprop(const float* w_hwio, int k, int cin, int cout, int f, void* out, void* stream);
/* Weight gradient of a "same" k x k conv (k in {1, 3}) over a nearest x f upsampling without the
 * upsampled tensor: g[n][h/f][w/f][k*k][c] (bf16) = the f x f block sums of dy shifted by
 * (k-1)/2 - t for every tap t; then dW = x_low^T g is a 1x1 wgrad with k*k*c output channels
 * (b2dl_conv_wgrad, defer_reduce) whose split-K partials b2dl_upsampled_wgrad_reduce sums in
 * fixed order into HWIO dw[k*k][cin][cout], and db[cout] from the centre tap's column sums. */
B2DL_API int b2dl_upsampled_wgrad_sums(b2dl_act dy, int k, int f, void* g, void* stream);
B2DL_API int b2dl_upsampled_wgrad_reduce(const void* partials, int w_parts, int b_parts, size_t b_offset, int cin,
                                         int k, int cout, float* dw, float* db, void* stream);
B2DL_API int b2dl_pack_upsampled_dgrad(const float* w_hwio, int k, int cin, int cout, int f, void* out, void* stream);

/* NCHW fp32 -> NHWC view, bf16 (or fp32 when dst_f32) (input tiles, reference-layout tensors). */
B2DL_API int b2dl_nchw_to_nhwc(const float* x, b2dl_act y, int dst_f32, void* stream);
/* NCHW fp32 [n][c][h][w] -> bf16 NHWC with a horizontal zero halo: y [n][h][wp][c], input
 * column xx at column left + xx, all other columns zero (the row-window conv input). */
B2DL_API int b2dl_nchw_to_nhwc_halo(const float* x, int n, int c, int h, int w, void* y, int wp, int left,
                                    void* stream);
/* NHWC (bf16, or fp32 when src_f32) view -> NCHW fp32. */
B2DL_API int b2dl_nhwc_to_nchw(b2dl_act x, int src_f32, float* y, void* stream);

/* avgpool window k (ops.py:133-138) and its VJP (ops.py:186-189). */
B2DL_API int b2dl_avgpool_fwd(b2dl_act x, b2dl_act y, int k, void* stream);
B2DL_API int b2dl_avgpool_bwd(b2dl_act dy, b2dl_act dx, int k, int accumulate, b2dl_act mask, void* stream);
/* nearest upsample factor f (ops.py:139-141) and its VJP, a block sum (ops.py:190-194). */
B2DL_API int b2dl_upsample_fwd(b2dl_act x, b2dl_act y, int f, void* stream);
B2DL_API int b2dl_upsample_bwd(b2dl_act dy, b2dl_act dx, int f, int accumulate, b2dl_act mask, void* stream);
/* y (+)= x, optionally masked by (mask > 0): elementwise-add VJP / fan-out sums. */
B2DL_API int b2dl_add(b2dl_act x, b2dl_act y, int accumulate, b2dl_act mask, void* stream);
/* Input gradient of a 1x1 conv with few output channels (the 3-class head): per pixel
 * dx[ci] (+)= mask * sum_k dy[k] * w[ci][k], w fp32 HWIO [cin][k] (k = dy.c <= 8).  A
 * memory-bound channel expansion, so it runs on CUDA cores rather than a K=16 GEMM. */
B2DL_API int b2dl_dgrad_1x1_small(b2dl_act dy, const float* w_hwio, b2dl_act dx, int accumulate, b2dl_act mask,
                                  void* stream);
/* Whole backward of such a head conv in one pass over its input x: per-block partial sums of
 * dW[ci][k] = sum_p x[p][ci] dy[p][k] (dw_partials [parts][cin*k]) and db[k] = sum_p dy[p][k]
 * (db_partials [parts][k]), parts = b2dl_head_backward_parts(), for a later deterministic
 * b2dl_reduce_segments; plus, when dx.ptr != NULL, the input gradient of
 * b2dl_dgrad_1x1_small with x itself as the relu mask (mask_dx != 0). */
B2DL_API int b2dl_head_backward_parts(void);
B2DL_API int b2dl_head_backward(b2dl_act dy, const float* w_hwio, b2dl_act x, b2dl_act dx, int accumulate,
                                int mask_dx, float* dw_partials, float* db_partials, void* stream);
/* in-place g *= (act > 0): relu VJP (ops.py:176-177). */
B2DL_API int b2dl_relu_mask(b2dl_act g, b2dl_act act, void* stream);
/* bias gradient: out[c] (+)= sum over pixels of g (ops.py:172-175). */
B2DL_API int b2dl_bias_grad(b2dl_act g, float* out, int accumulate, void* workspace, size_t workspace_bytes,
                   void* stream);
B2DL_API size_t b2dl_bias_grad_workspace_size(b2dl_act g);

/* Class-weighted softmax cross-entropy (loss.py:47-93), fused:
 *   counts[n][c]  exact per-sample label histogram (int32)
 *   loss_out[0]   mean over samples of sum_p w_y nll / sum_p w_y  (fp32)
 *   dlogits       (softmax - onehot) * w_y / (sum_p w_y * N) written as a bf16
 *                 NHWC view with `classes` channels
 *   pred          argmax over classes, ties to the lowest index (uint8)
 *   dlogits_scale multiplies dlogits (1; the fp16 build's static loss scale keeps the per-pixel
 *                 gradients, ~1e-7 at 1152 x 768, out of fp16's subnormal range)
 *   status[0]     (optional) 1 if any label is >= classes, else 0; the loss is then NaN
 *                 (the reference raises ValueError, loss.py:72-74; the host shim maps it)
 * logits: fp32 NHWC view with `classes` channels; labels uint8 [N*H*W]. */
B2DL_API int b2dl_wce(b2dl_act logits, const uint8_t* labels, const float* class_weights, int classes, float* loss_out,
             int* counts, b2dl_act dlogits, int dlogits_f32, float dlogits_scale, uint8_t* pred, int* status,
             void* workspace, size_t workspace_bytes, void* stream);
B2DL_API size_t b2dl_wce_workspace_size(int n, int h, int w, int classes);

/* LARC + SGD momentum over many tensors (optimizer.py:48-83) in two launches:
 *   per tensor t: wn = |w_t|, gn = |g_t| * grad_scale
 *   lr_t = lr if wn == 0 or (gn + wd*wn) < eps else min(trust*wn/(gn+wd*wn), lr)
 *   m = beta*m + g*grad_scale + wd*w ; w -= lr_t * m
 * Tensors are contiguous segments of flat fp32 buffers (offsets[t]..offsets[t+1]).
 * grad_scale folds the data-parallel mean (1/P).  lr_out[t] receives lr_t;
 * status[0] is set to 1 if any norm is non-finite (and no update is applied). */
typedef struct b2dl_larc_args {
  float* w;
  float* m;
  const float* g;
  const int64_t* offsets; /* device, ntensors+1 */
  int ntensors;
  float lr, momentum, trust, weight_decay, eps, grad_scale;
  float* lr_out;   /* device, ntensors */
  int* status;     /* device, 1 int */
  void* workspace; /* device scratch */
  size_t workspace_bytes;
  int mode; /* 0: norms + rates + update; 1: rates only (larc_effective_lr);
               2: update with the caller's lr_out (sgd_step); 3: only refresh w_bf16 from w */
  void* w_bf16; /* optional bf16 mirror of w written by the update (the conv weight operand) */
} b2dl_larc_args;
B2DL_API size_t b2dl_larc_workspace_size(int64_t total_elems, int ntensors);
B2DL_API int b2dl_larc_update(const b2dl_larc_args* a, void* stream);

/* Version / capability string (for smoke checks). */
/* ---------------------------------------------------------------- batch norm + bilinear
 * North-star extensions without a reference implementation; float64 oracle in
 * oracle/deskdl_port.py pinned by finite differences.  f32 != 0: fp32 views, else bf16. */
/* scratch for b2dl_bn_forward / b2dl_bn_backward on c channels */
B2DL_API size_t b2dl_bn_workspace_size(int c);
/* training-mode batch norm over N, H, W (biased variance) fused with an optional residual add and
 * relu: y = relu?(gamma * (x - mean) * rstd + beta (+ residual)); stats[4][c] receives mean, rstd,
 * scale = gamma*rstd and shift = beta - mean*scale (the backward reads mean and rstd). */
B2DL_API int b2dl_bn_forward(b2dl_act x, const float* gamma, const float* beta, float eps, b2dl_act residual,
                             int relu, b2dl_act y, float* stats, void* workspace, size_t workspace_bytes, int f32,
                             void* stream);
/* The same forward with the statistics already in `partials` ([tiles][2][c] fp32 sums / sums of
 * squares written by the producing conv's epilogue, b2dl_conv_args.bn_partial): a fixed-order fp64
 * reduction over the tiles, then the normalising pass -- no statistics pass over x. */
B2DL_API int b2dl_bn_forward_partials(const float* partials, int tiles, b2dl_act x, const float* gamma,
                                      const float* beta, float eps, b2dl_act residual, int relu, b2dl_act y,
                                      float* stats, void* workspace, size_t workspace_bytes, int f32,
                                      void* stream);
/* dgamma (+)= sum gy*xhat, dbeta (+)= sum gy (param_accumulate), and when dx.ptr != NULL
 * dx (+)= gamma*rstd*(gy - dbeta/M - xhat*dgamma/M) (accumulate); gy already relu-masked. */
B2DL_API int b2dl_bn_backward(b2dl_act x, b2dl_act gy, const float* gamma, const float* stats, float* dgamma,
                              float* dbeta, int param_accumulate, b2dl_act dx, int accumulate, void* workspace,
                              size_t workspace_bytes, int f32, void* stream);
/* b2dl_bn_backward with the statistics already reduced per row by the consumer conv's dgrad
 * epilogue (b2dl_conv_args.bnb_partial: [rows][2][c] sums of gy and gy * xhat): fixed-order fp64
 * reduction, then the input-gradient pass only (gy already relu-masked). */
B2DL_API int b2dl_bn_backward_partials(const float* partials, int rows, b2dl_act x, b2dl_act gy, const float* gamma,
                                       const float* stats, float* dgamma, float* dbeta, int param_accumulate,
                                       b2dl_act dx, int accumulate, void* workspace, size_t workspace_bytes, int f32,
                                       void* stream);
/* bilinear upsampling by integer factor f (half-pixel centres, align_corners=False) and its VJP
 * (separable and deterministic: a row pass into an fp32 workspace of dy.n*dy.h*(dy.w/f)*dy.c
 * floats, then a column pass; dx (+)= mask(>0) * ...). */
B2DL_API int b2dl_bilinear_fwd(b2dl_act x, b2dl_act y, int f, int f32, void* stream);
B2DL_API size_t b2dl_bilinear_workspace_size(b2dl_act dy, int f);
B2DL_API int b2dl_bilinear_bwd(b2dl_act dy, b2dl_act dx, int f, int accumulate, b2dl_act mask, int f32,
                               void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------- (3) fp32 parity mode
 * The reference's own arithmetic type end to end (north star: loss and gradients within 1e-3 in
 * fp32 mode): every b2dl_act below is NHWC fp32, weights are the fp32 HWIO master, FMA
 * accumulation in fp32 on the CUDA cores.  Same semantics as the bf16 entry points above. */
/* conv forward (w_mode 1: w_master = this conv's HWIO) or input gradient (w_mode 2: w_master =
 * the forward conv's HWIO, tap-flipped, "after" pads); fused bias / residual / relu / mask /
 * accumulate epilogue as in b2dl_conv_fprop.  w_packed, block_n, y_f32 and window are ignored. */
B2DL_API int b2dl_f32_conv_fprop(const b2dl_conv_args* a, void* stream);
/* dw fp32 HWIO (+)= wgrad, bias_grad (+)= column sums; split-K partials in `workspace`, reduced
 * in a fixed order before return (defer_reduce, splits and window are ignored / rejected). */
B2DL_API size_t b2dl_f32_wgrad_workspace_size(const b2dl_wgrad_args* a);
B2DL_API int b2dl_f32_conv_wgrad(const b2dl_wgrad_args* a, void* stream);
B2DL_API int b2dl_f32_avgpool_fwd(b2dl_act x, b2dl_act y, int k, void* stream);
B2DL_API int b2dl_f32_avgpool_bwd(b2dl_act dy, b2dl_act dx, int k, int accumulate, b2dl_act mask, void* stream);
B2DL_API int b2dl_f32_upsample_fwd(b2dl_act x, b2dl_act y, int f, void* stream);
B2DL_API int b2dl_f32_upsample_bwd(b2dl_act dy, b2dl_act dx, int f, int accumulate, b2dl_act mask, void* stream);
/* y (+)= x, masked by (mask > 0); with x == y and accumulate == 0 it is the in-place relu VJP. */
B2DL_API int b2dl_f32_add(b2dl_act x, b2dl_act y, int accumulate, b2dl_act mask, void* stream);

B2DL_API const char* b2dl_version(void);

/* ---------------------------------------------------------------- standalone op lowerings
 * (csrc/generic.cu) -- the reference op kinds that are not part of a conv-bias-relu chain, so any
 * graph over the reference's op set runs through the engine.  `f32` = 1: fp32 storage (parity
 * mode), else bf16.  Parameters (bias, B) are the fp32 master. */

/* y (+)= mask? . relu?( alpha . x0 . x1? + bias[c]? ): elementwise mul / scale (ops.py:142-148),
 * standalone bias_add (:122-126) and relu (:127-128), and their VJPs (:172-177, :195-202).
 * x1, mask: optional views (ptr NULL); bias: optional fp32 [c]. */
B2DL_API int b2dl_ewise(b2dl_act x0, b2dl_act x1, b2dl_act mask, b2dl_act y, const float* bias, float alpha,
                        int relu, int accumulate, int f32, void* stream);
/* Y = X @ B over the width axis of an NCHW activation (ops.py:120): NHWC views x [n][h][wi][c],
 * y [n][h][wo][c]; B fp32 row-major [wi][wo] (ldb = wo), or with trans = 1 the input gradient
 * dX = dY @ B^T (x = dY with wi = W2, y = dX, ldb = x.w).  Optional mask on the output. */
B2DL_API int b2dl_matmul_w(b2dl_act x, const float* b, int ldb, int trans, b2dl_act y, b2dl_act mask,
                           int accumulate, int f32, void* stream);
/* gB[i][j] (+)= sum_{n,h,c} X[n,h,i,c] G[n,h,j,c]  (ops.py:166-170), fixed order. */
B2DL_API int b2dl_matmul_w_grad(b2dl_act x, b2dl_act g, float* gb, int accumulate, int f32, void* stream);
/* out[c] (+)= sum over n,h,w of g (standalone bias_add VJP, ops.py:172-175), fixed order. */
B2DL_API int b2dl_channel_sum(b2dl_act g, float* out, int accumulate, int f32, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* B2DL_H */
