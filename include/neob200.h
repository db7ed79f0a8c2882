/*
 * neob200.h - C ABI of libneob200.so, the sm_100a kernels behind the
 * NCHW[x]c CNN-inference hot path (NeoCPU, arXiv 1809.02697).
 *
 * The reference (`neoplan`, /root/reference/pkg/src/neoplan) has no FFI: its
 * "operator API" is the Python surface in __init__.py:5-31 and executor.py is
 * the single dispatch point.  Each entry point below replaces one compute site
 * of that surface; the interface it replaces is cited beside it.  The Python
 * host package (paper_1809_02697_b200) binds these with ctypes.
 *
 * Conventions (all entry points):
 *   - plain pointers and sizes; every pointer argument is a DEVICE pointer
 *     unless stated otherwise; callers allocate outputs (no call allocates);
 *   - every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *     default stream) and returns before the work completes;
 *   - return value: NEO_OK (0) or a neo_status; neo_last_error() returns the
 *     thread-local message of the last failure.  The Python shim maps codes to
 *     the reference exception taxonomy (errors.py:4-59).
 *   - data types: NEO_F32 = IEEE float32, NEO_BF16 = bfloat16, NEO_FP8 = OCP
 *     e4m3 ("e4m3fn": no infinities, max 448) in one byte.  "tf32" values
 *     are float32 containers whose low 13 mantissa bits are zero.  An e4m3
 *     tensor carries a per-tensor scale s outside the buffer: the value of a
 *     stored byte q is e4m3(q) * s.
 */
#ifndef NEOB200_H
#define NEOB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* neo_stream_t; /* cudaStream_t */

typedef enum {
  NEO_OK = 0,
  NEO_ERR_SCHEDULE_INVALID = 1,   /* errors.ScheduleInvalid     */
  NEO_ERR_SHAPE_MISMATCH = 2,     /* errors.ShapeMismatch       */
  NEO_ERR_WRONG_LAYOUT = 3,       /* errors.WrongLayout         */
  NEO_ERR_INDIVISIBLE_CHANNEL = 4,/* errors.IndivisibleChannel  */
  NEO_ERR_UNSUPPORTED = 5,        /* configuration the kernels do not cover */
  NEO_ERR_CUDA = 6,               /* CUDA runtime/driver failure */
  NEO_ERR_INVALID_ARG = 7         /* bad pointer / size          */
} neo_status;

typedef enum { NEO_F32 = 0, NEO_BF16 = 1, NEO_FP8 = 2 } neo_dtype;

/* feature-map layout tags (layout.py:21-71).  NCHW == NCHW[1]c in memory. */
typedef enum { NEO_NCHW = 0, NEO_NHWC = 1, NEO_NCHWC = 2 } neo_layout_tag;

/* conv arithmetic */
typedef enum {
  NEO_MODE_FP32 = 0, /* SIMT fp32 direct conv (parity anchor; conv_reference) */
  NEO_MODE_TF32 = 1, /* tcgen05 kind::tf32, fp32 activations rounded to tf32 */
  NEO_MODE_BF16 = 2, /* tcgen05 kind::f16 (bf16 in, fp32 accumulate)        */
  NEO_MODE_FP8 = 3   /* tcgen05 kind::f8f6f4, e4m3 activations (per-tensor
                        scale) x e4m3 weights (per-output-channel scale),
                        fp32 accumulate; quantized inference, the paper's
                        stated future work                   */
} neo_conv_mode;

typedef enum { NEO_POOL_MAX = 0, NEO_POOL_AVG = 1 } neo_pool_mode;

typedef enum {
  NEO_ELT_RELU = 0,             /* out = max(a, 0)                           */
  NEO_ELT_ADD = 1,              /* out = a + b                               */
  NEO_ELT_ADD_RELU = 2,         /* out = max(a + b, 0)                       */
  NEO_ELT_SCALE_SHIFT = 3,      /* out = a * scale[c] + shift[c]   (BN)      */
  NEO_ELT_SCALE_SHIFT_RELU = 4  /* out = max(a * scale[c] + shift[c], 0)     */
} neo_eltwise_op;

/* flag bits */
#define NEO_FLAG_ROUND_TF32 0x1   /* round fp32 results to tf32 (RN)        */
#define NEO_FLAG_PAD_CHANNELS 0x2 /* allow C % x != 0: zero-filled pad lanes */
/* conv: the weight buffer is not written by any kernel that may still be
 * running (e.g. packed at load time), so a programmatically launched conv may
 * fetch its resident weight image before griddepcontrol.wait */
#define NEO_FLAG_STATIC_WEIGHTS 0x4
/* conv tile geometry: tile_w is the BAND width of a halo strip (tile_w - (s-1)
 * output columns per tile, see conv_tc.cu); set by neo_conv_default_tiles when
 * it picks strips for a map wider than one tile, or by a caller passing an
 * explicit strip geometry */
#define NEO_FLAG_HALO_STRIPS 0x8

const char* neo_last_error(void);
int neo_abi_version(void);
/* "name|sm_count|cc_major.cc_minor|hbm_bytes" of `device` into buf */
int neo_device_info(int device, char* buf, int buflen);

/* ---- layout transforms (layout.py:131-235) ------------------------------
 * Feature map (n, c, h, w) logical; src/dst tags NCHW, NHWC (src only) or
 * NCHW[x]c.  Replaces transform_array (layout.py:219-235): pack_nchw_array
 * :131, unpack_nchw_array :140, retile_nchw_array :163, nhwc_to_nchw_array
 * :180.  Bit-exact when src_dtype == dst_dtype and flags == 0.  With
 * NEO_FLAG_PAD_CHANNELS a blocked side may carry ceil(c/x) blocks whose pad
 * lanes are zero (pack) or dropped (unpack); without it c % x != 0 returns
 * NEO_ERR_INDIVISIBLE_CHANNEL like the reference. */
int neo_layout_transform(int src_dtype, int dst_dtype, const void* src, void* dst, int64_t n,
                         int64_t c, int64_t h, int64_t w, int src_tag, int src_x, int dst_tag,
                         int dst_x, int flags, neo_stream_t stream);

/* KCRS <-> KCRS[x]c[y]k, bit-exact (pack_kcrs_array layout.py:147,
 * unpack_kcrs_array :156).  dtype is the element type of both sides. */
int neo_pack_weights(int dtype, const void* src, void* dst, int64_t k, int64_t c, int64_t r,
                     int64_t s, int x, int y, neo_stream_t stream);
int neo_unpack_weights(int dtype, const void* src, void* dst, int64_t k, int64_t c, int64_t r,
                       int64_t s, int x, int y, neo_stream_t stream);

/* Device-private tensor-core weight image used by NEO_MODE_TF32/BF16 convs
 * (compile time, like pretransform_weights passes.py:258-286).  src is KCRS
 * float32.  dst layout is slice-major (R, S, ceil(C/x), K, x) - every
 * (r, s, channel-block) slice is a K x x K-major tile - padded with zero
 * slices up to `slices_padded` (see neo_conv_umma_slices).  dst_dtype NEO_BF16
 * rounds RN to bf16; NEO_F32 with NEO_FLAG_ROUND_TF32 rounds RN to tf32. */
int neo_pack_weights_umma(const float* src_kcrs, void* dst, int dst_dtype, int64_t k, int64_t c,
                          int64_t r, int64_t s, int x, int64_t slices_padded, int flags,
                          neo_stream_t stream);
/* NEO_MODE_FP8 weight image: the same slice-major layout in e4m3 bytes,
 * dst[.., k, ..] = e4m3_rn_satfinite(src[k, ..] / wscale[k]) (IEEE f32
 * division, then round-to-nearest-even to e4m3).  wscale: device f32 per
 * output channel (normally absmax_k / 448); the conv folds it back in through
 * its per-channel epilogue scale. */
int neo_pack_weights_umma_fp8(const float* src_kcrs, void* dst, const float* wscale, int64_t k,
                              int64_t c, int64_t r, int64_t s, int x, int64_t slices_padded,
                              int flags, neo_stream_t stream);
/* e4m3 NCHW[x]c (channel-block window cb_off of cb_total blocks; cb_total 0 =
 * dense) -> NCHW f32 / bf16 (dst_dtype): value = e4m3(q) * scale.  The FP8
 * mode's exit from the blocked chain (transform_array layout.py:219-235 with
 * the e4m3 decode). */
int neo_dequant_fp8(const void* src, void* dst, int dst_dtype, float scale, int64_t n, int64_t c,
                    int64_t h, int64_t w, int x, int64_t cb_off, int64_t cb_total,
                    neo_stream_t stream);
/* max |x| over n elements of a device buffer of `dtype` (fp8 bytes decoded
 * without scale) into *out (a device float); used by FP8 calibration. */
int neo_absmax(int dtype, const void* x, int64_t n, float* out, neo_stream_t stream);
/* number of slices the conv kernel expects for (c, r, s, x, mode, tile cfg);
 * the weight image must be packed with at least that many slices. */
int64_t neo_conv_umma_slices(int mode, int64_t c, int64_t r, int64_t s, int x,
                             int slices_per_stage);

/* Stem fold (B200 lowering, no reference counterpart): NCHW f32 src ->
 * NCHW[xf]c dst over folded channels f = s*C + c, width ow:
 *   dst[n, f/xf, h, w', f%xf] = src[n, c, h, stride_w*w' + s - pad_w] (0 if OOB)
 * A conv with kernel width S, stride_w, pad_w over src equals a conv with
 * kernel width 1, stride 1, pad 0 along w over dst with weights
 * W'[k, s*C + c, r, 0] = W[k, c, r, s]; used for 3-channel image stems. */
int neo_stem_fold(const float* src, void* dst, int dst_dtype, int64_t n, int64_t c, int64_t h,
                  int64_t w, int s, int stride_w, int pad_w, int64_t ow, int xf, int flags,
                  neo_stream_t stream);

/* Fused image stem (B200 lowering of the reference's first three operators:
 * conv_blocked kernels.py:250-303 on the packed image, its Epilogue
 * kernels.py:185-197, and _pool2d executor.py:103-128):
 *   out = maxpool3x3/2 pad 1 (-inf) ( relu?( conv7x7/2 pad 3 (x, w)
 *                                           * scale + shift + bias ) )
 * x: NCHW (n, c, h, w) f32 or bf16 (x_dtype; f32 is rounded RN to bf16, so a
 * host-rounded bf16 image gives identical results) with c <= 4 and 16-byte
 * rows (w % 4 == 0 f32, w % 8 == 0 bf16); K = 64 output
 * channels; out: bf16 NCHW[y]c (n, out_cb_total, ph, pw, y), written at
 * channel-block offset out_cb_offset (concat in place), y in {8,16,32,64};
 * scale/shift/bias per output channel or NULL.  wimg is the 28 KB image
 * neo_stem_pack_weights builds from the KCRS f32 weights (bf16 RN). */
int neo_stem_pack_weights(const float* w_kcrs, void* img, int64_t k, int64_t c, int64_t r,
                          int64_t s, neo_stream_t stream);
int64_t neo_stem_weight_bytes(void);
int neo_stem_conv_pool(const void* x, int x_dtype, const void* wimg, void* out, const float* scale,
                       const float* shift, const float* bias, int relu, int64_t n, int64_t c,
                       int64_t h, int64_t w, int y, int out_cb_offset, int out_cb_total,
                       neo_stream_t stream);
/* neo_stem_conv_pool with the output type chosen: out_dtype NEO_BF16 (as
 * above) or NEO_FP8, then every pooled bf16 value v is stored as
 * e4m3_rn_satfinite(v / out_scale) (out_scale > 0). */
int neo_stem_conv_pool_q(const void* x, int x_dtype, const void* wimg, void* out, int out_dtype,
                         float out_scale, const float* scale, const float* shift,
                         const float* bias, int relu, int64_t n, int64_t c, int64_t h, int64_t w,
                         int y, int out_cb_offset, int out_cb_total, neo_stream_t stream);

/* Fused classifier head (B200 lowering of the reference's global average
 * pool executor.py:103-128, Flatten, Dense executor.py:197-203 and Softmax
 * executor.py:167-170):
 *   pooled[n, c] = bf16(sum_t x[n, c, t] / hw)      (x: bf16 NCHW[y]c, H*W = hw)
 *   logits[n, u] = sum_c pooled[n, c] * w[u, c] + bias[u]   (w: bf16 (units, c))
 *   out = softmax ? softmax_rows(logits) : logits          (f32 (n, units))
 * C % 256 == 0.  pooled (n*c bf16), logits (2*n*units f32) and bar (3 ints,
 * zero-initialised once; the kernel re-arms them) are caller scratch. */
int neo_classifier_head(const void* x, const void* w_bf16, const float* bias, void* pooled,
                        float* logits, float* out, int* bar, int64_t n, int64_t c, int64_t hw,
                        int y, int64_t units, int softmax, neo_stream_t stream);
/* Same head over an e4m3 NCHW[y]c map with per-tensor scale x_scale:
 *   pooled[n, c] = bf16(x_scale * sum_t e4m3(x[n, c, t]) / hw)  (x_dtype
 *   NEO_FP8; NEO_BF16 ignores x_scale and equals neo_classifier_head). */
int neo_classifier_head_q(const void* x, int x_dtype, float x_scale, const void* w_bf16,
                          const float* bias, void* pooled, float* logits, float* out, int* bar,
                          int64_t n, int64_t c, int64_t hw, int y, int64_t units, int softmax,
                          neo_stream_t stream);

/* ---- fused blocked convolution (kernels.py:250-303 conv_blocked, with the
 * Epilogue kernels.py:74-87 applied in the order scale/shift -> bias ->
 * residual -> relu, kernels.py:185-197) --------------------------------- */
typedef struct neo_conv_params {
  /* sizeof(neo_conv_params) as the caller compiled it (ABI v2+): every entry
   * point taking the struct rejects a mismatch with NEO_ERR_INVALID_ARG, so a
   * binding written against an older layout fails loudly instead of letting
   * the library read fields past the end of a shorter struct. */
  int struct_size;
  int mode;            /* neo_conv_mode                                       */
  const void* x;       /* input  (n, cb_total_x, h, w, ic_bn); window below    */
  const void* w;       /* FP32: KCRS[ic_bn]c[oc_bn]k f32; TF32/BF16: umma image */
  void* out;           /* output (n, out_cb_total, oh, ow, oc_bn)              */
  const float* scale;  /* per out-channel, or NULL                             */
  const float* shift;  /* per out-channel, or NULL (0 when scale given)        */
  const float* bias;   /* per out-channel, or NULL                             */
  const void* residual;/* (n, res_cb_total, oh, ow, oc_bn) or NULL             */
  int relu;
  int64_t n, c, h, w_in, k, r, s;
  int stride_h, stride_w, pad_h, pad_w;
  int ic_bn, oc_bn;
  int x_cb_offset, x_cb_total;     /* input channel-block window (0,0 = dense) */
  int out_cb_offset, out_cb_total; /* concat-in-place destination window      */
  int res_cb_offset, res_cb_total;
  int out_dtype;       /* NEO_F32 / NEO_BF16 / NEO_FP8 (residual: same dtype) */
  int flags;           /* NEO_FLAG_ROUND_TF32 | NEO_FLAG_PAD_CHANNELS |
                        * NEO_FLAG_STATIC_WEIGHTS | NEO_FLAG_HALO_STRIPS      */
  /* tile configuration (0 = automatic).  tile_w x tile_h x tile_img output
   * pixels (<= 128) form the M tile; tile_n output channels (multiple of 16,
   * <= 256) the N tile; slices_per_stage (r, s, channel-block) slices per
   * pipeline stage; stages = pipeline depth (<= 8).  Halo (band-reuse) tiles of
   * stride-1 convs with a horizontal window (32/64/128-byte rows): tile_w =
   * ow + s - 1 > ow, tile_img = 1 (one band per kernel row and channel block,
   * the s taps are shifted views of it); with NEO_FLAG_HALO_STRIPS tile_w is
   * the band width of a column strip of tile_w - (s - 1) output columns. */
  int tile_w, tile_h, tile_img, tile_n, slices_per_stage, stages;
  /* split-K: the reduction is cut into split_k ranges run by separate CTAs
   * (0 = automatic: only when the output tiles leave most SMs idle; 1 = off).
   * Partials go to `workspace` (size from neo_conv_workspace_bytes; it must be
   * zero-filled before its first use and every launch leaves it zeroed) and
   * the last CTA of each output tile sums them in split order and applies
   * the epilogue.  Without a large enough workspace an automatic split is
   * dropped. */
  int split_k;
  void* workspace;
  int64_t workspace_bytes;
  /* CTA pairs (cta_group::2): two CTAs of a cluster compute one 256-row M
   * tile, each holding half of the A rows and half of the weight rows, so a
   * weight byte serves 256 pixels (0 = automatic, 1 = off, 2 = on). */
  int cta_pair;
  /* BN-ReLU prologue (DenseNet pre-activation, reference executor.py:174-181
   * + ReLU): with pro_scale != NULL the conv consumes
   * relu?(x * pro_scale[c] + pro_shift[c]) instead of x, computed on the
   * tiles in shared memory (unpadded 1x1 convs, TF32/BF16 modes). */
  const float* pro_scale;
  const float* pro_shift;
  int pro_relu;
  /* weight-stationary tiles: each CTA keeps the whole weight image of its N
   * block in shared memory and streams only activations (stride-1 KxK convs
   * then load one input band per channel block for all R*S taps)
   * (0 = automatic: when it fits beside >= 3 activation stages, 1 = off,
   * 2 = on). */
  int weight_stationary;
  /* second output (TF32/BF16, no residual, no split-K, no CTA pair): output
   * channels [k_split, k) go to out2 (n, out2_cb_total, oh, ow, oc_bn) at
   * channel block out2_cb_offset + (k - k_split) / oc_bn with relu2, so two
   * sibling convs over the same input (a bottleneck's reduce 1x1 and its
   * projection shortcut, passes.py:119-157 fuse nothing across siblings)
   * run as one launch over concatenated weights and epilogue vectors;
   * k_split must be a multiple of the N tile (0 = single output). */
  void* out2;
  int64_t k_split;
  int relu2;
  int out2_cb_offset, out2_cb_total;
  /* e4m3 storage scales (ABI v3; ignored unless the tensor is NEO_FP8; 0
   * means 1): a stored residual byte q stands for e4m3(q) * res_scale, and
   * an output value v is stored as e4m3_rn_satfinite(v / out_scale)
   * (out2_scale for the second output).  The input's own scale is not a
   * field: NEO_MODE_FP8 callers fold x_scale * wscale[k] into `scale`. */
  float res_scale;
  float out_scale;
  float out2_scale;
} neo_conv_params;

int neo_conv2d_nchwc_fused(const neo_conv_params* p, neo_stream_t stream);
/* sizeof(neo_conv_params) of the library build (what struct_size must hold) */
int neo_conv_params_size(void);
/* fill the automatic tile fields of *p the way neo_conv2d_nchwc_fused would */
int neo_conv_default_tiles(neo_conv_params* p);
/* Split-K workspace bytes the launch of *p needs with its resolved tiles
 * (0 when it will not split). */
int neo_conv_workspace_bytes(const neo_conv_params* p, int64_t* bytes);

/* Two chained 1x1 convolutions (bf16, NCHW[64]c) as ONE launch -- the junction
 * between two bottleneck blocks: y1 = relu1?(x * W1 + b1 + residual) (block
 * i's expand conv with its fused shortcut) and y2 = relu2?(y1 * W2 + b2)
 * (block i+1's reduce conv), y2 computed from y1 in shared memory.  Replaces
 * two conv_blocked calls (kernels.py:250-303, Epilogue :74-87 in the order
 * of :185-197); y1 and y2 are bit-identical to the two separate convs.
 * w1 / w2: neo_pack_weights_umma images (x = 64) of the (N1, C1, 1, 1) and
 * (N2, N1, 1, 1) weights.  Needs C1 % 64 == 0, N1 % 128 == 0, N2 in
 * {64, 128, 192, 256}; residual may be NULL.  Unpadded, stride 1. */
int neo_conv_junction(const void* x, const void* w1, const float* b1, const void* residual,
                      void* y1, const void* w2, const float* b2, void* y2, int64_t n, int64_t c1,
                      int64_t h, int64_t w, int64_t n1, int64_t n2, int relu1, int relu2,
                      neo_stream_t stream);

/* ---- memory-bound operators (executor.py:96-203) ------------------------ */
/* Max (pad -inf) / avg (pad 0, / win^2) pooling over h, w of NCHW[x]c
 * (x = 1 is NCHW), replaces _pool2d executor.py:103-128.  NEO_FP8 maps:
 * max pooling only, x % 16 == 0, the output keeps the input's scale. */
int neo_pool2d(int dtype, int mode, const void* in, void* out, int64_t n, int64_t cb, int64_t h,
               int64_t w, int x, int win, int stride, int pad, int flags, neo_stream_t stream);
/* Same with channel-block windows: the input is blocks [in_cb_off, +cb) of a
 * (n, in_cb_total, h, w, x) buffer and the output blocks [out_cb_off, +cb) of
 * a (n, out_cb_total, oh, ow, x) buffer (concat-in-place). */
int neo_pool2d_window(int dtype, int mode, const void* in, void* out, int64_t n, int64_t cb,
                      int64_t h, int64_t w, int x, int win, int stride, int pad,
                      int64_t in_cb_off, int64_t in_cb_total, int64_t out_cb_off,
                      int64_t out_cb_total, int flags, neo_stream_t stream);
/* e4m3 pooling with scales (FP8 mode): max or avg (reference order, /win^2)
 * of the dequantized inputs e4m3(q) * in_scale, stored as
 * e4m3_rn_satfinite(v / out_scale); windows as neo_pool2d_window; x % 16 == 0.
 * A max pool with out_scale == in_scale copies the winning bytes. */
int neo_pool2d_q(int mode, const void* in, void* out, int64_t n, int64_t cb, int64_t h, int64_t w,
                 int x, int win, int stride, int pad, int64_t in_cb_off, int64_t in_cb_total,
                 int64_t out_cb_off, int64_t out_cb_total, float in_scale, float out_scale,
                 neo_stream_t stream);
/* elementwise ops over (n, cb, hw, x) (x = 1 is NCHW); scale/shift indexed by
 * channel cb*x+lane.  Replaces executor.py:165-190 (ReLU, BatchNorm with
 * _channel_broadcast :96-100, ElementwiseAdd). */
int neo_eltwise(int dtype, int op, const void* a, const void* b, void* out, const float* scale,
                const float* shift, int64_t n, int64_t cb, int64_t hw, int x, int flags,
                neo_stream_t stream);
/* Same with channel-block windows on `a` and `out` (relu / scale-shift ops;
 * add requires dense operands). */
int neo_eltwise_window(int dtype, int op, const void* a, const void* b, void* out,
                       const float* scale, const float* shift, int64_t n, int64_t cb, int64_t hw,
                       int x, int64_t a_cb_off, int64_t a_cb_total, int64_t out_cb_off,
                       int64_t out_cb_total, int flags, neo_stream_t stream);
/* e4m3 relu / scale-shift / scale-shift-relu (FP8 mode; BN = a*scale+shift as
 * two rounded f32 ops on a = e4m3(q) * a_scale), stored as
 * e4m3_rn_satfinite(v / out_scale); channel-block windows on a and out. */
int neo_eltwise_q(int op, const void* a, void* out, const float* scale, const float* shift,
                  int64_t n, int64_t cb, int64_t hw, int x, int64_t a_cb_off, int64_t a_cb_total,
                  int64_t out_cb_off, int64_t out_cb_total, float a_scale, float out_scale,
                  neo_stream_t stream);
/* strided copy for np.concatenate (executor.py:191-193): src viewed as
 * (outer, chunk) elements is copied into dst viewed as (outer, dst_row) at
 * column dst_off.  Concat of k inputs = k calls. */
int neo_concat_copy(int dtype, const void* src, void* dst, int64_t outer, int64_t chunk,
                    int64_t dst_row, int64_t dst_off, neo_stream_t stream);
/* out(n, units) f32 = a(n, in) @ w(units, in)^T (+ bias), executor.py:197-203.
 * a and w share `dtype`. */
int neo_dense(int dtype, const void* a, const void* w, const float* bias, float* out, int64_t n,
              int64_t in_features, int64_t units, neo_stream_t stream);
/* row softmax with max subtraction, executor.py:167-170 (f32 in/out) */
int neo_softmax(const float* in, float* out, int64_t rows, int64_t cols, neo_stream_t stream);

/* ---- whole-graph capture (replaces the Python per-op dispatch loop,
 * executor.py:156-216, with one CUDA graph launch) ------------------------ */
int neo_capture_begin(neo_stream_t stream);
int neo_capture_end(neo_stream_t stream, void** graph_exec);
int neo_graph_launch(void* graph_exec, neo_stream_t stream);
int neo_graph_destroy(void* graph_exec);

#ifdef __cplusplus
}
#endif

#endif /* NEOB200_H */
