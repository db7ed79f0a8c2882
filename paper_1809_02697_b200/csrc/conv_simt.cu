// FP32 SIMT direct convolution on NCHW[x]c x KCRS[x]c[y]k (NEO_MODE_FP32).
//
// The parity anchor of the conv path.  One thread per output element
// out[n, kb, oh, ow, j]; the reduction runs in the reference blocked order
// co -> r -> s -> ci (kernels.py:159-184) with separately rounded multiply and
// add, and the epilogue is applied as separate rounded steps in the reference
// order scale/shift -> bias -> residual -> relu (kernels.py:234-246).  With
// ic_bn = oc_bn = 1 the tensors are plain NCHW / KCRS and the loop order is the
// naive c -> r -> s of _naive_nchw (kernels.py:117-132), which makes this the
// device conv_reference: padding taps are skipped, which is bit-identical to
// adding 0*w to a +0-initialised accumulator.
#include "neo_common.cuh"

namespace {

struct ConvSimtParams {
  const float* x;
  const float* w;
  float* out;
  const float* scale;
  const float* shift;
  const float* bias;
  const float* res;
  int relu, round_tf32;
  int N, Cb, H, W, K, R, S, OH, OW, x_bn, y;
  int sh, sw, ph, pw;
  int x_cb_off, x_cb_total, out_cb_off, out_cb_total, res_cb_off, res_cb_total;
};

__global__ void conv_simt_kernel(const ConvSimtParams p) {
  neo_pdl_enter();
  const int Kb = (p.K + p.y - 1) / p.y;
  const int64_t total = (int64_t)p.N * Kb * p.y * p.OH * p.OW;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    // output enumerated as (n, kb, oh, ow, j) so consecutive threads write
    // consecutive addresses of the blocked layout
    int64_t t = idx;
    const int j = (int)(t % p.y);
    t /= p.y;
    const int ow = (int)(t % p.OW);
    t /= p.OW;
    const int oh = (int)(t % p.OH);
    t /= p.OH;
    const int kb = (int)(t % Kb);
    const int n = (int)(t / Kb);
    const int k = kb * p.y + j;
    if (k >= p.K) continue;
    float acc = 0.f;
    for (int co = 0; co < p.Cb; ++co) {
      const float* xb = p.x + (((size_t)n * p.x_cb_total + p.x_cb_off + co) * p.H) * p.W * p.x_bn;
      const float* wb = p.w + ((size_t)kb * p.Cb + co) * p.R * p.S * p.x_bn * p.y;
      for (int r = 0; r < p.R; ++r) {
        const int ih = oh * p.sh + r - p.ph;
        if (ih < 0 || ih >= p.H) continue;
        for (int s = 0; s < p.S; ++s) {
          const int iw = ow * p.sw + s - p.pw;
          if (iw < 0 || iw >= p.W) continue;
          const float* xp = xb + ((size_t)ih * p.W + iw) * p.x_bn;
          const float* wp = wb + ((size_t)r * p.S + s) * p.x_bn * p.y + j;
          for (int ci = 0; ci < p.x_bn; ++ci)
            acc = __fadd_rn(acc, __fmul_rn(__ldg(xp + ci), __ldg(wp + (size_t)ci * p.y)));
        }
      }
    }
    float v = acc;
    if (p.scale) v = __fadd_rn(__fmul_rn(v, p.scale[k]), p.shift ? p.shift[k] : 0.f);
    else if (p.shift) v = __fadd_rn(v, p.shift[k]);
    if (p.bias) v = __fadd_rn(v, p.bias[k]);
    const size_t pix = ((size_t)oh * p.OW + ow) * p.y + j;
    const size_t plane = (size_t)p.OH * p.OW * p.y;
    if (p.res) v = __fadd_rn(v, p.res[((size_t)n * p.res_cb_total + p.res_cb_off + kb) * plane + pix]);
    if (p.relu) v = fmaxf(v, 0.f);
    if (p.round_tf32) v = neo_round_tf32(v);
    p.out[((size_t)n * p.out_cb_total + p.out_cb_off + kb) * plane + pix] = v;
  }
}

}  // namespace

int neo_conv_simt_launch(const neo_conv_params* p, cudaStream_t stream) {
  NEO_CHECK_ARG(p->out_dtype == NEO_F32, NEO_ERR_UNSUPPORTED, "fp32 conv writes f32");
  ConvSimtParams k;
  k.x = static_cast<const float*>(p->x);
  k.w = static_cast<const float*>(p->w);
  k.out = static_cast<float*>(p->out);
  k.scale = p->scale;
  k.shift = p->shift;
  k.bias = p->bias;
  k.res = static_cast<const float*>(p->residual);
  k.relu = p->relu;
  k.round_tf32 = (p->flags & NEO_FLAG_ROUND_TF32) ? 1 : 0;
  k.N = (int)p->n;
  k.x_bn = p->ic_bn;
  k.y = p->oc_bn;
  k.Cb = (int)neo_ceil_div(p->c, p->ic_bn);
  k.H = (int)p->h;
  k.W = (int)p->w_in;
  k.K = (int)p->k;
  k.R = (int)p->r;
  k.S = (int)p->s;
  k.sh = p->stride_h;
  k.sw = p->stride_w;
  k.ph = p->pad_h;
  k.pw = p->pad_w;
  k.OH = (int)((p->h + 2 * p->pad_h - p->r) / p->stride_h + 1);
  k.OW = (int)((p->w_in + 2 * p->pad_w - p->s) / p->stride_w + 1);
  const int kbt = (int)neo_ceil_div(p->k, p->oc_bn);
  k.x_cb_off = p->x_cb_offset;
  k.x_cb_total = p->x_cb_total > 0 ? p->x_cb_total : k.Cb;
  k.out_cb_off = p->out_cb_offset;
  k.out_cb_total = p->out_cb_total > 0 ? p->out_cb_total : kbt;
  k.res_cb_off = p->res_cb_offset;
  k.res_cb_total = p->res_cb_total > 0 ? p->res_cb_total : kbt;
  const int64_t total = (int64_t)k.N * kbt * p->oc_bn * k.OH * k.OW;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>(neo_ceil_div(total, threads), 148 * 64);
  neo_launch(conv_simt_kernel, (int)std::max<int64_t>(blocks, 1), threads, 0, stream, k);
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}
