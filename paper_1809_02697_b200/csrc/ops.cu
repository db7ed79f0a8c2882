// Memory-bound operators on the blocked layout (reference executor.py:96-203):
// K-POOL, K-ELTWISE, K-CONCAT, K-DENSE (SIMT, HBM-bound weight stream) and
// K-SOFTMAX.  Channel-blocked tensors are (n, cb, hw, x) with x innermost, so
// consecutive threads take consecutive lanes / pixels and every access is
// coalesced; fp32 arithmetic follows the reference's numpy op order.
#include <cfloat>
#include <type_traits>

#include "neo_common.cuh"

namespace {

// channel-block windows: a tensor that is the [off, off + Cb) block range of
// a (n, total, ...) buffer (concat-in-place destinations / sources)
struct Win {
  int64_t in_off, in_total, out_off, out_total;
  __device__ __forceinline__ int64_t in_plane(int64_t plane, int64_t Cb) const {
    return (plane / Cb) * in_total + in_off + plane % Cb;
  }
  __device__ __forceinline__ int64_t out_plane(int64_t plane, int64_t Cb) const {
    return (plane / Cb) * out_total + out_off + plane % Cb;
  }
};

int64_t grid_for(int64_t total, int threads = 256) {
  return std::max<int64_t>(1, std::min<int64_t>(neo_ceil_div(total, threads), 148 * 32));
}

// _pool2d (executor.py:103-128): max pads with -inf, avg pads with 0 and
// divides by win*win; window taps visited r-major like the reference
template <typename T>
__global__ void pool_kernel(const T* __restrict__ in, T* __restrict__ out, int64_t N, int64_t Cb,
                            int H, int W, int OH, int OW, int x, int win, int stride, int pad,
                            bool is_max, bool round, Win wnd) {
  neo_pdl_enter();
  const int64_t total = N * Cb * OH * OW * x;
  const float inv = (float)(win * win);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int j = (int)(t % x);
    t /= x;
    const int ow = (int)(t % OW);
    t /= OW;
    const int oh = (int)(t % OH);
    const int64_t plane = t / OH;  // n*Cb + cb
    const T* src = in + wnd.in_plane(plane, Cb) * H * W * x + j;
    float acc = is_max ? -INFINITY : 0.f;
    bool first = true;
    for (int r = 0; r < win; ++r) {
      const int ih = oh * stride + r - pad;
      for (int s = 0; s < win; ++s) {
        const int iw = ow * stride + s - pad;
        const bool inb = ih >= 0 && ih < H && iw >= 0 && iw < W;
        const float v = inb ? Elem<T>::to_f(src[((int64_t)ih * W + iw) * x]) : (is_max ? -INFINITY : 0.f);
        if (first) {
          acc = v;
          first = false;
        } else if (is_max) {
          acc = fmaxf(acc, v);
        } else {
          acc = __fadd_rn(acc, v);
        }
      }
    }
    if (!is_max) acc = __fdiv_rn(acc, inv);
    if (round) acc = neo_round_tf32(acc);
    out[((wnd.out_plane(plane, Cb) * OH + oh) * OW + ow) * x + j] = Elem<T>::from_f(acc);
  }
}

template <typename T>
__global__ void eltwise_kernel(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out,
                               const float* __restrict__ scale, const float* __restrict__ shift,
                               int64_t total, int64_t Cb, int64_t HW, int x, int op, bool round,
                               Win wnd) {
  neo_pdl_enter();
  const int64_t plane_sz = HW * x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t plane = i / plane_sz, inner = i % plane_sz;
    float v = Elem<T>::to_f(a[wnd.in_plane(plane, Cb) * plane_sz + inner]);
    switch (op) {
      case NEO_ELT_RELU: v = fmaxf(v, 0.f); break;
      case NEO_ELT_ADD: v = __fadd_rn(v, Elem<T>::to_f(b[i])); break;
      case NEO_ELT_ADD_RELU: v = fmaxf(__fadd_rn(v, Elem<T>::to_f(b[i])), 0.f); break;
      default: {
        const int64_t j = i % x;
        const int64_t cb = (i / ((int64_t)x * HW)) % Cb;
        const int64_t ch = cb * x + j;
        // executor.py:180-181: a * scale + shift as two rounded numpy ops
        v = __fadd_rn(__fmul_rn(v, scale[ch]), shift[ch]);
        if (op == NEO_ELT_SCALE_SHIFT_RELU) v = fmaxf(v, 0.f);
      }
    }
    if (round) v = neo_round_tf32(v);
    out[wnd.out_plane(plane, Cb) * plane_sz + inner] = Elem<T>::from_f(v);
  }
}

// Plane-major vector kernels: blockIdx.y walks the (n, cb) planes (window
// mapping once per plane), blockIdx.x the V-lane vectors inside a plane with
// 32-bit index math, 16-byte loads and stores.
inline __device__ void unpack_vec(const uint4& raw, float* v, const float*) {
  const float* e = reinterpret_cast<const float*>(&raw);
#pragma unroll
  for (int j = 0; j < 4; ++j) v[j] = e[j];
}
inline __device__ void unpack_vec(const uint4& raw, float* v, const __nv_bfloat16*) {
  const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = __bfloat162float(e[j]);
}
template <typename T, int V>
__device__ __forceinline__ uint4 pack_vec(const float* v) {
  uint4 raw;
  T* e = reinterpret_cast<T*>(&raw);
#pragma unroll
  for (int j = 0; j < V; ++j) e[j] = Elem<T>::from_f(v[j]);
  return raw;
}

dim3 plane_grid(int64_t planes, int64_t per_plane, int threads = 256) {
  const int64_t bx = std::max<int64_t>(1, std::min<int64_t>(neo_ceil_div(per_plane, threads), 1024));
  const int64_t by = std::max<int64_t>(1, std::min<int64_t>(planes, 65535));
  return dim3((unsigned)bx, (unsigned)by);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// 16-byte vector of V lanes as V/2 f32 pairs (sm_100 packed f32x2 adds)
template <typename T>
struct Pair;
template <>
struct Pair<float> {
  static __device__ __forceinline__ float2 get(const uint4& r, int k) {
    return reinterpret_cast<const float2*>(&r)[k];
  }
};
template <>
struct Pair<__nv_bfloat16> {
  static __device__ __forceinline__ float2 get(const uint4& r, int k) {
    return __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(&r)[k]);
  }
};

// a / d correctly rounded (== __fdiv_rn(a, d)) for a constant d that is not
// a power of two, with r = RN(1/d): q = RN(a r), the remainder a - d q is
// exact through one FMA, and q + rem r rounded once is RN(a / d)
// (Markstein's correction step; a / d is never a rounding midpoint because d
// is odd-scaled).  Three instructions instead of the ~20-instruction IEEE
// division with its special-case path; zero keeps its sign, and inf / NaN
// pass through from q (pinned on the CPU: tests/test_host.py).
__device__ __forceinline__ float div_rn_const(float a, float d, float r) {
  const float q = a * r;
  const float rem = fmaf(-q, d, a);
  const float q1 = fmaf(rem, r, q);
  return isfinite(q) ? copysignf(q1, a) : q;
}

// _pool2d (executor.py:103-128).  Avg: padding taps add zero (skipped) and
// the sum runs r-major then divides by win*win, lane pairs in packed f32x2
// adds; max: padding is -inf (skipped), bf16 max is exact in bf16x2.
template <typename T, int V, bool IS_MAX, int WIN>
__global__ void pool_plane_vec(const T* __restrict__ in, T* __restrict__ out, int64_t Cb,
                               int64_t P, int H, int W, int OH, int OW, int x, int win_rt,
                               int stride, int pad, bool round, Win wnd) {
  neo_pdl_enter();
  constexpr int NP = V / 2;
  const int win = WIN > 0 ? WIN : win_rt;
  const uint32_t groups = x / V;
  const uint32_t per_plane = (uint32_t)OH * OW * groups;
  const float inv = (float)(win * win);
  for (int64_t plane = blockIdx.y; plane < P; plane += gridDim.y) {
    const T* src = in + wnd.in_plane(plane, Cb) * H * W * x;
    T* dst = out + wnd.out_plane(plane, Cb) * OH * OW * x;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < per_plane;
         i += gridDim.x * blockDim.x) {
      const uint32_t gq = i % groups, t = i / groups;
      const int ow = (int)(t % (uint32_t)OW), oh = (int)(t / (uint32_t)OW);
      const int ih0 = oh * stride - pad, iw0 = ow * stride - pad;
      const T* base = src + gq * V;
      uint4 res;
      if constexpr (!IS_MAX && WIN > 0) {
        // average pooling, branch-free: all WIN*WIN taps are loaded at once
        // (clamped addresses, so every load is in bounds) and out-of-bounds
        // taps contribute the reference's zero padding (+0.0); the sum keeps
        // the reference order -- first tap, then + each tap r-major
        // (executor.py:116-126) -- and divides by win*win (count_include_pad)
        int rows[WIN], cols[WIN];
        bool rin[WIN], cin[WIN];
#pragma unroll
        for (int r = 0; r < WIN; ++r) {
          rin[r] = ih0 + r >= 0 && ih0 + r < H;
          rows[r] = min(max(ih0 + r, 0), H - 1) * W;
        }
#pragma unroll
        for (int q = 0; q < WIN; ++q) {
          cin[q] = iw0 + q >= 0 && iw0 + q < W;
          cols[q] = min(max(iw0 + q, 0), W - 1);
        }
        uint4 raw[WIN * WIN];
#pragma unroll
        for (int r = 0; r < WIN; ++r)
#pragma unroll
          for (int q = 0; q < WIN; ++q)
            raw[r * WIN + q] = __ldg(reinterpret_cast<const uint4*>(base + (rows[r] + cols[q]) * x));
        float2 acc[NP];
#pragma unroll
        for (int t2 = 0; t2 < WIN * WIN; ++t2) {
          const bool in_b = rin[t2 / WIN] && cin[t2 % WIN];
#pragma unroll
          for (int k = 0; k < NP; ++k) {
            const float2 v = in_b ? Pair<T>::get(raw[t2], k) : make_float2(0.f, 0.f);
            acc[k] = t2 == 0 ? v : __fadd2_rn(acc[k], v);
          }
        }
        float o[V];
        constexpr int kWin2 = WIN * WIN;
        constexpr bool kPow2 = (kWin2 & (kWin2 - 1)) == 0;
        const float rcp = 1.0f / (float)kWin2;     // RN(1/win^2), a compile-time constant
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          // power-of-two windows: the division is an exact scaling
          o[2 * k] = kPow2 ? acc[k].x * rcp : div_rn_const(acc[k].x, (float)kWin2, rcp);
          o[2 * k + 1] = kPow2 ? acc[k].y * rcp : div_rn_const(acc[k].y, (float)kWin2, rcp);
        }
        if (round) {
#pragma unroll
          for (int j = 0; j < V; ++j) o[j] = neo_round_tf32(o[j]);
        }
        res = pack_vec<T, V>(o);
      } else if constexpr (IS_MAX && sizeof(T) == 2 && WIN > 0) {
        // max pooling: an out-of-bounds tap is clamped to the nearest row /
        // column, which always lies inside the same window (pad < win), so
        // the maximum is unchanged and all WIN*WIN loads are issued
        // unconditionally before the reduction
        int rows[WIN], cols[WIN];
#pragma unroll
        for (int r = 0; r < WIN; ++r) rows[r] = min(max(ih0 + r, 0), H - 1) * W;
#pragma unroll
        for (int q = 0; q < WIN; ++q) cols[q] = min(max(iw0 + q, 0), W - 1);
        uint4 raw[WIN * WIN];
#pragma unroll
        for (int r = 0; r < WIN; ++r)
#pragma unroll
          for (int q = 0; q < WIN; ++q)
            raw[r * WIN + q] = __ldg(reinterpret_cast<const uint4*>(base + (rows[r] + cols[q]) * x));
        __nv_bfloat162 m[NP];
#pragma unroll
        for (int k = 0; k < NP; ++k) m[k] = reinterpret_cast<const __nv_bfloat162*>(&raw[0])[k];
#pragma unroll
        for (int t2 = 1; t2 < WIN * WIN; ++t2)
#pragma unroll
          for (int k = 0; k < NP; ++k)
            m[k] = __hmax2(m[k], reinterpret_cast<const __nv_bfloat162*>(&raw[t2])[k]);
#pragma unroll
        for (int k = 0; k < NP; ++k) reinterpret_cast<__nv_bfloat162*>(&res)[k] = m[k];
      } else if constexpr (IS_MAX && WIN > 0) {
        // f32 max: the same clamped-tap trick (max is order-independent)
        int rows[WIN], cols[WIN];
#pragma unroll
        for (int r = 0; r < WIN; ++r) rows[r] = min(max(ih0 + r, 0), H - 1) * W;
#pragma unroll
        for (int q = 0; q < WIN; ++q) cols[q] = min(max(iw0 + q, 0), W - 1);
        uint4 raw[WIN * WIN];
#pragma unroll
        for (int r = 0; r < WIN; ++r)
#pragma unroll
          for (int q = 0; q < WIN; ++q)
            raw[r * WIN + q] = __ldg(reinterpret_cast<const uint4*>(base + (rows[r] + cols[q]) * x));
        float o[V];
#pragma unroll
        for (int j = 0; j < V; ++j) o[j] = reinterpret_cast<const float*>(&raw[0])[j];
#pragma unroll
        for (int t2 = 1; t2 < WIN * WIN; ++t2)
#pragma unroll
          for (int j = 0; j < V; ++j) o[j] = fmaxf(o[j], reinterpret_cast<const float*>(&raw[t2])[j]);
        if (round) {
#pragma unroll
          for (int j = 0; j < V; ++j) o[j] = neo_round_tf32(o[j]);
        }
        res = pack_vec<T, V>(o);
      } else if constexpr (IS_MAX && sizeof(T) == 2) {
        __nv_bfloat162 m[NP];
#pragma unroll
        for (int k = 0; k < NP; ++k) m[k] = __bfloat162bfloat162(__float2bfloat16(-INFINITY));
#pragma unroll
        for (int r = 0; r < (WIN > 0 ? WIN : 1); ++r) {
          for (int rr = r; rr < (WIN > 0 ? r + 1 : win); ++rr) {
            const int ih = ih0 + rr;
            if (ih < 0 || ih >= H) continue;
#pragma unroll
            for (int s_ = 0; s_ < (WIN > 0 ? WIN : 1); ++s_) {
              for (int ss = s_; ss < (WIN > 0 ? s_ + 1 : win); ++ss) {
                const int iw = iw0 + ss;
                if (iw < 0 || iw >= W) continue;
                const uint4 raw = __ldg(reinterpret_cast<const uint4*>(base + (ih * W + iw) * x));
#pragma unroll
                for (int k = 0; k < NP; ++k)
                  m[k] = __hmax2(m[k], reinterpret_cast<const __nv_bfloat162*>(&raw)[k]);
              }
            }
          }
        }
#pragma unroll
        for (int k = 0; k < NP; ++k) reinterpret_cast<__nv_bfloat162*>(&res)[k] = m[k];
      } else {
        float2 acc[NP];
#pragma unroll
        for (int k = 0; k < NP; ++k) acc[k] = IS_MAX ? make_float2(-INFINITY, -INFINITY)
                                                     : make_float2(0.f, 0.f);
#pragma unroll
        for (int r = 0; r < (WIN > 0 ? WIN : 1); ++r) {
          for (int rr = r; rr < (WIN > 0 ? r + 1 : win); ++rr) {
            const int ih = ih0 + rr;
            if (ih < 0 || ih >= H) continue;
#pragma unroll
            for (int s_ = 0; s_ < (WIN > 0 ? WIN : 1); ++s_) {
              for (int ss = s_; ss < (WIN > 0 ? s_ + 1 : win); ++ss) {
                const int iw = iw0 + ss;
                if (iw < 0 || iw >= W) continue;
                const uint4 raw = __ldg(reinterpret_cast<const uint4*>(base + (ih * W + iw) * x));
#pragma unroll
                for (int k = 0; k < NP; ++k) {
                  const float2 v = Pair<T>::get(raw, k);
                  if (IS_MAX)
                    acc[k] = make_float2(fmaxf(acc[k].x, v.x), fmaxf(acc[k].y, v.y));
                  else
                    acc[k] = __fadd2_rn(acc[k], v);
                }
              }
            }
          }
        }
        float o[V];
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          o[2 * k] = IS_MAX ? acc[k].x : __fdiv_rn(acc[k].x, inv);
          o[2 * k + 1] = IS_MAX ? acc[k].y : __fdiv_rn(acc[k].y, inv);
        }
        if (round) {
#pragma unroll
          for (int j = 0; j < V; ++j) o[j] = neo_round_tf32(o[j]);
        }
        res = pack_vec<T, V>(o);
      }
      *reinterpret_cast<uint4*>(dst + (oh * OW + ow) * x + gq * V) = res;
    }
  }
}

// Global pooling (window == H == W, no padding, 1x1 output: the classifier
// head): one thread per lane pair, taps summed r-major in order like the
// reference, loads issued 8 at a time for memory-level parallelism.
template <typename T, bool IS_MAX>
__global__ void pool_global(const T* __restrict__ in, T* __restrict__ out, int64_t Cb,
                            int64_t P, int HW, int x, float inv, bool round, Win wnd) {
  neo_pdl_enter();
  using T2 = typename std::conditional<sizeof(T) == 2, __nv_bfloat162, float2>::type;
  const int pairs = x / 2;
  const int64_t total = P * pairs;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t plane = i / pairs;
    const int lp = (int)(i % pairs);
    const T2* src = reinterpret_cast<const T2*>(in + wnd.in_plane(plane, Cb) * HW * x) + lp;
    float2 acc = IS_MAX ? make_float2(-INFINITY, -INFINITY) : make_float2(0.f, 0.f);
    int t = 0;
    for (; t + 8 <= HW; t += 8) {
      T2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(src + (t + u) * pairs);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        float2 f;
        if constexpr (sizeof(T) == 2) f = __bfloat1622float2(v[u]);
        else f = v[u];
        acc = IS_MAX ? make_float2(fmaxf(acc.x, f.x), fmaxf(acc.y, f.y)) : __fadd2_rn(acc, f);
      }
    }
    for (; t < HW; ++t) {
      float2 f;
      if constexpr (sizeof(T) == 2) f = __bfloat1622float2(__ldg(src + t * pairs));
      else f = __ldg(src + t * pairs);
      acc = IS_MAX ? make_float2(fmaxf(acc.x, f.x), fmaxf(acc.y, f.y)) : __fadd2_rn(acc, f);
    }
    if (!IS_MAX) acc = make_float2(__fdiv_rn(acc.x, inv), __fdiv_rn(acc.y, inv));
    if (round) acc = make_float2(neo_round_tf32(acc.x), neo_round_tf32(acc.y));
    T2 o;
    if constexpr (sizeof(T) == 2) o = __float22bfloat162_rn(acc);
    else o = acc;
    reinterpret_cast<T2*>(out + wnd.out_plane(plane, Cb) * x)[lp] = o;
  }
}

// 3x3 stride-1 average pooling (Inception's branch pools, pad 1,
// count_include_pad) with a sliding window along W: a thread produces OUTW
// consecutive output pixels of one 8-lane group, loading each input row's
// OUTW + 2 taps once (3x fewer loads and bf16->f32 conversions than one
// output per thread), while every output still sums its nine taps in the
// reference order -- first tap, then + each tap r-major (executor.py:116-126)
// -- with the padding taps contributing +0.0, then one division by 9.
template <int OUTW>
__global__ void avgpool3s1_bf16(const __nv_bfloat16* __restrict__ in,
                                __nv_bfloat16* __restrict__ out, int64_t Cb, uint32_t P, int H,
                                int W, int x, uint32_t chunks_w, bool round, Win wnd) {
  neo_pdl_enter();
  constexpr int NP = 4;                           // float2 pairs per 16-byte vector
  const uint32_t groups = (uint32_t)x / 8u;
  const uint32_t per_plane = (uint32_t)H * chunks_w * groups;
  const uint32_t total = P * per_plane;
  const float rcp = 1.0f / 9.0f;
  for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += gridDim.x * blockDim.x) {
    const uint32_t plane = idx / per_plane;
    uint32_t rem = idx - plane * per_plane;
    const uint32_t gq = rem % groups;
    rem /= groups;
    const int oh = (int)(rem / chunks_w);
    const int ow0 = (int)(rem - (uint32_t)oh * chunks_w) * OUTW;
    const uint32_t pn = plane / (uint32_t)Cb, pc = plane - pn * (uint32_t)Cb;
    const __nv_bfloat16* src =
        in + ((int64_t)pn * wnd.in_total + wnd.in_off + pc) * (int64_t)H * W * x + gq * 8;
    __nv_bfloat16* dst =
        out + ((int64_t)pn * wnd.out_total + wnd.out_off + pc) * (int64_t)H * W * x + gq * 8;
    float2 acc[OUTW][NP];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int ih = oh - 1 + r;
      const bool rin = ih >= 0 && ih < H;
      const int ihc = min(max(ih, 0), H - 1);
      uint4 raw[OUTW + 2];
#pragma unroll
      for (int c = 0; c < OUTW + 2; ++c) {
        const int iw = min(max(ow0 - 1 + c, 0), W - 1);
        raw[c] = __ldg(reinterpret_cast<const uint4*>(src + ((int64_t)ihc * W + iw) * x));
      }
      float2 t[OUTW + 2][NP];
#pragma unroll
      for (int c = 0; c < OUTW + 2; ++c) {
        const int iw = ow0 - 1 + c;
        const bool in_b = rin && iw >= 0 && iw < W;
#pragma unroll
        for (int k = 0; k < NP; ++k)
          t[c][k] = in_b ? Pair<__nv_bfloat16>::get(raw[c], k) : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < OUTW; ++j)
#pragma unroll
        for (int s = 0; s < 3; ++s)
#pragma unroll
          for (int k = 0; k < NP; ++k)
            acc[j][k] = (r == 0 && s == 0) ? t[j + s][k] : __fadd2_rn(acc[j][k], t[j + s][k]);
    }
#pragma unroll
    for (int j = 0; j < OUTW; ++j) {
      if (ow0 + j >= W) break;
      float o[8];
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        o[2 * k] = div_rn_const(acc[j][k].x, 9.0f, rcp);
        o[2 * k + 1] = div_rn_const(acc[j][k].y, 9.0f, rcp);
      }
      if (round) {
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = neo_round_tf32(o[e]);
      }
      *reinterpret_cast<uint4*>(dst + ((int64_t)oh * W + ow0 + j) * x) =
          pack_vec<__nv_bfloat16, 8>(o);
    }
  }
}

// e4m3 pooling (FP8 mode), 16 lanes per thread.  Max: e4m3 -> f16 is exact,
// the maximum in f16x2 (padding -inf) is one of the stored values; avg: the
// reference's sum order (first tap, then + each tap r-major, padding +0)
// of the dequantized values in f32, / win^2 (count_include_pad).  The result
// times in_scale / out_scale (powers of two: exact) is rounded once to e4m3
// -- a max pool with out_scale == in_scale returns the winning bytes.
__device__ __forceinline__ void e4m3x16_to_f32(const uint4& raw, float* v) {
  const uint32_t w4[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const __nv_fp8x2_storage_t pr = (__nv_fp8x2_storage_t)(w4[k >> 1] >> (16 * (k & 1)));
    const float2 f = __half22float2(__half2(__nv_cvt_fp8x2_to_halfraw2(pr, __NV_E4M3)));
    v[2 * k] = f.x;
    v[2 * k + 1] = f.y;
  }
}
__device__ __forceinline__ uint4 f32x16_to_e4m3(const float* v) {
  uint32_t o[4];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    o[k] = (uint32_t)__nv_cvt_float2_to_fp8x2(make_float2(v[4 * k], v[4 * k + 1]), __NV_SATFINITE, __NV_E4M3) |
           ((uint32_t)__nv_cvt_float2_to_fp8x2(make_float2(v[4 * k + 2], v[4 * k + 3]), __NV_SATFINITE, __NV_E4M3) << 16);
  return make_uint4(o[0], o[1], o[2], o[3]);
}

__global__ void pool_fp8(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int64_t Cb,
                         int64_t P, int H, int W, int OH, int OW, int x, int win, int stride,
                         int pad, bool is_max, float in_scale, float qs, Win wnd) {
  neo_pdl_enter();
  const uint32_t groups = x / 16;
  const uint32_t per_plane = (uint32_t)OH * OW * groups;
  const float inv = (float)(win * win);
  for (int64_t plane = blockIdx.y; plane < P; plane += gridDim.y) {
    const uint8_t* src = in + wnd.in_plane(plane, Cb) * H * W * x;
    uint8_t* dst = out + wnd.out_plane(plane, Cb) * OH * OW * x;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < per_plane;
         i += gridDim.x * blockDim.x) {
      const uint32_t gq = i % groups, t = i / groups;
      const int ow = (int)(t % (uint32_t)OW), oh = (int)(t / (uint32_t)OW);
      float acc[16];
      bool first = true;
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[k] = is_max ? -INFINITY : 0.f;
      for (int r = 0; r < win; ++r) {
        const int ih = oh * stride + r - pad;
        for (int q = 0; q < win; ++q) {
          const int iw = ow * stride + q - pad;
          const bool inb = ih >= 0 && ih < H && iw >= 0 && iw < W;
          if (!inb && is_max) continue;                 // -inf padding
          float v[16];                                  // avg: +0 padding taps
          if (inb)
            e4m3x16_to_f32(__ldg(reinterpret_cast<const uint4*>(src + ((int64_t)ih * W + iw) * x + gq * 16)), v);
          else
#pragma unroll
            for (int k = 0; k < 16; ++k) v[k] = 0.f;
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            if (is_max) acc[k] = fmaxf(acc[k], v[k]);
            else acc[k] = first ? v[k] * in_scale : __fadd_rn(acc[k], v[k] * in_scale);
          }
          first = false;
        }
      }
#pragma unroll
      for (int k = 0; k < 16; ++k)
        acc[k] = is_max ? acc[k] * in_scale * qs : __fdiv_rn(acc[k], inv) * qs;
      *reinterpret_cast<uint4*>(dst + ((int64_t)oh * OW + ow) * x + gq * 16) = f32x16_to_e4m3(acc);
    }
  }
}

// e4m3 elementwise (FP8 mode): relu / scale-shift(-relu) (BN, executor.py:
// 174-181, a * scale + shift as two rounded ops) of the dequantized values,
// then one rounding to e4m3 at the output's scale; 16 lanes per thread
__global__ void eltwise_fp8(const uint8_t* __restrict__ a, uint8_t* __restrict__ out,
                            const float* __restrict__ scale, const float* __restrict__ shift,
                            int64_t Cb, int64_t P, int64_t HW, int x, int op, float a_scale,
                            float qs, Win wnd) {
  neo_pdl_enter();
  const int64_t groups = HW * (x / 16);
  const int64_t total = P * groups;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t plane = i / groups, g = i % groups;
    const int lane0 = (int)(g % (x / 16)) * 16;
    const int64_t cb = plane % Cb;
    float v[16];
    e4m3x16_to_f32(__ldg(reinterpret_cast<const uint4*>(a + wnd.in_plane(plane, Cb) * HW * x + g * 16)), v);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      float y = v[k] * a_scale;
      if (op == NEO_ELT_SCALE_SHIFT || op == NEO_ELT_SCALE_SHIFT_RELU) {
        const int64_t ch = cb * x + lane0 + k;
        y = __fadd_rn(__fmul_rn(y, __ldg(scale + ch)), __ldg(shift + ch));
      }
      if (op != NEO_ELT_SCALE_SHIFT) y = fmaxf(y, 0.f);
      v[k] = y * qs;
    }
    *reinterpret_cast<uint4*>(out + wnd.out_plane(plane, Cb) * HW * x + g * 16) = f32x16_to_e4m3(v);
  }
}

template <typename T, int V, bool IS_MAX>
void launch_pool_vec(const T* in, T* out, int64_t cb, int64_t P, int h, int w, int OH, int OW,
                     int x, int win, int stride, int pad, bool round, Win wnd, cudaStream_t st) {
  const dim3 grid = plane_grid(P, (int64_t)OH * OW * (x / V));
  if (win == 3)
    neo_launch(pool_plane_vec<T, V, IS_MAX, 3>, grid, 256, 0, st, in, out, cb, P, h, w, OH, OW, x, win,
                                                          stride, pad, round, wnd);
  else if (win == 2)
    neo_launch(pool_plane_vec<T, V, IS_MAX, 2>, grid, 256, 0, st, in, out, cb, P, h, w, OH, OW, x, win,
                                                          stride, pad, round, wnd);
  else
    neo_launch(pool_plane_vec<T, V, IS_MAX, 0>, grid, 256, 0, st, in, out, cb, P, h, w, OH, OW, x, win,
                                                          stride, pad, round, wnd);
}

// Elementwise ops over (plane, vector) flattened into one index space: a
// grid of a few CTAs per SM, each thread holding U independent 16-byte loads
// in flight (DenseNet's BN-ReLU launches are small, so per-block scheduling
// and a single outstanding load per thread, not HBM, bounded the old
// one-vector-per-thread plane grid).
template <typename T, int V, int U>
__global__ void eltwise_flat_vec(const T* __restrict__ a, const T* __restrict__ b,
                                 T* __restrict__ out, const float* __restrict__ scale,
                                 const float* __restrict__ shift, int64_t Cb, uint32_t total,
                                 uint32_t vecs, int64_t plane_sz, int x, int op, bool round,
                                 Win wnd) {
  neo_pdl_enter();
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint4* av = reinterpret_cast<const uint4*>(a);
  const uint4* bv = reinterpret_cast<const uint4*>(b);
  uint4* ov = reinterpret_cast<uint4*>(out);
  const int64_t pv = plane_sz / V;               // vectors per plane
  for (uint32_t base = blockIdx.x * blockDim.x + threadIdx.x; base < total; base += stride * U) {
    uint4 ra[U], rb[U];
    int64_t oo[U];
    int ch[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t idx = base + u * stride;
      const bool ok = idx < total;
      const uint32_t plane = ok ? idx / vecs : 0u;
      const uint32_t i = ok ? idx - plane * vecs : 0u;
      // 32-bit plane decode (image, channel block) -- the windows' int64
      // divisions would dominate this memory-bound loop
      const uint32_t pn = plane / (uint32_t)Cb, pc = plane - pn * (uint32_t)Cb;
      oo[u] = ok ? ((int64_t)pn * wnd.out_total + wnd.out_off + pc) * pv + i : -1;
      ch[u] = (int)pc * x + (int)((i * V) % (uint32_t)x);
      ra[u] = ok ? __ldg(av + ((int64_t)pn * wnd.in_total + wnd.in_off + pc) * pv + i)
                 : make_uint4(0, 0, 0, 0);
      if (op == NEO_ELT_ADD || op == NEO_ELT_ADD_RELU)
        rb[u] = ok ? __ldg(bv + (int64_t)plane * pv + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (oo[u] < 0) continue;
      float v[V];
      unpack_vec(ra[u], v, (const T*)nullptr);
      if (op == NEO_ELT_ADD || op == NEO_ELT_ADD_RELU) {
        float w[V];
        unpack_vec(rb[u], w, (const T*)nullptr);
#pragma unroll
        for (int j = 0; j < V; ++j) {
          v[j] = __fadd_rn(v[j], w[j]);
          if (op == NEO_ELT_ADD_RELU) v[j] = fmaxf(v[j], 0.f);
        }
      } else if (op == NEO_ELT_RELU) {
#pragma unroll
        for (int j = 0; j < V; ++j) v[j] = fmaxf(v[j], 0.f);
      } else {
        float sc[V], sh[V];
#pragma unroll
        for (int j = 0; j < V; j += 4) {
          const float4 s4 = __ldg(reinterpret_cast<const float4*>(scale + ch[u] + j));
          const float4 h4 = __ldg(reinterpret_cast<const float4*>(shift + ch[u] + j));
          sc[j] = s4.x; sc[j + 1] = s4.y; sc[j + 2] = s4.z; sc[j + 3] = s4.w;
          sh[j] = h4.x; sh[j + 1] = h4.y; sh[j + 2] = h4.z; sh[j + 3] = h4.w;
        }
#pragma unroll
        for (int j = 0; j < V; ++j) {
          // executor.py:180-181: a * scale + shift as two rounded numpy ops
          v[j] = __fadd_rn(__fmul_rn(v[j], sc[j]), sh[j]);
          if (op == NEO_ELT_SCALE_SHIFT_RELU) v[j] = fmaxf(v[j], 0.f);
        }
      }
      if (round) {
#pragma unroll
        for (int j = 0; j < V; ++j) v[j] = neo_round_tf32(v[j]);
      }
      ov[oo[u]] = pack_vec<T, V>(v);
    }
  }
}

// grid-stride launches: at most 8 CTAs of 256 threads per B200 SM (no device
// query here -- these launches are recorded inside CUDA-graph capture)
static unsigned flat_grid(uint64_t total_vecs, int U, int threads = 256) {
  const uint64_t want = (total_vecs + (uint64_t)threads * U - 1) / ((uint64_t)threads * U);
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, 148ull * 8));
}

template <typename T>
__global__ void concat_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t outer,
                              int64_t chunk, int64_t dst_row, int64_t dst_off) {
  neo_pdl_enter();
  const int64_t total = outer * chunk;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = i / chunk, c = i % chunk;
    dst[o * dst_row + dst_off + c] = src[i];
  }
}

// 16-byte vector variant when every row boundary is 16-byte aligned
__global__ void concat_kernel_v4(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                 int64_t outer, int64_t chunk, int64_t dst_row, int64_t dst_off) {
  neo_pdl_enter();
  const int64_t total = outer * chunk;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = i / chunk, c = i % chunk;
    dst[o * dst_row + dst_off + c] = src[i];
  }
}

// Dense: one warp per output unit, all (<= 8 per pass) batch rows at once so
// each weight row streams from HBM exactly once per pass.
template <typename T, int NB>
__global__ void dense_kernel(const T* __restrict__ a, const T* __restrict__ w,
                             const float* __restrict__ bias, float* __restrict__ out, int64_t n,
                             int64_t in_f, int64_t units) {
  neo_pdl_enter();
  const int warps = blockDim.x / 32;
  const int64_t u = (int64_t)blockIdx.x * warps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (u >= units) return;
  const T* wr = w + u * in_f;
  for (int64_t n0 = blockIdx.y * NB; n0 < n; n0 += (int64_t)gridDim.y * NB) {
    float acc[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[b] = 0.f;
    for (int64_t i = lane; i < in_f; i += 32) {
      const float wv = Elem<T>::to_f(wr[i]);
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if (n0 + b < n) acc[b] = fmaf(Elem<T>::to_f(a[(n0 + b) * in_f + i]), wv, acc[b]);
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      float v = acc[b];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && n0 + b < n) out[(n0 + b) * units + u] = bias ? v + bias[u] : v;
    }
  }
}

// softmax over the last axis: e = exp(a - max); e / sum(e)   (executor.py:167-170)
__global__ void softmax_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t rows,
                               int64_t cols) {
  neo_pdl_enter();
  __shared__ float red[32];
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const float* a = in + row * cols;
    float* o = out + row * cols;
    float mx = -INFINITY;
    for (int64_t i = threadIdx.x; i < cols; i += blockDim.x) mx = fmaxf(mx, a[i]);
    for (int s = 16; s > 0; s >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, s));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
      float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : -INFINITY;
      for (int s = 16; s > 0; s >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, s));
      if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    mx = red[0];
    __syncthreads();
    float sum = 0.f;
    for (int64_t i = threadIdx.x; i < cols; i += blockDim.x) {
      const float e = expf(a[i] - mx);
      o[i] = e;
      sum += e;
    }
    for (int s = 16; s > 0; s >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = sum;
    __syncthreads();
    if (threadIdx.x < 32) {
      float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
      for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
      if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const float inv = red[0];
    for (int64_t i = threadIdx.x; i < cols; i += blockDim.x) o[i] = o[i] / inv;
    __syncthreads();
  }
}

}  // namespace

extern "C" int neo_pool2d_window(int dtype, int mode, const void* in, void* out, int64_t n,
                                 int64_t cb, int64_t h, int64_t w, int x, int win, int stride,
                                 int pad, int64_t in_cb_off, int64_t in_cb_total,
                                 int64_t out_cb_off, int64_t out_cb_total, int flags,
                                 neo_stream_t stream) {
  NEO_CHECK_ARG(in && out, NEO_ERR_INVALID_ARG, "null tensor pointer");
  NEO_CHECK_ARG(win >= 1 && stride >= 1 && pad >= 0 && x >= 1, NEO_ERR_INVALID_ARG,
                "bad pool window/stride/pad");
  NEO_CHECK_ARG(in_cb_off >= 0 && in_cb_off + cb <= in_cb_total && out_cb_off >= 0 &&
                    out_cb_off + cb <= out_cb_total,
                NEO_ERR_SHAPE_MISMATCH, "channel-block window out of range");
  const int64_t OH = (h + 2 * pad - win) / stride + 1, OW = (w + 2 * pad - win) / stride + 1;
  NEO_CHECK_ARG(OH >= 1 && OW >= 1, NEO_ERR_SHAPE_MISMATCH, "pool has empty output");
  const int64_t total = n * cb * OH * OW * x;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool round = (flags & NEO_FLAG_ROUND_TF32) != 0;
  const Win wnd{in_cb_off, in_cb_total, out_cb_off, out_cb_total};
  const int64_t P = n * cb;
  const bool al = aligned16(in) && aligned16(out);
  const bool is_max = mode == NEO_POOL_MAX;
  const bool global = OH == 1 && OW == 1 && pad == 0 && win == h && win == w && x % 2 == 0;
  if (dtype == NEO_FP8) {
    // e4m3 maps without scales: max pooling (the map keeps its scale); an
    // average needs neo_pool2d_q's output scale
    NEO_CHECK_ARG(is_max, NEO_ERR_UNSUPPORTED, "e4m3 average pooling needs neo_pool2d_q");
    return neo_pool2d_q(mode, in, out, n, cb, h, w, x, win, stride, pad, in_cb_off, in_cb_total,
                        out_cb_off, out_cb_total, 1.f, 1.f, stream);
  }
  if (global) {
    const float inv = (float)(win * win);
    const unsigned grid = (unsigned)grid_for(P * (x / 2));
    if (dtype == NEO_BF16) {
      auto i = static_cast<const __nv_bfloat16*>(in);
      auto o = static_cast<__nv_bfloat16*>(out);
      if (is_max)
        neo_launch(pool_global<__nv_bfloat16, true>, grid, 256, 0, st, i, o, cb, P, (int)(h * w), x, inv,
                                                               round, wnd);
      else
        neo_launch(pool_global<__nv_bfloat16, false>, grid, 256, 0, st, i, o, cb, P, (int)(h * w), x,
                                                                inv, round, wnd);
    } else {
      auto i = static_cast<const float*>(in);
      auto o = static_cast<float*>(out);
      if (is_max)
        neo_launch(pool_global<float, true>, grid, 256, 0, st, i, o, cb, P, (int)(h * w), x, inv, round,
                                                       wnd);
      else
        neo_launch(pool_global<float, false>, grid, 256, 0, st, i, o, cb, P, (int)(h * w), x, inv, round,
                                                        wnd);
    }
  } else if (dtype == NEO_BF16 && x % 8 == 0 && al) {
    auto i = static_cast<const __nv_bfloat16*>(in);
    auto o = static_cast<__nv_bfloat16*>(out);
    if (is_max)
      launch_pool_vec<__nv_bfloat16, 8, true>(i, o, cb, P, (int)h, (int)w, (int)OH, (int)OW, x,
                                              win, stride, pad, round, wnd, st);
    else if (win == 3 && stride == 1 && pad == 1 &&
             (uint64_t)P * h * neo_ceil_div(w, 4) * (x / 8) < (1ull << 32)) {
      constexpr int kOutW = 4;
      const uint32_t chunks = (uint32_t)neo_ceil_div(w, kOutW);
      const uint64_t total = (uint64_t)P * h * chunks * (x / 8);
      neo_launch(avgpool3s1_bf16<kOutW>, flat_grid(total, 1), 256, 0, st, i, o, cb, (uint32_t)P,
                 (int)h, (int)w, x, chunks, round, wnd);
    } else
      launch_pool_vec<__nv_bfloat16, 8, false>(i, o, cb, P, (int)h, (int)w, (int)OH, (int)OW, x,
                                               win, stride, pad, round, wnd, st);
  } else if (dtype == NEO_F32 && x % 4 == 0 && al) {
    auto i = static_cast<const float*>(in);
    auto o = static_cast<float*>(out);
    if (is_max)
      launch_pool_vec<float, 4, true>(i, o, cb, P, (int)h, (int)w, (int)OH, (int)OW, x, win,
                                      stride, pad, round, wnd, st);
    else
      launch_pool_vec<float, 4, false>(i, o, cb, P, (int)h, (int)w, (int)OH, (int)OW, x, win,
                                       stride, pad, round, wnd, st);
  } else if (dtype == NEO_BF16)
    neo_launch(pool_kernel<__nv_bfloat16>, (unsigned)grid_for(total), 256, 0, st, 
        static_cast<const __nv_bfloat16*>(in), static_cast<__nv_bfloat16*>(out), n, cb, (int)h,
        (int)w, (int)OH, (int)OW, x, win, stride, pad, mode == NEO_POOL_MAX, round, wnd);
  else
    neo_launch(pool_kernel<float>, (unsigned)grid_for(total), 256, 0, st, 
        static_cast<const float*>(in), static_cast<float*>(out), n, cb, (int)h, (int)w, (int)OH,
        (int)OW, x, win, stride, pad, mode == NEO_POOL_MAX, round, wnd);
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}

extern "C" int neo_pool2d_q(int mode, const void* in, void* out, int64_t n, int64_t cb, int64_t h,
                            int64_t w, int x, int win, int stride, int pad, int64_t in_cb_off,
                            int64_t in_cb_total, int64_t out_cb_off, int64_t out_cb_total,
                            float in_scale, float out_scale, neo_stream_t stream) {
  NEO_CHECK_ARG(in && out && in_scale > 0.f && out_scale > 0.f, NEO_ERR_INVALID_ARG,
                "bad e4m3 pool arguments");
  NEO_CHECK_ARG(win >= 1 && stride >= 1 && pad >= 0 && pad < win, NEO_ERR_INVALID_ARG,
                "bad pool window/stride/pad");
  NEO_CHECK_ARG(in_cb_off >= 0 && in_cb_off + cb <= in_cb_total && out_cb_off >= 0 &&
                    out_cb_off + cb <= out_cb_total,
                NEO_ERR_SHAPE_MISMATCH, "channel-block window out of range");
  NEO_CHECK_ARG(x % 16 == 0 && aligned16(in) && aligned16(out), NEO_ERR_UNSUPPORTED,
                "e4m3 pooling needs 16-lane blocks");
  const int64_t OH = (h + 2 * pad - win) / stride + 1, OW = (w + 2 * pad - win) / stride + 1;
  NEO_CHECK_ARG(OH >= 1 && OW >= 1, NEO_ERR_SHAPE_MISMATCH, "pool has empty output");
  const Win wnd{in_cb_off, in_cb_total, out_cb_off, out_cb_total};
  const int64_t P = n * cb;
  neo_launch(pool_fp8, plane_grid(P, OH * OW * (x / 16)), 256, 0, static_cast<cudaStream_t>(stream),
             static_cast<const uint8_t*>(in), static_cast<uint8_t*>(out), cb, P, (int)h, (int)w,
             (int)OH, (int)OW, x, win, stride, pad, mode == NEO_POOL_MAX, in_scale,
             (float)(1.0 / (double)out_scale), wnd);
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}

extern "C" int neo_eltwise_q(int op, const void* a, void* out, const float* scale,
                             const float* shift, int64_t n, int64_t cb, int64_t hw, int x,
                             int64_t a_cb_off, int64_t a_cb_total, int64_t out_cb_off,
                             int64_t out_cb_total, float a_scale, float out_scale,
                             neo_stream_t stream) {
  NEO_CHECK_ARG(a && out && a_scale > 0.f && out_scale > 0.f, NEO_ERR_INVALID_ARG,
                "bad e4m3 eltwise arguments");
  NEO_CHECK_ARG(op == NEO_ELT_RELU || op == NEO_ELT_SCALE_SHIFT || op == NEO_ELT_SCALE_SHIFT_RELU,
                NEO_ERR_UNSUPPORTED, "e4m3 eltwise: relu / scale-shift(-relu) only (op %d)", op);
  NEO_CHECK_ARG(op == NEO_ELT_RELU || (scale && shift), NEO_ERR_INVALID_ARG,
                "scale/shift needs both vectors");
  NEO_CHECK_ARG(a_cb_off >= 0 && a_cb_off + cb <= a_cb_total && out_cb_off >= 0 &&
                    out_cb_off + cb <= out_cb_total,
                NEO_ERR_SHAPE_MISMATCH, "channel-block window out of range");
  NEO_CHECK_ARG(x % 16 == 0 && aligned16(a) && aligned16(out), NEO_ERR_UNSUPPORTED,
                "e4m3 eltwise needs 16-lane blocks");
  const Win wnd{a_cb_off, a_cb_total, out_cb_off, out_cb_total};
  const int64_t P = n * cb;
  neo_launch(eltwise_fp8, (unsigned)grid_for(P * hw * (x / 16)), 256, 0,
             static_cast<cudaStream_t>(stream), static_cast<const uint8_t*>(a),
             static_cast<uint8_t*>(out), scale, shift, cb, P, hw, x, op, a_scale,
             (float)(1.0 / (double)out_scale), wnd);
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}

extern "C" int neo_pool2d(int dtype, int mode, const void* in, void* out, int64_t n, int64_t cb,
                          int64_t h, int64_t w, int x, int win, int stride, int pad, int flags,
                          neo_stream_t stream) {
  return neo_pool2d_window(dtype, mode, in, out, n, cb, h, w, x, win, stride, pad, 0, cb, 0, cb,
                           flags, stream);
}

extern "C" int neo_eltwise_window(int dtype, int op, const void* a, const void* b, void* out,
                                  const float* scale, const float* shift, int64_t n, int64_t cb,
                                  int64_t hw, int x, int64_t a_cb_off, int64_t a_cb_total,
                                  int64_t out_cb_off, int64_t out_cb_total, int flags,
                                  neo_stream_t stream) {
  NEO_CHECK_ARG(a && out, NEO_ERR_INVALID_ARG, "null tensor pointer");
  NEO_CHECK_ARG(op >= 0 && op <= 4, NEO_ERR_INVALID_ARG, "bad eltwise op %d", op);
  NEO_CHECK_ARG(!(op == NEO_ELT_ADD || op == NEO_ELT_ADD_RELU) || b, NEO_ERR_INVALID_ARG,
                "add needs two inputs");
  NEO_CHECK_ARG(op < NEO_ELT_SCALE_SHIFT || (scale && shift), NEO_ERR_INVALID_ARG,
                "scale/shift needs both vectors");
  NEO_CHECK_ARG(!(op == NEO_ELT_ADD || op == NEO_ELT_ADD_RELU) ||
                    (a_cb_off == 0 && a_cb_total == cb && out_cb_off == 0 && out_cb_total == cb),
                NEO_ERR_UNSUPPORTED, "windowed add is not supported");
  NEO_CHECK_ARG(a_cb_off >= 0 && a_cb_off + cb <= a_cb_total && out_cb_off >= 0 &&
                    out_cb_off + cb <= out_cb_total,
                NEO_ERR_SHAPE_MISMATCH, "channel-block window out of range");
  const int64_t total = n * cb * hw * x;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool round = (flags & NEO_FLAG_ROUND_TF32) != 0;
  const Win wnd{a_cb_off, a_cb_total, out_cb_off, out_cb_total};
  const int64_t P = n * cb, plane_sz = hw * x;
  const bool al = aligned16(a) && aligned16(out) && (!b || aligned16(b)) &&
                  (op < NEO_ELT_SCALE_SHIFT || (aligned16(scale) && aligned16(shift)));
  const bool flat_ok = (uint64_t)P * (uint64_t)plane_sz < (1ull << 32);
  if (dtype == NEO_BF16 && x % 8 == 0 && al && flat_ok) {
    const uint32_t vecs = (uint32_t)(plane_sz / 8), tot = (uint32_t)(P * vecs);
    neo_launch(eltwise_flat_vec<__nv_bfloat16, 8, 4>, flat_grid(tot, 4), 256, 0, st,
        static_cast<const __nv_bfloat16*>(a), static_cast<const __nv_bfloat16*>(b),
        static_cast<__nv_bfloat16*>(out), scale, shift, cb, tot, vecs, plane_sz, x, op, round, wnd);
  } else if (dtype == NEO_F32 && x % 4 == 0 && al && flat_ok) {
    const uint32_t vecs = (uint32_t)(plane_sz / 4), tot = (uint32_t)(P * vecs);
    neo_launch(eltwise_flat_vec<float, 4, 4>, flat_grid(tot, 4), 256, 0, st,
        static_cast<const float*>(a), static_cast<const float*>(b), static_cast<float*>(out),
        scale, shift, cb, tot, vecs, plane_sz, x, op, round, wnd);
  } else if (dtype == NEO_BF16)
    neo_launch(eltwise_kernel<__nv_bfloat16>, (unsigned)grid_for(total), 256, 0, st, 
        static_cast<const __nv_bfloat16*>(a), static_cast<const __nv_bfloat16*>(b),
        static_cast<__nv_bfloat16*>(out), scale, shift, total, cb, hw, x, op, round, wnd);
  else
    neo_launch(eltwise_kernel<float>, (unsigned)grid_for(total), 256, 0, st, 
        static_cast<const float*>(a), static_cast<const float*>(b), static_cast<float*>(out), scale,
        shift, total, cb, hw, x, op, round, wnd);
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}

extern "C" int neo_eltwise(int dtype, int op, const void* a, const void* b, void* out,
                           const float* scale, const float* shift, int64_t n, int64_t cb,
                           int64_t hw, int x, int flags, neo_stream_t stream) {
  return neo_eltwise_window(dtype, op, a, b, out, scale, shift, n, cb, hw, x, 0, cb, 0, cb, flags,
                            stream);
}

extern "C" int neo_concat_copy(int dtype, const void* src, void* dst, int64_t outer, int64_t chunk,
                               int64_t dst_row, int64_t dst_off, neo_stream_t stream) {
  NEO_CHECK_ARG(src && dst, NEO_ERR_INVALID_ARG, "null tensor pointer");
  NEO_CHECK_ARG(outer >= 0 && chunk >= 0 && dst_off + chunk <= dst_row, NEO_ERR_SHAPE_MISMATCH,
                "concat slice out of range");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t es = neo_dtype_size(dtype);
  const int64_t per = 16 / es;
  if (outer * chunk == 0) return NEO_OK;
  if (chunk % per == 0 && dst_row % per == 0 && dst_off % per == 0 &&
      ((uintptr_t)src & 15) == 0 && ((uintptr_t)dst & 15) == 0) {
    const int64_t total = outer * (chunk / per);
    neo_launch(concat_kernel_v4, (unsigned)grid_for(total), 256, 0, st, 
        static_cast<const uint4*>(src), static_cast<uint4*>(dst), outer, chunk / per,
        dst_row / per, dst_off / per);
  } else if (es == 1) {
    neo_launch(concat_kernel<uint8_t>, (unsigned)grid_for(outer * chunk), 256, 0, st,
        static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), outer, chunk, dst_row,
        dst_off);
  } else if (es == 2) {
    neo_launch(concat_kernel<uint16_t>, (unsigned)grid_for(outer * chunk), 256, 0, st, 
        static_cast<const uint16_t*>(src), static_cast<uint16_t*>(dst), outer, chunk, dst_row,
        dst_off);
  } else {
    neo_launch(concat_kernel<uint32_t>, (unsigned)grid_for(outer * chunk), 256, 0, st, 
        static_cast<const uint32_t*>(src), static_cast<uint32_t*>(dst), outer, chunk, dst_row,
        dst_off);
  }
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}

extern "C" int neo_dense(int dtype, const void* a, const void* w, const float* bias, float* out,
                         int64_t n, int64_t in_features, int64_t units, neo_stream_t stream) {
  NEO_CHECK_ARG(a && w && out, NEO_ERR_INVALID_ARG, "null tensor pointer");
  NEO_CHECK_ARG(n >= 1 && in_features >= 1 && units >= 1, NEO_ERR_SHAPE_MISMATCH, "bad dense dims");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  constexpr int NB = 8;
  const int threads = 256;
  dim3 grid((unsigned)neo_ceil_div(units, threads / 32),
            (unsigned)std::min<int64_t>(neo_ceil_div(n, NB), 65535));
  if (dtype == NEO_BF16)
    neo_launch(dense_kernel<__nv_bfloat16, NB>, grid, threads, 0, st, 
        static_cast<const __nv_bfloat16*>(a), static_cast<const __nv_bfloat16*>(w), bias, out, n,
        in_features, units);
  else
    neo_launch(dense_kernel<float, NB>, grid, threads, 0, st, static_cast<const float*>(a),
                                                      static_cast<const float*>(w), bias, out, n,
                                                      in_features, units);
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}

extern "C" int neo_softmax(const float* in, float* out, int64_t rows, int64_t cols,
                           neo_stream_t stream) {
  NEO_CHECK_ARG(in && out, NEO_ERR_INVALID_ARG, "null tensor pointer");
  NEO_CHECK_ARG(rows >= 1 && cols >= 1, NEO_ERR_SHAPE_MISMATCH, "bad softmax dims");
  neo_launch(softmax_kernel, (unsigned)std::min<int64_t>(rows, 148 * 8), 256, 0,
                   static_cast<cudaStream_t>(stream), in, out, rows, cols);
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}
