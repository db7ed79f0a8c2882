// K-LAYOUT / K-WPACK: bit-exact layout transforms between NCHW, NHWC and
// NCHW[x]c feature maps and between KCRS and KCRS[x]c[y]k weights
// (reference layout.py:131-235), plus the device-private slice-major weight
// image consumed by the tensor-core conv.
//
// Pack / unpack / NHWC ingest are batched 2-D transposes staged through a
// 32x33 shared-memory tile so both the read and the write side are coalesced;
// retile and the weight permutations are gathers (compile time / rare).
#include "neo_common.cuh"

namespace {

template <typename T>
__device__ __forceinline__ float ld_as_f(const T* p, int64_t i) {
  return Elem<T>::to_f(p[i]);
}

// bit-preserving element move with optional dtype conversion / tf32 rounding
template <typename Ts, typename Td>
struct Conv {
  static __device__ __forceinline__ Td cvt(Ts v, bool) { return Elem<Td>::from_f(Elem<Ts>::to_f(v)); }
};
template <>
struct Conv<float, float> {
  static __device__ __forceinline__ float cvt(float v, bool round) {
    return round ? neo_round_tf32(v) : v;
  }
};
template <>
struct Conv<__nv_bfloat16, __nv_bfloat16> {
  static __device__ __forceinline__ __nv_bfloat16 cvt(__nv_bfloat16 v, bool) { return v; }
};

// Batched transpose: for each batch b, src viewed (R rows x C cols) is written
// to dst viewed (C rows x R cols).  Index maps are supplied by Map.
struct PackMap {  // NCHW -> NCHW[x]c; b = (n, cb); rows = lanes j, cols = pixels
  int64_t Call, HW, Cb;
  int x;
  __device__ bool src(int64_t b, int64_t r, int64_t c, int64_t& off) const {
    const int64_t n = b / Cb, cb = b % Cb, ch = cb * x + r;
    off = (n * Call + ch) * HW + c;
    return ch < Call;
  }
  __device__ bool dst(int64_t b, int64_t c, int64_t r, int64_t& off) const {
    off = (b * HW + c) * x + r;
    return true;
  }
};
struct UnpackMap {  // NCHW[x]c -> NCHW; b = (n, cb); rows = pixels, cols = lanes
  int64_t Call, HW, Cb;
  int x;
  __device__ bool src(int64_t b, int64_t r, int64_t c, int64_t& off) const {
    off = (b * HW + r) * x + c;
    return true;
  }
  __device__ bool dst(int64_t b, int64_t c, int64_t r, int64_t& off) const {
    const int64_t n = b / Cb, cb = b % Cb, ch = cb * x + c;
    off = (n * Call + ch) * HW + r;
    return ch < Call;
  }
};
struct NhwcMap {  // NHWC -> NCHW; b = n; rows = pixels, cols = channels
  int64_t Call, HW;
  __device__ bool src(int64_t b, int64_t r, int64_t c, int64_t& off) const {
    off = (b * HW + r) * Call + c;
    return true;
  }
  __device__ bool dst(int64_t b, int64_t c, int64_t r, int64_t& off) const {
    off = (b * Call + c) * HW + r;
    return true;
  }
};

template <typename Ts, typename Td, class Map>
__global__ void transpose_kernel(const Ts* __restrict__ src, Td* __restrict__ dst, Map m,
                                 int64_t B, int64_t R, int64_t C, bool round) {
  neo_pdl_enter();
  __shared__ Ts tile[32][33];
  __shared__ bool ok[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int64_t b = blockIdx.z; b < B; b += gridDim.z) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t r = r0 + ty + 8 * i, c = c0 + tx;
      int64_t off = 0;
      bool v = r < R && c < C && m.src(b, r, c, off);
      tile[ty + 8 * i][tx] = v ? src[off] : Elem<Ts>::from_f(0.f);
      ok[ty + 8 * i][tx] = r < R && c < C;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t c = c0 + ty + 8 * i, r = r0 + tx;
      int64_t off = 0;
      if (ok[tx][ty + 8 * i] && m.dst(b, c, r, off))
        dst[off] = Conv<Ts, Td>::cvt(tile[tx][ty + 8 * i], round);
    }
    __syncthreads();
  }
}

template <typename Ts, typename Td, class Map>
void launch_transpose(const void* src, void* dst, Map m, int64_t B, int64_t R, int64_t C,
                      bool round, cudaStream_t st) {
  dim3 block(32, 8);
  dim3 grid((unsigned)neo_ceil_div(C, 32), (unsigned)neo_ceil_div(R, 32),
            (unsigned)std::min<int64_t>(B, 65535));
  neo_launch(transpose_kernel<Ts, Td, Map>, grid, block, 0, st, static_cast<const Ts*>(src),
                                                        static_cast<Td*>(dst), m, B, R, C, round);
}

// NCHW[a]c -> NCHW[b]c (retile_nchw_array layout.py:163-177), also same-layout
// copies/conversions (a == b, or NCHW as a = 1)
template <typename Ts, typename Td>
__global__ void retile_kernel(const Ts* __restrict__ src, Td* __restrict__ dst, int64_t N,
                              int64_t Call, int64_t HW, int a, int b, bool round) {
  neo_pdl_enter();
  const int64_t cbd = (Call + b - 1) / b, cbs = (Call + a - 1) / a;
  const int64_t total = N * cbd * HW * b;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int j = (int)(t % b);
    t /= b;
    const int64_t p = t % HW;
    t /= HW;
    const int64_t cb = t % cbd;
    const int64_t n = t / cbd;
    const int64_t ch = cb * b + j;
    if (ch < Call) {
      const int64_t so = ((n * cbs + ch / a) * HW + p) * a + ch % a;
      dst[i] = Conv<Ts, Td>::cvt(src[so], round);
    } else {
      dst[i] = Elem<Td>::from_f(0.f);
    }
  }
}

// NCHW -> NCHW[x]c for small x (x*sizeof(dst) <= 64 B, e.g. the 3-channel
// image into 8 padded bf16 lanes): one thread per (n, cb, pixel) gathers its
// x channels (coalesced across threads) and writes them as one contiguous row.
template <typename Ts, typename Td, int X>
__global__ void pack_small_kernel(const Ts* __restrict__ src, Td* __restrict__ dst, int64_t N,
                                  int64_t Call, int64_t HW, bool round) {
  neo_pdl_enter();
  const int64_t Cb = (Call + X - 1) / X;
  const int64_t total = N * Cb * HW;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i % HW;
    const int64_t b = i / HW;
    const int64_t n = b / Cb, cb = b % Cb;
    Td row[X];
#pragma unroll
    for (int j = 0; j < X; ++j) {
      const int64_t ch = cb * X + j;
      row[j] = ch < Call ? Conv<Ts, Td>::cvt(src[(n * Call + ch) * HW + p], round)
                         : Elem<Td>::from_f(0.f);
    }
    constexpr int kVec = (int)(X * sizeof(Td) / 16);
    if constexpr (kVec >= 1) {
      const uint4* r4 = reinterpret_cast<const uint4*>(row);
      uint4* d4 = reinterpret_cast<uint4*>(dst + i * X);
#pragma unroll
      for (int v = 0; v < kVec; ++v) d4[v] = r4[v];
    } else {
#pragma unroll
      for (int j = 0; j < X; ++j) dst[i * X + j] = row[j];
    }
  }
}

template <typename Ts, typename Td>
bool try_pack_small(const void* src, void* dst, int64_t n, int64_t c, int64_t hw, int x,
                    bool round, cudaStream_t st) {
  const int64_t total = n * ((c + x - 1) / x) * hw;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 32));
  auto s = static_cast<const Ts*>(src);
  auto d = static_cast<Td*>(dst);
  switch (x) {
    case 4: neo_launch(pack_small_kernel<Ts, Td, 4>, grid, 256, 0, st, s, d, n, c, hw, round); return true;
    case 8: neo_launch(pack_small_kernel<Ts, Td, 8>, grid, 256, 0, st, s, d, n, c, hw, round); return true;
    case 16: neo_launch(pack_small_kernel<Ts, Td, 16>, grid, 256, 0, st, s, d, n, c, hw, round); return true;
    default: return false;
  }
}

template <typename Ts, typename Td>
int dispatch_layout(const void* src, void* dst, int64_t n, int64_t c, int64_t h, int64_t w,
                    int src_tag, int src_x, int dst_tag, int dst_x, bool round, cudaStream_t st) {
  const int64_t HW = h * w;
  if (src_tag == NEO_NCHW && dst_tag == NEO_NCHWC && dst_x <= 16 &&
      try_pack_small<Ts, Td>(src, dst, n, c, HW, dst_x, round, st)) {
    // small block: per-pixel gather kernel
  } else if (src_tag == NEO_NCHW && dst_tag == NEO_NCHWC) {
    const int64_t cb = neo_ceil_div(c, dst_x);
    launch_transpose<Ts, Td>(src, dst, PackMap{c, HW, cb, dst_x}, n * cb, dst_x, HW, round, st);
  } else if (src_tag == NEO_NCHWC && dst_tag == NEO_NCHW) {
    const int64_t cb = neo_ceil_div(c, src_x);
    launch_transpose<Ts, Td>(src, dst, UnpackMap{c, HW, cb, src_x}, n * cb, HW, src_x, round, st);
  } else if (src_tag == NEO_NHWC && dst_tag == NEO_NCHW) {
    launch_transpose<Ts, Td>(src, dst, NhwcMap{c, HW}, n, HW, c, round, st);
  } else {
    // NCHW[a]c -> NCHW[b]c, NCHW -> NCHW (a = b = 1)
    const int a = src_tag == NEO_NCHW ? 1 : src_x;
    const int b = dst_tag == NEO_NCHW ? 1 : dst_x;
    const int64_t total = n * neo_ceil_div(c, b) * HW * b;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(neo_ceil_div(total, 256), 148 * 32));
    neo_launch(retile_kernel<Ts, Td>, (unsigned)blocks, 256, 0, st, static_cast<const Ts*>(src),
                                                            static_cast<Td*>(dst), n, c, HW, a, b,
                                                            round);
  }
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}

// KCRS -> KCRS[x]c[y]k and back (pack_kcrs_array :147, unpack_kcrs_array :156);
// 32-bit / 16-bit payloads moved as raw bits
template <typename T>
__global__ void weights_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t K, int64_t C,
                               int64_t RS, int x, int y, bool pack) {
  neo_pdl_enter();
  const int64_t total = K * C * RS;
  const int64_t Cb = C / x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    // i enumerates the packed layout (ko, co, rs, ci, kj)
    int64_t t = i;
    const int kj = (int)(t % y);
    t /= y;
    const int ci = (int)(t % x);
    t /= x;
    const int64_t rs = t % RS;
    t /= RS;
    const int64_t co = t % Cb;
    const int64_t ko = t / Cb;
    const int64_t plain = ((ko * y + kj) * C + co * x + ci) * RS + rs;
    if (pack) dst[i] = src[plain];
    else dst[plain] = src[i];
  }
}

template <typename Td>
__global__ void weights_umma_kernel(const float* __restrict__ src, Td* __restrict__ dst, int64_t K,
                                    int64_t C, int64_t R, int64_t S, int x, int64_t slices,
                                    int64_t nslices, bool round) {
  neo_pdl_enter();
  const int64_t Cb = (C + x - 1) / x;
  const int64_t total = slices * K * x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int j = (int)(t % x);
    t /= x;
    const int64_t k = t % K;
    const int64_t sl = t / K;
    float v = 0.f;
    if (sl < nslices) {
      const int64_t cb = sl % Cb, rs = sl / Cb;
      const int64_t s = rs % S, r = rs / S;
      const int64_t ch = cb * x + j;
      if (ch < C) v = src[((k * C + ch) * R + r) * S + s];
    }
    if constexpr (sizeof(Td) == 4) dst[i] = round ? neo_round_tf32(v) : v;
    else dst[i] = Elem<Td>::from_f(v);
  }
}

// e4m3 weight image (NEO_MODE_FP8): the slice-major layout of
// weights_umma_kernel, value src / wscale[k] rounded RN (satfinite) to e4m3
__global__ void weights_umma_fp8_kernel(const float* __restrict__ src, uint8_t* __restrict__ dst,
                                        const float* __restrict__ wscale, int64_t K, int64_t C,
                                        int64_t R, int64_t S, int x, int64_t slices,
                                        int64_t nslices) {
  neo_pdl_enter();
  const int64_t Cb = (C + x - 1) / x;
  const int64_t total = slices * K * x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int j = (int)(t % x);
    t /= x;
    const int64_t k = t % K;
    const int64_t sl = t / K;
    float v = 0.f;
    if (sl < nslices) {
      const int64_t cb = sl % Cb, rs = sl / Cb;
      const int64_t s = rs % S, r = rs / S;
      const int64_t ch = cb * x + j;
      if (ch < C) v = __fdiv_rn(src[((k * C + ch) * R + r) * S + s], wscale[k]);
    }
    dst[i] = (uint8_t)__nv_cvt_float_to_fp8(v, __NV_SATFINITE, __NV_E4M3);
  }
}

// max |x|: grid-stride partial maxima, one atomicMax per warp on the float
// bits (non-negative floats order like their bit patterns)
template <int DT>
__global__ void absmax_kernel(const void* __restrict__ x, int64_t n, float* __restrict__ out) {
  neo_pdl_enter();
  float m = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v;
    if constexpr (DT == NEO_F32) v = static_cast<const float*>(x)[i];
    else if constexpr (DT == NEO_BF16) v = __bfloat162float(static_cast<const __nv_bfloat16*>(x)[i]);
    else v = __half2float(__half(__nv_cvt_fp8_to_halfraw(static_cast<const uint8_t*>(x)[i], __NV_E4M3)));
    m = fmaxf(m, fabsf(v));
  }
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<unsigned int*>(out), __float_as_uint(m));
}

int64_t grid_for(int64_t total) {
  return std::max<int64_t>(1, std::min<int64_t>(neo_ceil_div(total, 256), 148 * 32));
}

}  // namespace

extern "C" int neo_layout_transform(int src_dtype, int dst_dtype, const void* src, void* dst,
                                    int64_t n, int64_t c, int64_t h, int64_t w, int src_tag,
                                    int src_x, int dst_tag, int dst_x, int flags,
                                    neo_stream_t stream) {
  NEO_CHECK_ARG(src && dst, NEO_ERR_INVALID_ARG, "null tensor pointer");
  NEO_CHECK_ARG(n >= 1 && c >= 1 && h >= 1 && w >= 1, NEO_ERR_SHAPE_MISMATCH,
                "non-positive dim in (%lld,%lld,%lld,%lld)", (long long)n, (long long)c,
                (long long)h, (long long)w);
  NEO_CHECK_ARG((src_dtype == NEO_F32 || src_dtype == NEO_BF16) &&
                    (dst_dtype == NEO_F32 || dst_dtype == NEO_BF16),
                NEO_ERR_INVALID_ARG, "bad dtype");
  NEO_CHECK_ARG(src_tag >= 0 && src_tag <= 2 && dst_tag >= 0 && dst_tag <= 2, NEO_ERR_WRONG_LAYOUT,
                "unknown layout tag");
  NEO_CHECK_ARG(dst_tag != NEO_NHWC, NEO_ERR_WRONG_LAYOUT, "no transform to NHWC");
  NEO_CHECK_ARG(src_tag != NEO_NHWC || dst_tag == NEO_NCHW, NEO_ERR_WRONG_LAYOUT,
                "NHWC is only ingested into NCHW");
  const bool padc = (flags & NEO_FLAG_PAD_CHANNELS) != 0;
  if (src_tag == NEO_NCHWC) {
    NEO_CHECK_ARG(src_x >= 1, NEO_ERR_WRONG_LAYOUT, "NCHW[x]c needs x >= 1");
    NEO_CHECK_ARG(padc || c % src_x == 0, NEO_ERR_INDIVISIBLE_CHANNEL,
                  "C=%lld not divisible by x=%d", (long long)c, src_x);
  }
  if (dst_tag == NEO_NCHWC) {
    NEO_CHECK_ARG(dst_x >= 1, NEO_ERR_WRONG_LAYOUT, "NCHW[x]c needs x >= 1");
    NEO_CHECK_ARG(padc || c % dst_x == 0, NEO_ERR_INDIVISIBLE_CHANNEL,
                  "C=%lld not divisible by x=%d", (long long)c, dst_x);
  }
  const bool round = (flags & NEO_FLAG_ROUND_TF32) != 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (src_dtype == NEO_F32 && dst_dtype == NEO_F32)
    return dispatch_layout<float, float>(src, dst, n, c, h, w, src_tag, src_x, dst_tag, dst_x, round, st);
  if (src_dtype == NEO_F32 && dst_dtype == NEO_BF16)
    return dispatch_layout<float, __nv_bfloat16>(src, dst, n, c, h, w, src_tag, src_x, dst_tag, dst_x, round, st);
  if (src_dtype == NEO_BF16 && dst_dtype == NEO_F32)
    return dispatch_layout<__nv_bfloat16, float>(src, dst, n, c, h, w, src_tag, src_x, dst_tag, dst_x, round, st);
  return dispatch_layout<__nv_bfloat16, __nv_bfloat16>(src, dst, n, c, h, w, src_tag, src_x, dst_tag, dst_x, round, st);
}

static int weights_common(int dtype, const void* src, void* dst, int64_t k, int64_t c, int64_t r,
                          int64_t s, int x, int y, bool pack, cudaStream_t st) {
  NEO_CHECK_ARG(src && dst, NEO_ERR_INVALID_ARG, "null tensor pointer");
  NEO_CHECK_ARG(k >= 1 && c >= 1 && r >= 1 && s >= 1, NEO_ERR_SHAPE_MISMATCH, "non-positive dim");
  NEO_CHECK_ARG(x >= 1 && y >= 1, NEO_ERR_WRONG_LAYOUT, "KCRS[x]c[y]k needs x >= 1 and y >= 1");
  NEO_CHECK_ARG(c % x == 0 && k % y == 0, NEO_ERR_INDIVISIBLE_CHANNEL,
                "(K=%lld, C=%lld) not divisible by (y=%d, x=%d)", (long long)k, (long long)c, y, x);
  const int64_t total = k * c * r * s;
  if (dtype == NEO_BF16)
    neo_launch(weights_kernel<uint16_t>, (unsigned)grid_for(total), 256, 0, st, 
        static_cast<const uint16_t*>(src), static_cast<uint16_t*>(dst), k, c, r * s, x, y, pack);
  else
    neo_launch(weights_kernel<uint32_t>, (unsigned)grid_for(total), 256, 0, st, 
        static_cast<const uint32_t*>(src), static_cast<uint32_t*>(dst), k, c, r * s, x, y, pack);
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}

extern "C" int neo_pack_weights(int dtype, const void* src, void* dst, int64_t k, int64_t c,
                                int64_t r, int64_t s, int x, int y, neo_stream_t stream) {
  return weights_common(dtype, src, dst, k, c, r, s, x, y, true, static_cast<cudaStream_t>(stream));
}

extern "C" int neo_unpack_weights(int dtype, const void* src, void* dst, int64_t k, int64_t c,
                                  int64_t r, int64_t s, int x, int y, neo_stream_t stream) {
  return weights_common(dtype, src, dst, k, c, r, s, x, y, false, static_cast<cudaStream_t>(stream));
}

extern "C" int neo_pack_weights_umma(const float* src_kcrs, void* dst, int dst_dtype, int64_t k,
                                     int64_t c, int64_t r, int64_t s, int x,
                                     int64_t slices_padded, int flags, neo_stream_t stream) {
  NEO_CHECK_ARG(src_kcrs && dst, NEO_ERR_INVALID_ARG, "null tensor pointer");
  NEO_CHECK_ARG(k >= 1 && c >= 1 && r >= 1 && s >= 1 && x >= 1, NEO_ERR_SHAPE_MISMATCH,
                "non-positive dim");
  const int64_t nslices = r * s * neo_ceil_div(c, x);
  NEO_CHECK_ARG((flags & NEO_FLAG_PAD_CHANNELS) || c % x == 0, NEO_ERR_INDIVISIBLE_CHANNEL,
                "C=%lld not divisible by x=%d", (long long)c, x);
  if (slices_padded < nslices) slices_padded = nslices;
  const int64_t total = slices_padded * k * x;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool round = (flags & NEO_FLAG_ROUND_TF32) != 0;
  if (dst_dtype == NEO_BF16)
    neo_launch(weights_umma_kernel<__nv_bfloat16>, (unsigned)grid_for(total), 256, 0, st, 
        src_kcrs, static_cast<__nv_bfloat16*>(dst), k, c, r, s, x, slices_padded, nslices, round);
  else
    neo_launch(weights_umma_kernel<float>, (unsigned)grid_for(total), 256, 0, st, 
        src_kcrs, static_cast<float*>(dst), k, c, r, s, x, slices_padded, nslices, round);
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}

extern "C" int neo_pack_weights_umma_fp8(const float* src_kcrs, void* dst, const float* wscale,
                                         int64_t k, int64_t c, int64_t r, int64_t s, int x,
                                         int64_t slices_padded, int flags, neo_stream_t stream) {
  NEO_CHECK_ARG(src_kcrs && dst && wscale, NEO_ERR_INVALID_ARG, "null tensor pointer");
  NEO_CHECK_ARG(k >= 1 && c >= 1 && r >= 1 && s >= 1 && x >= 1, NEO_ERR_SHAPE_MISMATCH,
                "non-positive dim");
  const int64_t nslices = r * s * neo_ceil_div(c, x);
  NEO_CHECK_ARG((flags & NEO_FLAG_PAD_CHANNELS) || c % x == 0, NEO_ERR_INDIVISIBLE_CHANNEL,
                "C=%lld not divisible by x=%d", (long long)c, x);
  if (slices_padded < nslices) slices_padded = nslices;
  const int64_t total = slices_padded * k * x;
  neo_launch(weights_umma_fp8_kernel, (unsigned)grid_for(total), 256, 0,
             static_cast<cudaStream_t>(stream), src_kcrs, static_cast<uint8_t*>(dst), wscale, k,
             c, r, s, x, slices_padded, nslices);
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}

// e4m3 NCHW[x]c (scale) -> NCHW f32 / bf16: value = e4m3(q) * scale (the
// FP8 mode's exit from the blocked chain, e.g. into a classifier)
template <typename Td>
__global__ void dequant_fp8_kernel(const uint8_t* __restrict__ src, Td* __restrict__ dst,
                                   float scale, int64_t N, int64_t C, int64_t HW, int x,
                                   int64_t cb_off, int64_t cb_total) {
  neo_pdl_enter();
  const int64_t total = N * C * HW;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i % HW;
    const int64_t c = (i / HW) % C;
    const int64_t n = i / (HW * C);
    const uint8_t q = src[((n * cb_total + cb_off + c / x) * HW + p) * x + c % x];
    const float v = __half2float(__half(__nv_cvt_fp8_to_halfraw(q, __NV_E4M3))) * scale;
    dst[i] = Elem<Td>::from_f(v);
  }
}

extern "C" int neo_dequant_fp8(const void* src, void* dst, int dst_dtype, float scale, int64_t n,
                               int64_t c, int64_t h, int64_t w, int x, int64_t cb_off,
                               int64_t cb_total, neo_stream_t stream) {
  NEO_CHECK_ARG(src && dst && scale > 0.f, NEO_ERR_INVALID_ARG, "bad dequant arguments");
  NEO_CHECK_ARG(x >= 1 && c % x == 0, NEO_ERR_INDIVISIBLE_CHANNEL, "C=%lld not divisible by x=%d",
                (long long)c, x);
  if (cb_total <= 0) cb_total = c / x;
  const int64_t total = n * c * h * w;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dst_dtype == NEO_BF16)
    neo_launch(dequant_fp8_kernel<__nv_bfloat16>, (unsigned)grid_for(total), 256, 0, st,
               static_cast<const uint8_t*>(src), static_cast<__nv_bfloat16*>(dst), scale, n, c,
               h * w, x, cb_off, cb_total);
  else if (dst_dtype == NEO_F32)
    neo_launch(dequant_fp8_kernel<float>, (unsigned)grid_for(total), 256, 0, st,
               static_cast<const uint8_t*>(src), static_cast<float*>(dst), scale, n, c, h * w, x,
               cb_off, cb_total);
  else {
    neo_set_error("dequant writes f32 or bf16");
    return NEO_ERR_INVALID_ARG;
  }
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}

extern "C" int neo_absmax(int dtype, const void* x, int64_t n, float* out, neo_stream_t stream) {
  NEO_CHECK_ARG(x && out && n >= 0, NEO_ERR_INVALID_ARG, "bad absmax arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  NEO_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(float), st));
  if (n == 0) return NEO_OK;
  const unsigned grid = (unsigned)grid_for(n);
  switch (dtype) {
    case NEO_F32: neo_launch(absmax_kernel<NEO_F32>, grid, 256, 0, st, x, n, out); break;
    case NEO_BF16: neo_launch(absmax_kernel<NEO_BF16>, grid, 256, 0, st, x, n, out); break;
    case NEO_FP8: neo_launch(absmax_kernel<NEO_FP8>, grid, 256, 0, st, x, n, out); break;
    default: neo_set_error("bad dtype %d", dtype); return NEO_ERR_INVALID_ARG;
  }
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}

// ---------------------------------------------------------------------------
// Stem folding (B200 lowering of a small-channel graph-entry conv input):
// X'[n, cb, h, w', j] with folded channel f = cb*xf + j = s*C + c holds
// X[n, c, h, sw*w' + s - pw] (0 outside the image or for pad lanes), for
// w' in [0, ow).  A conv with an S-wide kernel, stride sw and pad pw over X
// equals a conv with an S=1 kernel, stride 1 and pad 0 along w over X' with
// weights W'[k, s*C + c, r, 0] = W[k, c, r, s]: the horizontal taps become
// input channels, so a 3-channel 7x7/2 stem reads 21 (of 32) useful lanes
// instead of 3 (of 8) and the tensor cores see 64-byte rows.
namespace {
template <typename Td, int XF>
__global__ void stem_fold_kernel(const float* __restrict__ src, Td* __restrict__ dst, int64_t N,
                                 int C, int H, int W, int S, int sw, int pw, int OW, bool round) {
  neo_pdl_enter();
  const int F = S * C;
  const int Cb = (F + XF - 1) / XF;
  const int64_t total = N * Cb * H * (int64_t)OW;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int wq = (int)(i % OW);
    const int64_t rest = i / OW;
    const int h = (int)(rest % H);
    const int64_t ncb = rest / H;
    const int cb = (int)(ncb % Cb);
    const int64_t n = ncb / Cb;
    float vals[XF];
#pragma unroll
    for (int j = 0; j < XF; ++j) vals[j] = 0.f;
    const float* plane = src + (n * C) * (int64_t)H * W + (int64_t)h * W;
    const int iw0 = sw * wq - pw;
    // folded channel f = s*C + c, lanes [cb*XF, cb*XF + XF)
    int f = cb * XF;
    int s = f / C, c = f % C;
#pragma unroll
    for (int j = 0; j < XF; ++j) {
      if (s < S) {
        const int iw = iw0 + s;
        if (iw >= 0 && iw < W) vals[j] = __ldg(plane + (int64_t)c * H * W + iw);
      }
      if (++c == C) {
        c = 0;
        ++s;
      }
    }
    Td row[XF];
#pragma unroll
    for (int j = 0; j < XF; ++j) {
      if constexpr (sizeof(Td) == 4) row[j] = round ? neo_round_tf32(vals[j]) : vals[j];
      else row[j] = Elem<Td>::from_f(vals[j]);
    }
    constexpr int kVec = (int)(XF * sizeof(Td) / 16);
    uint4* d4 = reinterpret_cast<uint4*>(dst + i * XF);
    const uint4* r4 = reinterpret_cast<const uint4*>(row);
#pragma unroll
    for (int v = 0; v < kVec; ++v) d4[v] = r4[v];
  }
}

// Row-tiled fold: one CTA per (n, h) input row (many small CTAs per SM hide
// the load latency); the C input rows are staged in shared memory with
// coalesced 16-byte loads, then every thread builds 16-byte pieces of the
// folded output row (consecutive threads -> consecutive pieces: coalesced
// stores).  CC = C (compile-time: no divisions).  Same values as
// stem_fold_kernel.
template <typename Td, int XF, int CC>
__global__ void stem_fold_rows_kernel(const float* __restrict__ src, Td* __restrict__ dst,
                                      int H, int W, int S, int sw, int pw, int OW, bool round) {
  extern __shared__ float rows[];   // CC x W
  neo_pdl_enter();
  constexpr int kLanes = 16 / (int)sizeof(Td);   // lanes per 16-byte piece
  constexpr int kPieces = XF / kLanes;
  const int F = S * CC;
  const int Cb = (F + XF - 1) / XF;
  const int64_t row = blockIdx.x;
  const int64_t n = row / H;
  const int h = (int)(row - n * H);
#pragma unroll
  for (int c = 0; c < CC; ++c) {
    const float* plane = src + ((n * CC + c) * H + h) * (int64_t)W;
    if ((W & 3) == 0) {
      for (int i = threadIdx.x; i < W / 4; i += blockDim.x)
        reinterpret_cast<float4*>(rows + c * W)[i] = __ldg(reinterpret_cast<const float4*>(plane) + i);
    } else {
      for (int i = threadIdx.x; i < W; i += blockDim.x) rows[c * W + i] = __ldg(plane + i);
    }
  }
  __syncthreads();
  const int per_cb = OW * kPieces;
  for (int it = threadIdx.x; it < Cb * per_cb; it += blockDim.x) {
    const int cb = it / per_cb;
    const int rem = it - cb * per_cb;
    const int wq = rem / kPieces, pc = rem - wq * kPieces;
    const int iw0 = sw * wq - pw;
    Td vals[kLanes];
#pragma unroll
    for (int j = 0; j < kLanes; ++j) {
      const int f = cb * XF + pc * kLanes + j;   // folded channel = s*CC + c
      const int ss = f / CC, c = f - ss * CC;
      const int iw = iw0 + ss;
      float v = 0.f;
      if (f < F && iw >= 0 && iw < W) v = rows[c * W + iw];
      if constexpr (sizeof(Td) == 4) vals[j] = round ? neo_round_tf32(v) : v;
      else vals[j] = Elem<Td>::from_f(v);
    }
    Td* out = dst + (((n * Cb + cb) * H + h) * (int64_t)OW + wq) * XF + pc * kLanes;
    *reinterpret_cast<uint4*>(out) = *reinterpret_cast<const uint4*>(vals);
  }
}
}  // namespace

extern "C" int neo_stem_fold(const float* src, void* dst, int dst_dtype, int64_t n, int64_t c,
                             int64_t h, int64_t w, int s, int stride_w, int pad_w, int64_t ow,
                             int xf, int flags, neo_stream_t stream) {
  NEO_CHECK_ARG(src && dst, NEO_ERR_INVALID_ARG, "null tensor pointer");
  NEO_CHECK_ARG(n >= 1 && c >= 1 && h >= 1 && w >= 1 && s >= 1 && ow >= 1 && stride_w >= 1,
                NEO_ERR_SHAPE_MISMATCH, "bad stem fold geometry");
  const int64_t total = n * neo_ceil_div(s * c, xf) * h * ow;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(neo_ceil_div(total, 256), 148 * 32));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool round = (flags & NEO_FLAG_ROUND_TF32) != 0;
  // row-tiled kernel when the C input rows fit in shared memory
  const size_t row_smem = (size_t)c * w * sizeof(float);
  const bool rows_ok = row_smem <= 48 * 1024 && c <= 4 && n * h < (1ll << 31) &&
                       !getenv("NEOB200_FOLD_PIXEL");
#define NEO_FOLD_ROWS(T, X, CC)                                                               \
  neo_launch(stem_fold_rows_kernel<T, X, CC>, (unsigned)(n * h), 128, row_smem, st, src,     \
             static_cast<T*>(dst), (int)h, (int)w, s, stride_w, pad_w, (int)ow, round)
#define NEO_FOLD(T, X)                                                                      \
  do {                                                                                      \
    if (rows_ok) {                                                                          \
      if (c == 1) NEO_FOLD_ROWS(T, X, 1);                                                   \
      else if (c == 2) NEO_FOLD_ROWS(T, X, 2);                                              \
      else if (c == 3) NEO_FOLD_ROWS(T, X, 3);                                              \
      else NEO_FOLD_ROWS(T, X, 4);                                                          \
    } else {                                                                                \
      neo_launch(stem_fold_kernel<T, X>, grid, 256, 0, st, src, static_cast<T*>(dst), n, (int)c, \
                 (int)h, (int)w, s, stride_w, pad_w, (int)ow, round);                       \
    }                                                                                       \
  } while (0)
  if (dst_dtype == NEO_BF16) {
    if (xf == 8) NEO_FOLD(__nv_bfloat16, 8);
    else if (xf == 16) NEO_FOLD(__nv_bfloat16, 16);
    else if (xf == 32) NEO_FOLD(__nv_bfloat16, 32);
    else if (xf == 64) NEO_FOLD(__nv_bfloat16, 64);
    else NEO_CHECK_ARG(false, NEO_ERR_UNSUPPORTED, "stem fold block %d", xf);
  } else {
    if (xf == 4) NEO_FOLD(float, 4);
    else if (xf == 8) NEO_FOLD(float, 8);
    else if (xf == 16) NEO_FOLD(float, 16);
    else if (xf == 32) NEO_FOLD(float, 32);
    else NEO_CHECK_ARG(false, NEO_ERR_UNSUPPORTED, "stem fold block %d", xf);
  }
#undef NEO_FOLD
#undef NEO_FOLD_ROWS
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}
