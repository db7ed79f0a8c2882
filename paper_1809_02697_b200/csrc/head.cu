// K-HEAD: the classifier head of ResNet / DenseNet / Inception as ONE launch:
//   global average pool  (reference executor.py:103-128, avg: sum / win^2)
//   -> flatten -> dense + bias  (executor.py:197-203, a @ w.T + b)
//   -> softmax over the classes (executor.py:167-170, max-subtracted)
// In the reference (and in the unfused device path) these are three or four
// operators; here one cooperative launch runs them as three phases separated
// by grid-wide barriers (every CTA is co-resident: the grid is tiny), so the
// 7x7x2048 map is read once and the pooled features and logits never leave
// L2.  Arithmetic matches the unfused bf16 path: the pooled mean is rounded
// to bf16 (the pool's output type), the dense runs bf16 x bf16 -> fp32 on the
// tensor cores (warp-level mma.sync m16n8k16 fed from a cp.async ring: a
// 64 x 1000 x 2048 GEMM is too small for a TMA/tcgen05 pipeline to pay
// off), softmax in fp32.
// Requires C % 256 == 0 (two K halves of whole 128-wide chunks).
#include "neo_common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kImgTile = 16;                 // mma M
constexpr int kUnitTile = 64;                // 8 warps x n8

struct HeadParams {
  const __nv_bfloat16* x;   // (N, C/y, HW, y) bf16, NCHW[y]c with H*W = HW
  const __nv_bfloat16* w;   // (units, C) bf16 row-major
  const float* bias;        // (units) or null
  __nv_bfloat16* pooled;    // (N, C) scratch
  float* logits;            // (2, N, units) scratch: per-K-half partial logits
  float* out;               // (N, units)
  int* bar;                 // 3 counters, zero between launches
  int N, C, HW, y, units, softmax;
  float div;                // window size (H*W), the reference divides by it
  int x_fp8;                // x holds e4m3 bytes with per-tensor scale x_scale
  float x_scale;
  int dbg;                  // NEOB200_HEAD_DBG: phase timestamps of CTA 0 -> neo_head_dbg
};

__device__ unsigned long long g_head_clk[8];
__device__ __forceinline__ void head_stamp(const HeadParams& p, int i) {
  if (p.dbg && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_head_clk[i] = t;
  }
}

__device__ __forceinline__ void grid_barrier(int* ctr, int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1);
    const long long t0 = clock64();
    for (;;) {                                        // tight spin: a few us at most
      int v;
      asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (v >= target) break;
      if (clock64() - t0 > 20000000000ll) __trap();
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads) head_kernel(const __grid_constant__ HeadParams p) {
  head_stamp(p, 0);
  neo_pdl_wait();
  neo_pdl_trigger();
  head_stamp(p, 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- phase 1: global average pool.  A warp takes 8 consecutive
  // 8-channel groups of one image (coalesced 128-byte rows); lane = (pixel
  // slice lane / 8, group lane % 8) sums every 4th pixel with 4 loads in
  // flight, then the 4 slices are added across the warp ----
  {
    const int groups = p.C / 8, cb_total = p.C / p.y;
    const int wtasks = p.N * ((groups + 7) / 8);
    const int gw = blockIdx.x * (kThreads / 32) + warp, nw = gridDim.x * (kThreads / 32);
    const int slice = lane >> 3, j = lane & 7;
    const int step = p.y / 8;                         // uint4s per pixel of a channel block
    for (int task = gw; task < wtasks; task += nw) {
      const int n = task / ((groups + 7) / 8);
      const int grp = (task - n * ((groups + 7) / 8)) * 8 + j;
      float acc[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = 0.f;
      const bool live = grp < groups;
      const int c0 = grp * 8;
      const int cb = c0 / p.y, l0 = c0 - cb * p.y;
      const size_t eoff = ((size_t)(n * cb_total + (live ? cb : 0)) * p.HW) * p.y + l0;
      const uint4* src = reinterpret_cast<const uint4*>(p.x + eoff);
      // e4m3 input: 8 channels = 8 bytes per pixel, same pixel stride in uint2s
      const uint2* src8 = reinterpret_cast<const uint2*>(reinterpret_cast<const uint8_t*>(p.x) + eoff);
      for (int t0 = slice; p.x_fp8 && live && t0 < p.HW; t0 += 32) {
        uint2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          v[u] = t0 + 4 * u < p.HW ? __ldg(src8 + (size_t)(t0 + 4 * u) * step) : make_uint2(0, 0);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t w2[2] = {v[u].x, v[u].y};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const __nv_fp8x2_storage_t pr = (__nv_fp8x2_storage_t)(w2[e >> 1] >> (16 * (e & 1)));
            const float2 f = __half22float2(__half2(__nv_cvt_fp8x2_to_halfraw2(pr, __NV_E4M3)));
            acc[2 * e] += f.x;
            acc[2 * e + 1] += f.y;
          }
        }
      }
      // this slice's pixels t = slice + 4u: up to 8 loads in flight per batch
      for (int t0 = slice; !p.x_fp8 && live && t0 < p.HW; t0 += 32) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          v[u] = t0 + 4 * u < p.HW ? __ldg(src + (size_t)(t0 + 4 * u) * step) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v[u]);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(h[e]);
            acc[2 * e] += f.x;
            acc[2 * e + 1] += f.y;
          }
        }
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 8);
        acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 16);
      }
      if (slice == 0 && live) {
        uint4 o;
        uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          // e4m3: sum of the stored values, times the (power-of-two) scale
          const float a = acc[2 * e] * p.x_scale / p.div, b = acc[2 * e + 1] * p.x_scale / p.div;
          asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(ow[e]) : "f"(a), "f"(b));
        }
        *reinterpret_cast<uint4*>(p.pooled + (size_t)n * p.C + c0) = o;
      }
    }
  }
  head_stamp(p, 2);
  grid_barrier(p.bar, gridDim.x);
  head_stamp(p, 3);
  // ---- phase 2: logits = pooled @ w.T + bias (mma.sync bf16, fp32 acc).
  // A CTA tile is 16 images x 64 units; K streams through shared memory in
  // 128-wide chunks (4-stage cp.async ring, rows padded to 136 bf16 so the
  // fragment loads are bank-conflict free); warp w owns units [8w, 8w+8) ----
  {
    extern __shared__ __align__(16) uint8_t hsm[];
    constexpr int kChunk = 128, kPad = 136, kStages = 4;
    constexpr int kStageElems = (kImgTile + kUnitTile) * kPad;   // bf16 per stage
    __nv_bfloat16* ring = reinterpret_cast<__nv_bfloat16*>(hsm);
    const int img_tiles = (p.N + kImgTile - 1) / kImgTile;
    const int unit_tiles = (p.units + kUnitTile - 1) / kUnitTile;
    const int g = lane >> 2, q = lane & 3;            // fragment row group / k pair
    // K split in two halves over twice the CTAs; the halves' partial logits
    // are summed in a fixed order afterwards (deterministic)
    const int nch = p.C / kChunk / 2;
    for (int job = blockIdx.x; job < 2 * img_tiles * unit_tiles; job += gridDim.x) {
      const int half = job & 1, tile = job >> 1;
      const int n0 = (tile / unit_tiles) * kImgTile;
      const int u0 = (tile % unit_tiles) * kUnitTile;
      const int kbase = half * nch * kChunk;
      // chunk ch -> stage ch % kStages: rows 0..15 pooled images, 16..79 units;
      // 16-byte pieces: 80 rows x 16 = 1280 per chunk, 5 per thread
      auto issue = [&](int ch) {
        __nv_bfloat16* st = ring + (ch % kStages) * kStageElems;
        const int k0 = kbase + ch * kChunk;
#pragma unroll
        for (int i = 0; i < 5; ++i) {
          const int piece = tid + i * kThreads;
          const int row = piece >> 4, c16 = piece & 15;
          const __nv_bfloat16* src;
          bool ok;
          if (row < kImgTile) {
            ok = n0 + row < p.N;
            src = p.pooled + (size_t)(ok ? n0 + row : 0) * p.C + k0 + c16 * 8;
          } else {
            ok = u0 + row - kImgTile < p.units;
            src = p.w + (size_t)(ok ? u0 + row - kImgTile : 0) * p.C + k0 + c16 * 8;
          }
          const uint32_t d = smem_u32(st + row * kPad + c16 * 8);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src),
                       "r"(ok ? 16 : 0) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      float c[4] = {0.f, 0.f, 0.f, 0.f};
      for (int ch = 0; ch < kStages - 1; ++ch) {
        if (ch < nch) issue(ch);
        else asm volatile("cp.async.commit_group;" ::: "memory");
      }
      for (int ch = 0; ch < nch; ++ch) {
        asm volatile("cp.async.wait_group %0;" ::"n"(kStages - 2) : "memory");
        __syncthreads();                              // chunk ch landed for every thread
        if (ch + kStages - 1 < nch) issue(ch + kStages - 1);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        const __nv_bfloat16* st = ring + (ch % kStages) * kStageElems;
        const uint32_t* ra = reinterpret_cast<const uint32_t*>(st + g * kPad);
        const uint32_t* rb = reinterpret_cast<const uint32_t*>(st + (g + 8) * kPad);
        const uint32_t* rw = reinterpret_cast<const uint32_t*>(st + (kImgTile + warp * 8 + g) * kPad);
#pragma unroll
        for (int ks = 0; ks < kChunk / 16; ++ks) {
          const int kk = ks * 8 + q;
          asm volatile(
              "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
              "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
              : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
              : "r"(ra[kk]), "r"(rb[kk]), "r"(ra[kk + 4]), "r"(rb[kk + 4]), "r"(rw[kk]),
                "r"(rw[kk + 4]));
        }
      }
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();                                // ring free for the next tile
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int row = n0 + g + (e >= 2 ? 8 : 0);
        const int col = u0 + warp * 8 + 2 * q + (e & 1);
        if (row < p.N && col < p.units)
          p.logits[((size_t)half * p.N + row) * p.units + col] = c[e];
      }
    }
  }
  head_stamp(p, 4);
  grid_barrier(p.bar + 1, gridDim.x);
  head_stamp(p, 5);
  // ---- phase 3: logits = part0 + part1 + bias, then the row softmax with
  // max subtraction (or the plain logits) ----
  {
    __shared__ float red[kThreads / 32];
    for (int row = blockIdx.x; row < p.N; row += gridDim.x) {
      const float* a0 = p.logits + (size_t)row * p.units;
      const float* a1 = p.logits + ((size_t)p.N + row) * p.units;
      float* o = p.out + (size_t)row * p.units;
      if (!p.softmax) {
        for (int i = tid; i < p.units; i += kThreads)
          o[i] = __ldcg(a0 + i) + __ldcg(a1 + i) + (p.bias ? __ldg(p.bias + i) : 0.f);
        continue;
      }
      float mx = -INFINITY;
      for (int i = tid; i < p.units; i += kThreads) {
        const float v = __ldcg(a0 + i) + __ldcg(a1 + i) + (p.bias ? __ldg(p.bias + i) : 0.f);
        o[i] = v;
        mx = fmaxf(mx, v);
      }
      for (int s = 16; s > 0; s >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, s));
      if (lane == 0) red[warp] = mx;
      __syncthreads();
      mx = red[0];
      for (int w = 1; w < kThreads / 32; ++w) mx = fmaxf(mx, red[w]);
      __syncthreads();
      float sum = 0.f;
      for (int i = tid; i < p.units; i += kThreads) {
        const float e = expf(o[i] - mx);
        o[i] = e;
        sum += e;
      }
      for (int s = 16; s > 0; s >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, s);
      if (lane == 0) red[warp] = sum;
      __syncthreads();
      sum = 0.f;
      for (int w = 0; w < kThreads / 32; ++w) sum += red[w];
      __syncthreads();
      for (int i = tid; i < p.units; i += kThreads) o[i] = o[i] / sum;
    }
  }
  // the last CTA out re-arms the barriers for the next launch
  __syncthreads();
  head_stamp(p, 6);
  if (tid == 0 && atomicAdd(p.bar + 2, 1) == (int)gridDim.x - 1) {
    p.bar[0] = 0;
    p.bar[1] = 0;
    p.bar[2] = 0;
    __threadfence();
  }
}

}  // namespace

extern "C" int neo_classifier_head(const void* x, const void* w_bf16, const float* bias,
                                   void* pooled, float* logits, float* out, int* bar, int64_t n,
                                   int64_t c, int64_t hw, int y, int64_t units, int softmax,
                                   neo_stream_t stream) {
  return neo_classifier_head_q(x, NEO_BF16, 1.f, w_bf16, bias, pooled, logits, out, bar, n, c, hw,
                               y, units, softmax, stream);
}

extern "C" int neo_classifier_head_q(const void* x, int x_dtype, float x_scale,
                                     const void* w_bf16, const float* bias, void* pooled,
                                     float* logits, float* out, int* bar, int64_t n, int64_t c,
                                     int64_t hw, int y, int64_t units, int softmax,
                                     neo_stream_t stream) {
  NEO_CHECK_ARG(x && w_bf16 && pooled && out && bar, NEO_ERR_INVALID_ARG, "null pointer");
  NEO_CHECK_ARG(x_dtype == NEO_BF16 || (x_dtype == NEO_FP8 && x_scale > 0.f), NEO_ERR_INVALID_ARG,
                "head input must be bf16 or e4m3 with a positive scale");
  NEO_CHECK_ARG(logits, NEO_ERR_INVALID_ARG, "head needs a 2*n*units logits scratch");
  NEO_CHECK_ARG(n >= 1 && hw >= 1 && units >= 1 && c >= 256 && c % 256 == 0,
                NEO_ERR_SHAPE_MISMATCH, "head needs C a multiple of 256 (C=%lld)", (long long)c);
  NEO_CHECK_ARG(y >= 8 && y % 8 == 0 && c % y == 0, NEO_ERR_UNSUPPORTED,
                "head input block y=%d must be a multiple of 8 dividing C", y);
  NEO_CHECK_ARG(n * c < (1ll << 31) && n * units < (1ll << 31), NEO_ERR_UNSUPPORTED,
                "head too large");
  HeadParams p;
  p.x = static_cast<const __nv_bfloat16*>(x);
  p.w = static_cast<const __nv_bfloat16*>(w_bf16);
  p.bias = bias;
  p.pooled = static_cast<__nv_bfloat16*>(pooled);
  p.logits = logits;
  p.out = out;
  p.bar = bar;
  p.N = (int)n;
  p.C = (int)c;
  p.HW = (int)hw;
  p.y = y;
  p.units = (int)units;
  p.softmax = softmax;
  p.div = (float)hw;
  p.x_fp8 = x_dtype == NEO_FP8;
  p.x_scale = p.x_fp8 ? x_scale : 1.f;
  {
    static const char* dbg = getenv("NEOB200_HEAD_DBG");
    p.dbg = dbg ? 1 : 0;
  }
  // every CTA must be resident at once (grid barriers): one small CTA per SM
  // at most (the pool phase uses all of them, the GEMM phase its tiles)
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t work = std::max<int64_t>(2 * neo_ceil_div(n, kImgTile) * neo_ceil_div(units, kUnitTile),
                                         neo_ceil_div(n * (c / 64), 8));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(work, sms));
  constexpr size_t kSmem = 4 * (kImgTile + kUnitTile) * 136 * 2;
  static bool attr_done[64] = {};
  if (!attr_done[dev & 63]) {
    NEO_CUDA_TRY(cudaFuncSetAttribute(head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kSmem));
    attr_done[dev & 63] = true;
  }
  // cooperative: the grid barriers need every CTA resident; the launch fails
  // (instead of deadlocking) where that cannot be guaranteed (e.g. an MPS
  // client limited to fewer SMs)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = neo_pdl_enabled() ? 2 : 1;
  NEO_CUDA_TRY(cudaLaunchKernelEx(&cfg, head_kernel, p));
  return NEO_OK;
}

extern "C" __attribute__((visibility("default"))) int neo_head_dbg(unsigned long long* host) {
  return (int)cudaMemcpyFromSymbol(host, g_head_clk, 8 * sizeof(unsigned long long));
}
