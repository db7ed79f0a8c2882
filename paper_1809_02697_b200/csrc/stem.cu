// K-STEM: the image stem of ResNet / DenseNet / SSD-ResNet as ONE kernel:
//   conv 7x7 stride 2 pad 3 over a C<=4 channel NCHW f32 or bf16 image, K = 64
//   -> scale/shift -> bias -> relu      (Epilogue, reference kernels.py:185-197)
//   -> max pool 3x3 stride 2 pad 1      (reference executor.py:103-128, -inf pad)
//   -> NCHW[y]c bf16 (optionally a channel-block window of a concat buffer).
// In the reference these are three operators (conv_blocked on the packed
// 3-channel input, kernels.py:250-303, then _pool2d); here neither the packed
// input nor the 112x112 conv map ever reaches HBM.
//
// Work unit = one 7x7 tile of pooled outputs of one image.  Its 3x3/2 pool
// windows cover a 15x15 conv tile, computed as two M=128 tcgen05 MMA tiles of
// 16 conv rows x 8 conv columns (16 x 16, row 15 / column 15 unused).
//
// No im2col: the input patch sits in shared memory as bf16 [row][col][4
// channels] (8 bytes per pixel, channel 3 zero).  For kernel row r and a pair
// of horizontal taps (s, s+1), the 8 K-elements (2 taps x 4 channels) of conv
// pixel (g, i) are the 16 contiguous bytes at input (2g + r, 2i + s), and conv
// pixel (g, i+1) starts exactly 16 bytes later (stride 2).  So eight conv
// columns form an 8-row x 16-byte no-swizzle UMMA core matrix in place:
//   A(step r, q) = patch + r*pitch + 32*q,  LBO = 16 B (next tap pair),
//                  SBO = 2*pitch (next conv row = two input rows down).
// K per step = 16 = taps {4q..4q+3} x 4 channels; 7 kernel rows x 2 steps =
// 14 MMAs (M=128, N=64) per 16x8 conv tile.  Tap 7 and channel 3 carry zero
// weights.  The weights are a resident 28 KB image [step][chunk][64 k][8].
//
// Warp roles (768 threads, persistent over units, one CTA per SM):
//   warp 0      TMA producer: f32/bf16 patch box (37 rows x C planes,
//               zero fill outside the image) into a 4-deep ring
//   warp 1      TMEM allocator + single-thread MMA issuer (4 accumulators of
//               2 x 64 columns)
//   warps 2-7   converters: planar box -> bf16 [row][col][4] patch (RN)
//               (4-deep ring), then fence.proxy.async for the tensor core
//   warps 8-23  epilogue: tcgen05.ld -> scale/shift/bias/relu -> bf16 conv
//               tile in shared memory (double buffered, XOR-swizzled 16-byte
//               chunks; pixels outside the conv map stored as -inf) -> 3x3/2
//               max pool -> 16-byte global stores
#include <cudaTypedefs.h>

#include <mutex>

#include "neo_common.cuh"

namespace {

constexpr int kConvWarps = 6;                 // warps 2..7
constexpr int kEpiThreads = 512;               // warps 8..23
constexpr int kThreads = 64 + kConvWarps * 32 + kEpiThreads;
constexpr int kRawStages = 4;                  // max f32 box ring depth
constexpr int kPatchStages = 4;                // converted patches in flight
// input box per unit: 37 rows x kBoxW columns starting at the conv tile's
// first tap column 4*q0 - 5 rounded down to a 16-byte boundary (a TMA box
// must start 16-byte aligned in its innermost dimension; an unaligned,
// negative start column faults), so patch column j is box column j + off
// with off = (4*q0 - 5) - start: f32 boxes start 4 columns aligned (off = 3,
// 44 columns), bf16 boxes 8 columns aligned (off 3 or 7, 48 columns)
constexpr int kBoxH = 37;
template <typename TX> struct BoxOf;
template <> struct BoxOf<float> { static constexpr int W = 44, kAlign = 4; };
template <> struct BoxOf<__nv_bfloat16> { static constexpr int W = 48, kAlign = 8; };
__device__ __forceinline__ float to_float(float v) { return v; }
__device__ __forceinline__ float to_float(__nv_bfloat16 v) { return __bfloat162float(v); }
constexpr int kPatchCols = 38;                 // input columns the MMAs read
constexpr int kPitch = kPatchCols * 8;         // bytes per bf16x4 patch row
constexpr int kPatchBytes = kBoxH * kPitch;    // 11248
constexpr int kPatchSlot = 11264;              // patch slot (16-byte multiple)
static_assert(kPatchBytes <= kPatchSlot, "patch slot too small");
constexpr int kSteps = 14;                     // (r, q) K steps per conv tile
constexpr int kWBytes = kSteps * 2 * 64 * 16;  // 28672
constexpr int kCtileBytes = 16 * 16 * 128;     // 16x16 conv px x 64 bf16
constexpr int kPool = 7;                       // pooled tile edge

struct StemParams {
  CUtensorMap tmX;          // 3-D f32 (W, H, N*C), box (44, 37, C)
  const void* wimg;         // bf16 [14][2][64][8]
  const float* scale;
  const float* shift;
  const float* bias;
  __nv_bfloat16* out;
  int N, C, OH, OW, PH, PW;
  int tiles_h, tiles_w, num_units;
  int y, out_cb_off, out_cb_total;
  int relu;
  int out_fp8;              // store e4m3(pooled * out_qscale) bytes instead of bf16
  float out_qscale;
  uint32_t raw_bytes;       // BoxOf<TX>::W * 37 * C * sizeof(TX)
  int raw_stages;           // f32 box ring depth (4, 3 for C = 4)
  int dbg;                  // NEOB200_STEM_DBG: 1 no MMAs, 2 no TMEM loads, 4 no TMA,
                            // 8 no pooling, 16 no conversion, 32 phase clocks
};

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(lo), "f"(hi));
  return r;
}

__device__ __forceinline__ uint32_t bmax2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("max.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// NEOB200_STEM_DBG & 32: per-CTA phase clocks of the MMA thread and of
// epilogue warp 8 (lane 0) -> neo_stem_dbg_clk
__device__ unsigned long long g_stem_clk[148 * 8];

__device__ __forceinline__ void unit_origin(const StemParams& p, int u, int& n, int& p0, int& q0) {
  const int tw = u % p.tiles_w;
  const int t = u / p.tiles_w;
  const int th = t % p.tiles_h;
  n = t / p.tiles_h;
  p0 = th * kPool;
  q0 = tw * kPool;
}

template <typename TX>
__global__ void __launch_bounds__(kThreads, 1) stem_conv_pool_kernel(const __grid_constant__ StemParams p) {
  constexpr int kBoxW = BoxOf<TX>::W;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (sbase - smem_u32(smem_raw));
  // layout: weights | ctile x2 | raw ring | patch x2 | params | barriers
  const uint32_t sW = sbase;
  const uint32_t sCt = sW + kWBytes;
  const uint32_t sRaw = sCt + 2 * kCtileBytes;
  const uint32_t raw_slot = (p.raw_bytes + 127u) & ~127u;
  const uint32_t sPatch = sRaw + p.raw_stages * raw_slot;
  const uint32_t sPar = sPatch + kPatchStages * kPatchSlot;
  const uint32_t sBar = sPar + 3 * 64 * 4;
  auto raw_full = [&](int i) { return sBar + 8u * i; };
  auto raw_empty = [&](int i) { return sBar + 32u + 8u * i; };
  auto patch_full = [&](int i) { return sBar + 64u + 8u * i; };
  auto patch_empty = [&](int i) { return sBar + 96u + 8u * i; };
  auto tfull = [&](int i) { return sBar + 128u + 8u * i; };
  auto tempty = [&](int i) { return sBar + 160u + 8u * i; };
  const uint32_t wbar = sBar + 192u;
  const uint32_t tslot = sBar + 200u;
  float* par = reinterpret_cast<float*>(gbase + (sPar - sbase));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&p.tmX);
    for (int i = 0; i < kRawStages; ++i) {
      mbar_init(raw_full(i), 1);
      mbar_init(raw_empty(i), kConvWarps);
    }
    for (int i = 0; i < kPatchStages; ++i) {
      mbar_init(patch_full(i), kConvWarps);
      mbar_init(patch_empty(i), 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(tfull(i), 1);
      mbar_init(tempty(i), kEpiThreads / 32);
    }
    mbar_init(wbar, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(tslot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(gbase + (tslot - sbase));
  neo_pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      // weights are static (packed at load time): fetch before the PDL wait
      mbar_arrive_expect_tx(wbar, kWBytes);
      bulk_load(sW, p.wimg, kWBytes, wbar);
      neo_pdl_wait();
      int s = 0;
      uint32_t ph = 0;
      for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
        int n, p0, q0;
        unit_origin(p, u, n, p0, q0);
        mbar_wait(raw_empty(s), ph ^ 1u);
        if (p.dbg & 4) {
          mbar_arrive(raw_full(s));
        } else {
        mbar_arrive_expect_tx(raw_full(s), p.raw_bytes);
        // input origin: conv row 2*p0 - 1 -> input row 2*(2*p0 - 1) - 3;
        // first column 4*q0 - 5 rounded down to the 16-byte boundary
        const int c0 = (4 * q0 - 5) & ~(BoxOf<TX>::kAlign - 1);
        tma_load_3d(sRaw + s * raw_slot, &p.tmX, raw_full(s), c0, 4 * p0 - 5, n * p.C);
        }
        if (++s == p.raw_stages) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc(1u, 128, 64);
      // descriptors: A no-swizzle K-major, LBO 16 B, SBO two patch rows;
      // B [step][chunk][k][8]: LBO 1024 B (chunk), SBO 128 B (8 k rows)
      const uint64_t a0 = umma_smem_desc(sPatch, 16, 2 * kPitch, 0);
      const uint64_t b0 = umma_smem_desc(sW, 1024, 128, 0);
      const uint32_t alo0 = (uint32_t)a0, ahi = (uint32_t)(a0 >> 32);
      const uint32_t blo0 = (uint32_t)b0, bhi = (uint32_t)(b0 >> 32);
      mbar_wait(wbar, 0);
      const bool prof = (p.dbg & 32) != 0;
      long long m_pf = 0, m_te = 0, m_is = 0;
      int it = 0;
      for (int u = blockIdx.x; u < p.num_units; u += gridDim.x, ++it) {
        const int pb = it % kPatchStages, a = it & 3;
        long long t0 = prof ? clock64() : 0;
        mbar_wait(patch_full(pb), (uint32_t)(it / kPatchStages) & 1u);
        if (prof) { const long long t = clock64(); m_pf += t - t0; t0 = t; }
        mbar_wait(tempty(a), ((uint32_t)(it >> 2) & 1u) ^ 1u);
        if (prof) { const long long t = clock64(); m_te += t - t0; t0 = t; }
        tc_fence_after();
        const uint32_t abase = alo0 + (uint32_t)(pb * kPatchSlot) / 16u;
#pragma unroll
        for (int j = 0; j < 2 && !(p.dbg & 1); ++j) {
          const uint32_t d = tmem_base + (uint32_t)(a * 128 + j * 64);
#pragma unroll
          for (int t = 0; t < kSteps; ++t) {
            const int r = t >> 1, q = t & 1;
            const uint32_t alo = abase + (uint32_t)(r * kPitch + 32 * q + 128 * j) / 16u;
            const uint32_t blo = blo0 + (uint32_t)(t * 2048) / 16u;
            asm volatile(
                "{\n\t.reg .pred pa;\n\t.reg .b64 ad, bd;\n\t"
                "setp.ne.b32 pa, %6, 0;\n\t"
                "mov.b64 ad, {%1, %2};\n\t"
                "mov.b64 bd, {%3, %4};\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], ad, bd, %5, pa;\n\t}" ::"r"(d),
                "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(t == 0 ? 0u : 1u)
                : "memory");
          }
        }
        umma_commit(patch_empty(pb));
        umma_commit(tfull(a));
        if (prof) m_is += clock64() - t0;
      }
      if (prof) {
        g_stem_clk[blockIdx.x * 8 + 0] = m_pf;
        g_stem_clk[blockIdx.x * 8 + 1] = m_te;
        g_stem_clk[blockIdx.x * 8 + 2] = m_is;
      }
    }
  } else if (warp < 2 + kConvWarps) {
    // ---- converters: f32 [c][37][44] -> bf16 [37][38][4] ----
    const int ctid = threadIdx.x - 64;
    const int C = p.C;
    int s = 0;
    uint32_t ph = 0;
    int it = 0;
    const int nconv = (p.dbg & 16) ? 0 : kBoxH * kPatchCols;
    for (int u = blockIdx.x; u < p.num_units; u += gridDim.x, ++it) {
      const int pb = it % kPatchStages;
      mbar_wait(raw_full(s), ph);
      mbar_wait(patch_empty(pb), ((uint32_t)(it / kPatchStages) & 1u) ^ 1u);
      const TX* raw = reinterpret_cast<const TX*>(gbase + (sRaw + s * raw_slot - sbase));
      int un, up0, uq0;
      unit_origin(p, u, un, up0, uq0);
      const int off = (4 * uq0 - 5) - ((4 * uq0 - 5) & ~(BoxOf<TX>::kAlign - 1));
      uint8_t* patch = gbase + (sPatch + pb * kPatchSlot - sbase);
      constexpr int plane = kBoxW * kBoxH;
#pragma unroll 4
      for (int idx = ctid; idx < nconv; idx += kConvWarps * 32) {
        const int row = idx / kPatchCols, col = idx - row * kPatchCols;
        const TX* rp = raw + row * kBoxW + col + off;
        const float v0 = to_float(rp[0]);
        const float v1 = C > 1 ? to_float(rp[plane]) : 0.f;
        const float v2 = C > 2 ? to_float(rp[2 * plane]) : 0.f;
        const float v3 = C > 3 ? to_float(rp[3 * plane]) : 0.f;
        *reinterpret_cast<uint2*>(patch + row * kPitch + col * 8) =
            make_uint2(pack_bf16x2(v0, v1), pack_bf16x2(v2, v3));
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(patch_full(pb));
        mbar_arrive(raw_empty(s));
      }
      if (++s == p.raw_stages) {
        s = 0;
        ph ^= 1u;
      }
    }
  } else {
    // ---- epilogue: 16 warps; warp = (TMEM lane quarter q, M tile j, column
    // half) drains 32 accumulator columns of 32 conv pixels ----
    const int ew = warp - 2 - kConvWarps;
    const int q = warp & 3;
    const int j = (ew >> 2) & 1;
    const int half = ew >> 3;
    const int etid = threadIdx.x - 64 - kConvWarps * 32;
    neo_pdl_wait();
    if (etid < 64) {
      par[etid] = p.scale ? p.scale[etid] : 1.f;
      par[64 + etid] = p.shift ? p.shift[etid] : 0.f;
      par[128 + etid] = p.bias ? p.bias[etid] : 0.f;
    }
    named_bar_sync(1, kEpiThreads);
    const bool affine = p.scale != nullptr || p.shift != nullptr;
    const int m = q * 32 + lane;            // accumulator row = conv pixel (g, i)
    const int g = m >> 3;
    const int i = (m & 7) + 8 * j;
    const uint32_t relu_bits = p.relu ? 1u : 0u;
    const bool prof = (p.dbg & 32) != 0 && warp == 2 + kConvWarps && lane == 0;
    long long t0 = 0, c_wait = 0, c_math = 0, c_bar = 0, c_pool = 0;
    int it = 0;
    for (int u = blockIdx.x; u < p.num_units; u += gridDim.x, ++it) {
      int n, p0, q0;
      unit_origin(p, u, n, p0, q0);
      const int cr0 = 2 * p0 - 1, cc0 = 2 * q0 - 1;
      // conv pixels outside the conv map hold -inf: the pool below then needs
      // no bounds checks (reference -inf padding, executor.py:103-128)
      const bool valid = cr0 + g >= 0 && cr0 + g < p.OH && cc0 + i >= 0 && cc0 + i < p.OW;
      const int a = it & 3;
      if (prof) t0 = clock64();
      mbar_wait(tfull(a), (uint32_t)(it >> 2) & 1u);
      if (prof) { const long long t = clock64(); c_wait += t - t0; t0 = t; }
      tc_fence_after();
      uint8_t* ct = gbase + (sCt + (it & 1) * kCtileBytes - sbase);
      uint8_t* row_base = ct + (g * 16 + i) * 128;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) +
                             (uint32_t)(a * 128 + j * 64 + half * 32);
#pragma unroll
      for (int c16 = 0; c16 < 2; ++c16) {
        uint32_t v[16];
        if (p.dbg & 2) {
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] = 0u;
        } else {
          tmem_ld16(taddr + c16 * 16, v);
          tmem_ld_wait_regs(v);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k0 = half * 32 + c16 * 16 + h * 8;
          float f[8];
          const float4 b0 = *reinterpret_cast<const float4*>(par + 128 + k0);
          const float4 b1 = *reinterpret_cast<const float4*>(par + 128 + k0 + 4);
          const float bi[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
          if (affine) {
            const float4 s0 = *reinterpret_cast<const float4*>(par + k0);
            const float4 s1 = *reinterpret_cast<const float4*>(par + k0 + 4);
            const float4 t0 = *reinterpret_cast<const float4*>(par + 64 + k0);
            const float4 t1 = *reinterpret_cast<const float4*>(par + 64 + k0 + 4);
            const float sc[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
            const float sh[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
#pragma unroll
            for (int e = 0; e < 8; ++e) f[e] = fmaf(__uint_as_float(v[h * 8 + e]), sc[e], sh[e]) + bi[e];
          } else {
            // identity scale/shift: fma(v, 1, 0) == v; packed f32x2 adds
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              const float2 r = __fadd2_rn(make_float2(__uint_as_float(v[h * 8 + e]),
                                                      __uint_as_float(v[h * 8 + e + 1])),
                                          make_float2(bi[e], bi[e + 1]));
              f[e] = r.x;
              f[e + 1] = r.y;
            }
          }
          uint32_t o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (relu_bits)
              asm("cvt.rn.relu.bf16x2.f32 %0, %2, %1;" : "=r"(o[e]) : "f"(f[2 * e]), "f"(f[2 * e + 1]));
            else
              asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(o[e]) : "f"(f[2 * e]), "f"(f[2 * e + 1]));
            if (!valid) o[e] = 0xFF80FF80u;
          }
          const int chunk = k0 >> 3;
          *reinterpret_cast<uint4*>(row_base + ((chunk ^ (i & 7)) << 4)) =
              make_uint4(o[0], o[1], o[2], o[3]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty(a));
      if (prof) { const long long t = clock64(); c_math += t - t0; t0 = t; }
      named_bar_sync(1, kEpiThreads);       // conv tile complete
      if (prof) { const long long t = clock64(); c_bar += t - t0; t0 = t; }
      // 3x3/2 max pool over the conv tile: item = (pooled row, col, 8-ch chunk)
      for (int item = etid; item < ((p.dbg & 8) ? 0 : kPool * kPool * 8); item += kEpiThreads) {
        const int pp = item / 56, rem = item - pp * 56;
        const int pq = rem >> 3, chunk = rem & 7;
        const int P = p0 + pp, Q = q0 + pq;
        if (P >= p.PH || Q >= p.PW) continue;
        uint32_t b0 = 0xFF80FF80u, b1 = b0, b2 = b0, b3 = b0;   // -inf pairs
#pragma unroll
        for (int dg = 0; dg < 3; ++dg) {
#pragma unroll
          for (int di = 0; di < 3; ++di) {
            const int gg = 2 * pp + dg, ii = 2 * pq + di;
            const uint4 v = *reinterpret_cast<const uint4*>(ct + (gg * 16 + ii) * 128 +
                                                            ((chunk ^ (ii & 7)) << 4));
            b0 = bmax2(b0, v.x);
            b1 = bmax2(b1, v.y);
            b2 = bmax2(b2, v.z);
            b3 = bmax2(b3, v.w);
          }
        }
        const int k = chunk * 8;
        const int kb = k / p.y, j0 = k - kb * p.y;
        const size_t off =
            ((((size_t)n * p.out_cb_total + p.out_cb_off + kb) * p.PH + P) * p.PW + Q) * p.y + j0;
        if (p.out_fp8) {
          // e4m3 output: the pooled bf16 value (exact in f32) times the
          // output scale, rounded once (RN, satfinite)
          const uint32_t bw[4] = {b0, b1, b2, b3};
          uint32_t q[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float2 lo = make_float2(__uint_as_float(bw[2 * e] << 16) * p.out_qscale,
                                          __uint_as_float(bw[2 * e] & 0xFFFF0000u) * p.out_qscale);
            const float2 hi = make_float2(__uint_as_float(bw[2 * e + 1] << 16) * p.out_qscale,
                                          __uint_as_float(bw[2 * e + 1] & 0xFFFF0000u) * p.out_qscale);
            q[e] = (uint32_t)__nv_cvt_float2_to_fp8x2(lo, __NV_SATFINITE, __NV_E4M3) |
                   ((uint32_t)__nv_cvt_float2_to_fp8x2(hi, __NV_SATFINITE, __NV_E4M3) << 16);
          }
          *reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(p.out) + off) = make_uint2(q[0], q[1]);
        } else {
          *reinterpret_cast<uint4*>(p.out + off) = make_uint4(b0, b1, b2, b3);
        }
      }
      if (prof) { const long long t = clock64(); c_pool += t - t0; t0 = t; }
    }
    if (prof) {
      g_stem_clk[blockIdx.x * 8 + 3] = c_wait;
      g_stem_clk[blockIdx.x * 8 + 4] = c_math;
      g_stem_clk[blockIdx.x * 8 + 5] = c_bar;
      g_stem_clk[blockIdx.x * 8 + 6] = c_pool;
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

__global__ void stem_pack_kernel(const float* __restrict__ w, __nv_bfloat16* __restrict__ img,
                                 int C) {
  // img[t][h][k][e]: step t = (r, q), chunk h, element e -> tap s = 4q + 2h + e/4, channel e%4
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= kSteps * 2 * 64 * 8) return;
  const int e = idx & 7, k = (idx >> 3) & 63, h = (idx >> 9) & 1, t = idx >> 10;
  const int r = t >> 1, q = t & 1;
  const int s = 4 * q + 2 * h + (e >> 2), c = e & 3;
  const float v = (s < 7 && c < C) ? w[((k * C + c) * 7 + r) * 7 + s] : 0.f;
  img[idx] = __float2bfloat16_rn(v);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

}  // namespace

extern "C" int neo_stem_pack_weights(const float* w_kcrs, void* img, int64_t k, int64_t c,
                                     int64_t r, int64_t s, neo_stream_t stream) {
  NEO_CHECK_ARG(w_kcrs && img, NEO_ERR_INVALID_ARG, "null pointer");
  NEO_CHECK_ARG(k == 64 && r == 7 && s == 7 && c >= 1 && c <= 4, NEO_ERR_UNSUPPORTED,
                "stem image needs K=64, 7x7, C<=4 (got K=%lld C=%lld %lldx%lld)", (long long)k,
                (long long)c, (long long)r, (long long)s);
  const int total = kSteps * 2 * 64 * 8;
  neo_launch(stem_pack_kernel, dim3((total + 255) / 256), dim3(256), 0,
             static_cast<cudaStream_t>(stream), w_kcrs, static_cast<__nv_bfloat16*>(img), (int)c);
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}

extern "C" int64_t neo_stem_weight_bytes(void) { return kWBytes; }

extern "C" int neo_stem_conv_pool(const void* x, int x_dtype, const void* wimg, void* out,
                                  const float* scale, const float* shift, const float* bias,
                                  int relu, int64_t n, int64_t c, int64_t h, int64_t w, int y,
                                  int out_cb_offset, int out_cb_total, neo_stream_t stream) {
  return neo_stem_conv_pool_q(x, x_dtype, wimg, out, NEO_BF16, 1.f, scale, shift, bias, relu, n,
                              c, h, w, y, out_cb_offset, out_cb_total, stream);
}

extern "C" int neo_stem_conv_pool_q(const void* x, int x_dtype, const void* wimg, void* out,
                                    int out_dtype, float out_scale, const float* scale,
                                    const float* shift, const float* bias, int relu, int64_t n,
                                    int64_t c, int64_t h, int64_t w, int y, int out_cb_offset,
                                    int out_cb_total, neo_stream_t stream) {
  NEO_CHECK_ARG(x && wimg && out, NEO_ERR_INVALID_ARG, "null tensor pointer");
  NEO_CHECK_ARG(out_dtype == NEO_BF16 || (out_dtype == NEO_FP8 && out_scale > 0.f),
                NEO_ERR_INVALID_ARG, "stem output must be bf16 or e4m3 with a positive scale");
  NEO_CHECK_ARG(x_dtype == NEO_F32 || x_dtype == NEO_BF16, NEO_ERR_INVALID_ARG, "bad input dtype");
  const bool xbf = x_dtype == NEO_BF16;
  const int es = xbf ? 2 : 4, box_w = xbf ? BoxOf<__nv_bfloat16>::W : BoxOf<float>::W;
  NEO_CHECK_ARG(n >= 1 && c >= 1 && c <= 4 && h >= 1 && w >= 1, NEO_ERR_SHAPE_MISMATCH,
                "stem needs 1..4 input channels (C=%lld)", (long long)c);
  NEO_CHECK_ARG((w * es) % 16 == 0, NEO_ERR_UNSUPPORTED,
                "stem input rows must be 16-byte multiples (width %lld)", (long long)w);
  NEO_CHECK_ARG(y == 8 || y == 16 || y == 32 || y == 64, NEO_ERR_UNSUPPORTED,
                "stem output block %d not in {8,16,32,64}", y);
  const int64_t OH = (h + 6 - 7) / 2 + 1, OW = (w + 6 - 7) / 2 + 1;
  const int64_t PH = (OH + 2 - 3) / 2 + 1, PW = (OW + 2 - 3) / 2 + 1;
  NEO_CHECK_ARG(OH >= 1 && OW >= 1 && PH >= 1 && PW >= 1, NEO_ERR_SHAPE_MISMATCH, "empty stem output");
  const int cbt = out_cb_total > 0 ? out_cb_total : 64 / y;
  NEO_CHECK_ARG(out_cb_offset >= 0 && out_cb_offset + 64 / y <= cbt, NEO_ERR_SHAPE_MISMATCH,
                "output window [%d, %d) outside %d blocks", out_cb_offset, out_cb_offset + 64 / y,
                cbt);
  auto encode = encode_fn();
  NEO_CHECK_ARG(encode != nullptr, NEO_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  StemParams kp;
  memset(&kp, 0, sizeof(kp));
  {
    cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)(n * c)};
    cuuint64_t strides[2] = {(cuuint64_t)(w * es), (cuuint64_t)(h * w * es)};
    cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)kBoxH, (cuuint32_t)c};
    cuuint32_t estr[3] = {1u, 1u, 1u};
    CUresult r = encode(&kp.tmX, xbf ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        3, const_cast<void*>(x), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    NEO_CHECK_ARG(r == CUDA_SUCCESS, NEO_ERR_CUDA, "stem tensor map encode failed (%d)", (int)r);
  }
  kp.wimg = wimg;
  kp.scale = scale;
  kp.shift = shift;
  kp.bias = bias;
  kp.out = static_cast<__nv_bfloat16*>(out);
  kp.N = (int)n;
  kp.C = (int)c;
  kp.OH = (int)OH;
  kp.OW = (int)OW;
  kp.PH = (int)PH;
  kp.PW = (int)PW;
  kp.tiles_h = (int)neo_ceil_div(PH, kPool);
  kp.tiles_w = (int)neo_ceil_div(PW, kPool);
  const int64_t units = n * kp.tiles_h * kp.tiles_w;
  NEO_CHECK_ARG(units < (1ll << 31), NEO_ERR_UNSUPPORTED, "too many stem tiles");
  kp.num_units = (int)units;
  kp.y = y;
  kp.out_cb_off = out_cb_offset;
  kp.out_cb_total = cbt;
  kp.relu = relu;
  kp.out_fp8 = out_dtype == NEO_FP8;
  kp.out_qscale = kp.out_fp8 ? (float)(1.0 / (double)out_scale) : 1.f;
  kp.raw_bytes = (uint32_t)(box_w * kBoxH * c * es);
  {
    static const char* dbg = getenv("NEOB200_STEM_DBG");
    kp.dbg = dbg ? atoi(dbg) : 0;
  }
  const uint32_t raw_slot = (kp.raw_bytes + 127u) & ~127u;
  const size_t fixed = 1024 + kWBytes + 2 * kCtileBytes + kPatchStages * kPatchSlot + 3 * 64 * 4 + 256;
  kp.raw_stages = (int)std::min<size_t>(kRawStages, (227 * 1024 - fixed) / raw_slot);
  NEO_CHECK_ARG(kp.raw_stages >= 2, NEO_ERR_UNSUPPORTED, "stem input ring does not fit");
  const size_t smem = fixed + (size_t)kp.raw_stages * raw_slot;
  static bool attr_done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_done[dev & 63]) {
    NEO_CUDA_TRY(cudaFuncSetAttribute(stem_conv_pool_kernel<float>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    NEO_CUDA_TRY(cudaFuncSetAttribute(stem_conv_pool_kernel<__nv_bfloat16>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr_done[dev & 63] = true;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>(units, sms);
  if (xbf)
    neo_launch(stem_conv_pool_kernel<__nv_bfloat16>, dim3(grid), dim3(kThreads), smem,
               static_cast<cudaStream_t>(stream), kp);
  else
    neo_launch(stem_conv_pool_kernel<float>, dim3(grid), dim3(kThreads), smem,
               static_cast<cudaStream_t>(stream), kp);
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}

extern "C" __attribute__((visibility("default"))) int neo_stem_dbg_clk(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_stem_clk, n * sizeof(unsigned long long));
}
