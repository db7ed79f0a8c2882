// K-JUNCTION: two chained 1x1 convolutions as ONE tcgen05 kernel -- the
// junction between two ResNet bottleneck blocks:
//
//   y1 = relu(x  * W1 + b1 + residual)     block i's 1x1 expand  (+ shortcut)
//   y2 = relu(y1 * W2 + b2)                block i+1's 1x1 reduce
//
// (reference: two conv_blocked calls, kernels.py:250-303, each with the
// Epilogue of :74-87 applied in the order of :185-197; the layout pass keeps
// both in NCHW[64]c so neither needs a transform, passes.py:167-255).  y1 is
// still written -- it is block i+1's shortcut -- but the reduce conv reads it
// from shared memory instead of HBM, and one launch's fill and drain go away.
//
// Per 128-pixel M tile the N1 expand channels are walked in chunks of 128:
//   GEMM1(c): D1[c % 2] = x_tile * W1[c]          (TMEM, double buffered)
//   epilogue(c): D1 -> +b1 +residual -> relu -> bf16 -> two 64-channel
//                SW128 K-major slots in shared memory (the residual block was
//                TMA-loaded into the same slot) -> TMA store to y1
//   GEMM2(c): D2 += slot[c % 2][0..1] * W2[:, c]   (the slots ARE the A operand)
// and after the last chunk D2 -> +b2 -> relu -> bf16 -> TMA store to y2.  The
// MMA thread issues GEMM1(c + 1) before GEMM2(c), so the tensor core works on
// the next chunk while the epilogue drains this one.  GEMM2 accumulates y1's
// channel blocks in order, 16 channels per step -- the same sequence as the
// stand-alone reduce conv, so y2 is bit-identical to running the two convs.
//
// Warp roles (576 threads, persistent over M tiles, one CTA per SM):
//   warp 0      TMA producer (x / W1 slices into ring 1, W2 slices into ring 2)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-17  epilogue: warp w drains TMEM lane quarter w % 4 and 32 of the
//               128 columns of each chunk ((w - 2) / 4 = which 32); biases
//               are staged in shared memory once per CTA
#include <cudaTypedefs.h>

#include <mutex>

#include "neo_common.cuh"

namespace {

constexpr int kThreads = 576;
constexpr int kEpiWarps = 16;
constexpr int kTileM = 128;
constexpr int kChunk = 128;          // expand channels per chunk (two 64-lane blocks)
constexpr int kSlot = 128 * 128;     // one 64-channel bf16 block of 128 pixels (SW128)
constexpr int kSmemBudget = 227 * 1024;

struct JunctionParams {
  CUtensorMap tmX;    // 5-D (64, W, H, C1/64, N), box (64, BW, BH, 1, BNI)
  CUtensorMap tmW1;   // 3-D (64, N1, C1/64) over the umma weight image, box (64, 128, 1)
  CUtensorMap tmW2;   // 3-D (64, N2, N1/64), box (64, N2, 1)
  CUtensorMap tmR;    // 5-D (64, W, H, N1/64, N) residual, box (64, BW, BH, 1, BNI)
  CUtensorMap tmY1;   // 5-D (64, W, H, N1/64, N) expand output
  CUtensorMap tmY2;   // 5-D (64, W, H, N2/64, N) reduce output
  const float* b1;    // N1 (may be null)
  const float* b2;    // N2 (may be null)
  int N, H, W, C1, N1, N2;
  int BW, BH, BNI;
  int tiles_w, tiles_h, num_tiles;
  int k1;             // C1 / 64 slices per GEMM1 chunk
  int chunks;         // N1 / 128
  int stages1, stages2;
  int relu1, relu2, has_res;
  uint32_t tx_a1, tx_b1, tx_b2, box_bytes;
};

__device__ __forceinline__ void tile_origin(const JunctionParams& p, int t, int& n0, int& h0,
                                            int& w0) {
  const int tw = t % p.tiles_w;
  const int q = t / p.tiles_w;
  const int th = q % p.tiles_h;
  n0 = (q / p.tiles_h) * p.BNI;
  h0 = th * p.BH;
  w0 = tw * p.BW;
}

__device__ __forceinline__ void mma_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// one 64-channel K slice (4 steps of 16) from SW128 K-major tiles
__device__ __forceinline__ void mma_slice(uint32_t d, uint32_t a_addr, uint32_t b_addr,
                                          uint32_t idesc, uint32_t acc0) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
    mma_bf16(d, umma_smem_desc(a_addr + 32u * k, 16, 1024, 2),
             umma_smem_desc(b_addr + 32u * k, 16, 1024, 2), idesc, (k == 0 ? acc0 : 1u));
}

// 32 accumulator columns (half a 64-channel block) of one pixel row ->
// (+bias, +residual from the slot, relu) -> bf16 into the same swizzled slot
// row; `bias` points at the block's 64 staged (shared-memory) biases
template <bool RES>
__device__ __forceinline__ void drain32(uint32_t tcol, const float* bias, int cb, int m,
                                        uint8_t* slot, bool relu) {
  const uint32_t srow = (uint32_t)m * 128u, sx = (uint32_t)m & 7u;
  uint32_t v[2][16];
  tmem_ld16(tcol, v[0]);
  tmem_ld16(tcol + 16, v[1]);
  tmem_ld_wait_regs(v[0]);
  tmem_ld_wait_regs(v[1]);
#pragma unroll
  for (int c = 0; c < 2; ++c) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int chunk = cb * 4 + c * 2 + q;                 // 16-byte piece of the row
      uint4* piece = reinterpret_cast<uint4*>(slot + srow + ((((uint32_t)chunk) ^ sx) << 4));
      const float4 b0 = *reinterpret_cast<const float4*>(bias + chunk * 8);
      const float4 b1 = *reinterpret_cast<const float4*>(bias + chunk * 8 + 4);
      const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
      float f[8];
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        const float2 r = __fadd2_rn(make_float2(__uint_as_float(v[c][q * 8 + j]),
                                                __uint_as_float(v[c][q * 8 + j + 1])),
                                    make_float2(bb[j], bb[j + 1]));
        f[j] = r.x;
        f[j + 1] = r.y;
      }
      if constexpr (RES) {
        // residual (bf16 -> f32 is exact) added to the f32 result, one
        // rounding at the store: the reference order of kernels.py:185-197
        const uint4 rv = *piece;
        const uint32_t* rr = reinterpret_cast<const uint32_t*>(&rv);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 s2 = __fadd2_rn(make_float2(f[2 * e], f[2 * e + 1]),
                                       make_float2(__uint_as_float(rr[e] << 16),
                                                   __uint_as_float(rr[e] & 0xFFFF0000u)));
          f[2 * e] = s2.x;
          f[2 * e + 1] = s2.y;
        }
      }
      uint4 packed;
      uint32_t* h = reinterpret_cast<uint32_t*>(&packed);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (relu)
          asm("cvt.rn.relu.bf16x2.f32 %0, %2, %1;" : "=r"(h[e]) : "f"(f[2 * e]), "f"(f[2 * e + 1]));
        else
          asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(h[e]) : "f"(f[2 * e]), "f"(f[2 * e + 1]));
      }
      *piece = packed;
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1) junction_kernel(const __grid_constant__ JunctionParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t pad = (1024u - (sraw & 1023u)) & 1023u;
  uint8_t* gbase = smem_raw + pad;
  // layout: ring1 (A1 16 KB | B1 16 KB per stage) | ring2 (N2 x 128 B per
  // stage) | 4 slots (2 chunk buffers x 2 blocks) | barriers
  const uint32_t sR1 = sraw + pad;
  const uint32_t s1 = 2u * kSlot;
  const uint32_t sR2 = sR1 + p.stages1 * s1;
  const uint32_t s2 = (uint32_t)p.N2 * 128u;
  const uint32_t sSl = sR2 + p.stages2 * s2;
  const uint32_t sBar = sSl + 4u * kSlot;
  auto full1 = [&](int i) { return sBar + 8u * i; };          // 8 max
  auto empty1 = [&](int i) { return sBar + 64u + 8u * i; };
  auto full2 = [&](int i) { return sBar + 128u + 8u * i; };
  auto empty2 = [&](int i) { return sBar + 192u + 8u * i; };
  auto d1full = [&](int b) { return sBar + 256u + 8u * b; };
  auto d1empty = [&](int b) { return sBar + 272u + 8u * b; };
  auto a2full = [&](int b) { return sBar + 288u + 8u * b; };
  auto a2empty = [&](int b) { return sBar + 304u + 8u * b; };
  auto rbar = [&](int b) { return sBar + 320u + 8u * b; };
  const uint32_t d2full = sBar + 336u, d2empty = sBar + 344u;
  const uint32_t tslot = sBar + 352u;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&p.tmX);
    tma_prefetch_desc(&p.tmW1);
    tma_prefetch_desc(&p.tmW2);
    tma_prefetch_desc(&p.tmY1);
    tma_prefetch_desc(&p.tmY2);
    if (p.has_res) tma_prefetch_desc(&p.tmR);
    for (int i = 0; i < p.stages1; ++i) {
      mbar_init(full1(i), 1);
      mbar_init(empty1(i), 1);
    }
    for (int i = 0; i < p.stages2; ++i) {
      mbar_init(full2(i), 1);
      mbar_init(empty2(i), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(d1full(b), 1);
      mbar_init(d1empty(b), kEpiWarps);
      mbar_init(a2full(b), 1);
      mbar_init(a2empty(b), 1);
      mbar_init(rbar(b), 1);
    }
    mbar_init(d2full, 1);
    mbar_init(d2empty, kEpiWarps);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(tslot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(gbase + (tslot - sR1));
  neo_pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- producer ----------------
      neo_pdl_wait();
      int st1 = 0, st2 = 0;
      uint32_t ph1 = 0, ph2 = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int n0, h0, w0;
        tile_origin(p, t, n0, h0, w0);
        for (int c = 0; c < p.chunks; ++c) {
          for (int k = 0; k < p.k1; ++k) {
            mbar_wait(empty1(st1), ph1 ^ 1u);
            mbar_arrive_expect_tx(full1(st1), p.tx_a1 + p.tx_b1);
            const uint32_t dst = sR1 + st1 * s1;
            tma_load_5d(dst, &p.tmX, full1(st1), 0, w0, h0, k, n0);
            tma_load_3d(dst + kSlot, &p.tmW1, full1(st1), 0, c * kChunk, k);
            if (++st1 == p.stages1) {
              st1 = 0;
              ph1 ^= 1u;
            }
          }
          for (int j = 0; j < 2; ++j) {
            mbar_wait(empty2(st2), ph2 ^ 1u);
            mbar_arrive_expect_tx(full2(st2), p.tx_b2);
            tma_load_3d(sR2 + st2 * s2, &p.tmW2, full2(st2), 0, 0, 2 * c + j);
            if (++st2 == p.stages2) {
              st2 = 0;
              ph2 ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      const uint32_t idesc1 = umma_idesc(1u, kTileM, kChunk);
      const uint32_t idesc2 = umma_idesc(1u, kTileM, p.N2);
      const uint32_t d2 = tmem + 2u * kChunk;
      int st1 = 0, st2 = 0;
      uint32_t ph1 = 0, ph2 = 0;
      uint32_t gc = 0;          // global chunk counter (buffer = gc & 1)
      uint32_t tcount = 0;
      // GEMM2 of chunk `g2` (global index), issued one chunk behind GEMM1
      auto gemm2 = [&](uint32_t g, bool first) {
        const int b = (int)(g & 1u);
        mbar_wait(a2full(b), (g >> 1) & 1u);
        tc_fence_after();
        for (int j = 0; j < 2; ++j) {
          mbar_wait(full2(st2), ph2);
          tc_fence_after();
          mma_slice(d2, sSl + (uint32_t)(2 * b + j) * kSlot, sR2 + st2 * s2, idesc2,
                    (first && j == 0) ? 0u : 1u);
          umma_commit(empty2(st2));
          if (++st2 == p.stages2) {
            st2 = 0;
            ph2 ^= 1u;
          }
        }
        umma_commit(a2empty(b));
      };
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++tcount) {
        const uint32_t gc0 = gc;
        for (int c = 0; c < p.chunks; ++c, ++gc) {
          const int b = (int)(gc & 1u);
          mbar_wait(d1empty(b), ((gc >> 1) & 1u) ^ 1u);    // epilogue drained this buffer
          tc_fence_after();
          const uint32_t d1 = tmem + (uint32_t)b * kChunk;
          for (int k = 0; k < p.k1; ++k) {
            mbar_wait(full1(st1), ph1);
            tc_fence_after();
            mma_slice(d1, sR1 + st1 * s1, sR1 + st1 * s1 + kSlot, idesc1, k ? 1u : 0u);
            umma_commit(empty1(st1));
            if (++st1 == p.stages1) {
              st1 = 0;
              ph1 ^= 1u;
            }
          }
          umma_commit(d1full(b));
          if (c == 0) {
            // D2 of the previous tile must have been drained before GEMM2(0)
            mbar_wait(d2empty, (tcount & 1u) ^ 1u);
            tc_fence_after();
          } else {
            gemm2(gc - 1, c - 1 == 0);
          }
        }
        gemm2(gc - 1, p.chunks == 1);
        umma_commit(d2full);
        (void)gc0;
      }
    }
  } else {
    // ---------------- epilogue (16 warps) ----------------
    const int e = warp - 2;
    const int q = warp & 3;               // TMEM lane quarter
    const int part = e >> 2;              // which 32 of a chunk's 128 columns
    const int half = part >> 1;           // channel block within the chunk
    const int cb = part & 1;              // 32-column half of that block
    const int m = q * 32 + lane;          // pixel row of the tile
    const bool leader = e == 0 && lane == 0;
    float* sb1 = reinterpret_cast<float*>(gbase + (sSl - sR1) + 4 * kSlot + 512);
    float* sb2 = sb1 + p.N1;
    neo_pdl_wait();
    // biases staged once per CTA (zeros when absent)
    for (int i = e * 32 + lane; i < p.N1 + p.N2; i += kEpiWarps * 32) {
      const bool first = i < p.N1;
      const float* src = first ? p.b1 : p.b2;
      sb1[i] = src ? __ldg(src + (first ? i : i - p.N1)) : 0.f;
    }
    named_bar_sync(1, kEpiWarps * 32);
    uint32_t gc = 0, tcount = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++tcount) {
      int n0, h0, w0;
      tile_origin(p, t, n0, h0, w0);
      for (int c = 0; c < p.chunks; ++c, ++gc) {
        const int b = (int)(gc & 1u);
        const uint32_t ph = (gc >> 1) & 1u;
        if (leader) {
          // the chunk buffer's slots: GEMM2 of two chunks ago is done with
          // them, and at most one later store group (the previous chunk's)
          // may still be reading shared memory
          mbar_wait(a2empty(b), ph ^ 1u);
          // the previous tile's y2 store used every slot: wait for all reads
          if (c == 0) bulk_wait_read<0>();
          else bulk_wait_read<1>();
          if (p.has_res) {
            mbar_arrive_expect_tx(rbar(b), 2u * p.box_bytes);
            for (int j = 0; j < 2; ++j)
              tma_load_5d(sSl + (uint32_t)(2 * b + j) * kSlot, &p.tmR, rbar(b), 0, w0, h0,
                          2 * c + j, n0);
          }
        }
        mbar_wait(d1full(b), ph);
        tc_fence_after();
        if (p.has_res) mbar_wait(rbar(b), ph);
        else {
          // no residual: the slot must still be free (leader waited above)
          named_bar_sync(1, kEpiWarps * 32);
        }
        uint8_t* slot = gbase + (sSl - sR1) + (uint32_t)(2 * b + half) * kSlot;
        const uint32_t tcol = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)b * kChunk + part * 32;
        const float* bias = sb1 + c * kChunk + half * 64;
        if (p.has_res) drain32<true>(tcol, bias, cb, m, slot, p.relu1);
        else drain32<false>(tcol, bias, cb, m, slot, p.relu1);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(d1empty(b));
        fence_proxy_async_smem();              // generic writes -> TMA store / MMA reads
        named_bar_sync(1, kEpiWarps * 32);
        if (leader) {
          for (int j = 0; j < 2; ++j)
            tma_store_5d(&p.tmY1, sSl + (uint32_t)(2 * b + j) * kSlot, 0, w0, h0, 2 * c + j, n0);
          bulk_commit();
          mbar_arrive(a2full(b));
        }
      }
      // ---- reduce output: D2 -> +b2 -> relu -> bf16 -> y2 (through the slots)
      mbar_wait(d2full, tcount & 1u);
      tc_fence_after();
      if (leader) bulk_wait_read<0>();          // y1 stores left every slot
      named_bar_sync(1, kEpiWarps * 32);
      const int nb2 = p.N2 / 64;
      for (int pc = part; pc < 2 * nb2; pc += 4) {         // 32-column pieces
        const int blk = pc >> 1;
        uint8_t* slot = gbase + (sSl - sR1) + (uint32_t)blk * kSlot;
        const uint32_t tcol = tmem + ((uint32_t)(q * 32) << 16) + 2u * kChunk + pc * 32;
        drain32<false>(tcol, sb2 + blk * 64, pc & 1, m, slot, p.relu2);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(d2empty);
      fence_proxy_async_smem();
      named_bar_sync(1, kEpiWarps * 32);
      if (leader) {
        for (int blk = 0; blk < nb2; ++blk)
          tma_store_5d(&p.tmY2, sSl + (uint32_t)blk * kSlot, 0, w0, h0, blk, n0);
        bulk_commit();
      }
    }
    if (leader) bulk_wait_read<0>();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
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

// M-tile geometry maximising useful rows of the 128-row tile (same rule as
// the conv kernel's picker)
void pick_geometry(int64_t N, int64_t OH, int64_t OW, int& BW, int& BH, int& BNI) {
  double best = -1.0;
  BW = BH = BNI = 1;
  for (int bw = 1; bw <= std::min<int64_t>(OW, kTileM); ++bw)
    for (int bh = 1; bh <= std::min<int64_t>(OH, kTileM / bw); ++bh)
      for (int bni = 1; bni <= std::min<int64_t>(N, kTileM / (bw * bh)); ++bni) {
        const double tiles = (double)neo_ceil_div(OW, bw) * neo_ceil_div(OH, bh) * neo_ceil_div(N, bni);
        const double eff = (double)N * OH * OW / (tiles * kTileM);
        if (eff > best + 1e-9 ||
            (eff > best - 1e-9 && (bw > BW || (bw == BW && bw * bh * bni > BW * BH * BNI)))) {
          best = eff;
          BW = bw;
          BH = bh;
          BNI = bni;
        }
      }
}

}  // namespace

extern "C" int neo_conv_junction(const void* x, const void* w1, const float* b1,
                                 const void* residual, void* y1, const void* w2, const float* b2,
                                 void* y2, int64_t n, int64_t c1, int64_t h, int64_t w, int64_t n1,
                                 int64_t n2, int relu1, int relu2, neo_stream_t stream) {
  NEO_CHECK_ARG(x && w1 && y1 && w2 && y2, NEO_ERR_INVALID_ARG, "null tensor pointer");
  NEO_CHECK_ARG(n >= 1 && h >= 1 && w >= 1, NEO_ERR_SHAPE_MISMATCH, "empty junction input");
  NEO_CHECK_ARG(c1 % 64 == 0 && c1 >= 64 && n1 % kChunk == 0 && n2 % 64 == 0 && n2 >= 64 &&
                    n2 <= 256,
                NEO_ERR_UNSUPPORTED,
                "junction needs C1 %% 64 == 0, N1 %% 128 == 0, N2 in {64, 128, 192, 256} "
                "(C1=%lld N1=%lld N2=%lld)", (long long)c1, (long long)n1, (long long)n2);
  auto encode = encode_fn();
  NEO_CHECK_ARG(encode != nullptr, NEO_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  JunctionParams kp;
  memset(&kp, 0, sizeof(kp));
  pick_geometry(n, h, w, kp.BW, kp.BH, kp.BNI);
  const CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  auto map5 = [&](CUtensorMap* m, const void* base, int64_t cb) {
    cuuint64_t dims[5] = {64, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)cb, (cuuint64_t)n};
    cuuint64_t strides[4] = {128, (cuuint64_t)w * 128, (cuuint64_t)h * w * 128,
                             (cuuint64_t)cb * h * w * 128};
    cuuint32_t box[5] = {64, (cuuint32_t)kp.BW, (cuuint32_t)kp.BH, 1, (cuuint32_t)kp.BNI};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    return encode(m, dt, 5, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  auto map3 = [&](CUtensorMap* m, const void* base, int64_t k, int64_t slices, int rows) {
    cuuint64_t dims[3] = {64, (cuuint64_t)k, (cuuint64_t)slices};
    cuuint64_t strides[2] = {128, (cuuint64_t)k * 128};
    cuuint32_t box[3] = {64, (cuuint32_t)rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return encode(m, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  CUresult r = map5(&kp.tmX, x, c1 / 64);
  NEO_CHECK_ARG(r == CUDA_SUCCESS, NEO_ERR_CUDA, "junction map X failed (%d)", (int)r);
  r = map3(&kp.tmW1, w1, n1, c1 / 64, kChunk);
  NEO_CHECK_ARG(r == CUDA_SUCCESS, NEO_ERR_CUDA, "junction map W1 failed (%d)", (int)r);
  r = map3(&kp.tmW2, w2, n2, n1 / 64, (int)n2);
  NEO_CHECK_ARG(r == CUDA_SUCCESS, NEO_ERR_CUDA, "junction map W2 failed (%d)", (int)r);
  r = map5(&kp.tmY1, y1, n1 / 64);
  NEO_CHECK_ARG(r == CUDA_SUCCESS, NEO_ERR_CUDA, "junction map Y1 failed (%d)", (int)r);
  r = map5(&kp.tmY2, y2, n2 / 64);
  NEO_CHECK_ARG(r == CUDA_SUCCESS, NEO_ERR_CUDA, "junction map Y2 failed (%d)", (int)r);
  if (residual) {
    r = map5(&kp.tmR, residual, n1 / 64);
    NEO_CHECK_ARG(r == CUDA_SUCCESS, NEO_ERR_CUDA, "junction map R failed (%d)", (int)r);
  }
  kp.b1 = b1;
  kp.b2 = b2;
  kp.N = (int)n;
  kp.H = (int)h;
  kp.W = (int)w;
  kp.C1 = (int)c1;
  kp.N1 = (int)n1;
  kp.N2 = (int)n2;
  kp.tiles_w = (int)neo_ceil_div(w, kp.BW);
  kp.tiles_h = (int)neo_ceil_div(h, kp.BH);
  const int64_t tiles = (int64_t)kp.tiles_w * kp.tiles_h * neo_ceil_div(n, kp.BNI);
  NEO_CHECK_ARG(tiles < (1ll << 31), NEO_ERR_UNSUPPORTED, "too many junction tiles");
  kp.num_tiles = (int)tiles;
  kp.k1 = (int)(c1 / 64);
  kp.chunks = (int)(n1 / kChunk);
  kp.relu1 = relu1;
  kp.relu2 = relu2;
  kp.has_res = residual != nullptr;
  kp.box_bytes = (uint32_t)(kp.BW * kp.BH * kp.BNI * 128);
  kp.tx_a1 = kp.box_bytes;
  kp.tx_b1 = kChunk * 128;
  kp.tx_b2 = (uint32_t)n2 * 128;
  // shared memory: 4 slots + as many ring stages as fit (ring 2 holds W2
  // slices, two per chunk; ring 1 the x / W1 slice pairs)
  const int64_t fixed = 1024 + 4 * kSlot + 512 + (n1 + n2) * 4;
  const int64_t s1 = 2 * kSlot, s2 = n2 * 128;
  int st2 = 4, st1 = 4;
  auto need = [&]() { return fixed + st1 * s1 + st2 * s2; };
  while (need() > kSmemBudget && st2 > 2) --st2;
  while (need() > kSmemBudget && st1 > 2) --st1;
  NEO_CHECK_ARG(need() <= kSmemBudget, NEO_ERR_UNSUPPORTED, "junction tile does not fit");
  kp.stages1 = st1;
  kp.stages2 = st2;
  const size_t smem = (size_t)need();
  static bool attr_done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_done[dev & 63]) {
    NEO_CUDA_TRY(cudaFuncSetAttribute(junction_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kSmemBudget));
    attr_done[dev & 63] = true;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>(tiles, sms);
  neo_launch(junction_kernel, dim3(grid), dim3(kThreads), smem, static_cast<cudaStream_t>(stream), kp);
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}
