// K-CONV: NCHW[x]c convolution as a tcgen05/TMEM implicit GEMM.
//
// Replaces conv_blocked (reference kernels.py:250-303, hot loop _blocked_rows
// :135-198) for NEO_MODE_BF16 / NEO_MODE_TF32 / NEO_MODE_FP8 (e4m3 x e4m3
// through tcgen05 kind::f8f6f4: the same byte geometry as bf16 -- a K step
// is 32 bytes of a 128-byte swizzled row either way -- so the operand
// pipeline is shared and only the instruction kind and the epilogue's
// storage conversion differ).
//
// GEMM view:  M = output pixels (n, oh, ow), N = output channels k,
//             K = (r, s, c) reduction.
// The K loop walks "slices": one slice = one (r, s, input-channel-block) triple
// = x channels.  In NCHW[x]c a slice of the input for an M tile is a
// (BNI images x BH rows x BW cols x x lanes) box that TMA fetches with zero
// fill for the padding halo (negative / past-the-end coordinates) and with
// traversal strides for stride-2 convs, so no padded copy is ever made
// (reference _pad_nchwc :211-218 disappears).  x*sizeof(elem) is exactly the
// swizzle span (16/32/64/128 B), so each slice lands as a K-major UMMA
// sub-tile of 128 rows without any reshuffle.  Weights use a device-private
// slice-major image (R, S, C/x, K, x) so B sub-tiles have the same shape.
//
// Warp roles (192 threads, persistent over output tiles):
//   warp 0     : TMA producer (one lane)     smem ring full/empty mbarriers
//   warp 1     : TMEM alloc + MMA issuer     double-buffered TMEM accumulator
//   warps 2..5 : epilogue (TMEM lane quarter = warp % 4): tcgen05.ld, then
//                scale/shift -> bias -> residual -> relu (kernels.py:185-197)
//                in registers, stored straight into NCHW[y]c (optionally into
//                a channel-block window of a concat buffer).
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "neo_common.cuh"

namespace {

constexpr int kMaxStages = 8;
// operand kinds (template parameter KIND): tcgen05.mma .kind and idesc format
// kKindBF16Q: bf16 operands writing e4m3 (an image stem entering an fp8
// chain) -- a separate instantiation so the hot bf16 kernel carries no e4m3
// epilogue code (its size costs the bf16 step ~1% in I-cache pressure)
enum { kKindBF16 = 0, kKindTF32 = 1, kKindFP8 = 2, kKindBF16Q = 3 };
// epilogue storage types (template parameter OUT of epi_block_tma)
enum { kOutBF16 = 0, kOutF32 = 1, kOutFP8 = 2 };
constexpr int kThreads = 576;   // warp 0 TMA, warp 1 MMA, warps 2-17 epilogue (2 groups of 8)
constexpr int kEpiWarps = 16;          // warps 2..17
constexpr int kProWarps = 8;           // prologue mode: warps 10..17 rewrite A slices
constexpr int kMaxGroups = 4;          // epilogue groups = TMEM accumulator stages
constexpr int kTileM = 128;
#ifdef NEO_TRACE
constexpr int kSmemBudget = 226 * 1024;   // trace builds keep a little static smem
#else
constexpr int kSmemBudget = 227 * 1024;
#endif

struct ConvTCParams {
  CUtensorMap tmA;  // 5-D: (x, W, H, Cb, N)
  CUtensorMap tmB;  // 3-D: (x, K, slices)
  CUtensorMap tmO;  // 5-D output store map: (y, OW, OH, Kb_total, N)   (tma_epi)
  CUtensorMap tmR;  // 5-D residual load map, same geometry              (tma_epi)
  CUtensorMap tmO2; // second output (k_split > 0), same geometry      (tma_epi)
  int N, OH, OW, K;
  int BW, BH, BNI, BN;
  int BWo;       // output columns a tile advances by: BW, or BW - (S-1) for halo strips
  int tiles_w, tiles_h, tiles_k;
  int num_tiles;
  int G, kstages, Cb, S, nslices;
  int stride_h, stride_w, pad_h, pad_w;
  int rowb;      // x * sizeof(elem)
  int swz;       // UMMA layout code for rowb
  int stages;
  uint32_t a_sub, b_sub, a_stage, b_stage, tx_bytes, tmem_cols;
  // epilogue groups (2 or 4): group g drains TMEM accumulator stage g; each
  // group has kEpiWarps / ngroups warps covering the 4 TMEM lane quarters
  int ngroups;
  const float* scale;
  const float* shift;
  const float* bias;
  const void* res;
  void* out;
  int y, out_cb_off, out_cb_total, res_cb_off, res_cb_total;
  int relu, out_f32, round_tf32;
  int k_split, relu2, out2_cb_off;   // channels >= k_split -> tmO2 (0: one output)
  int out_kind;       // kOutBF16 / kOutF32 / kOutFP8 (the residual has the same type)
  // e4m3 storage: residual value = e4m3(q) * res_scale; stored output
  // q = e4m3_rn_satfinite(v * out_qscale) (out2_qscale for the second output)
  float res_scale, out_qscale, out2_qscale;
  int tma_epi;        // stage output blocks in smem and store them with TMA
  int rowb_out;       // y * sizeof(out elem) for the TMA epilogue
  uint32_t stage_out; // bytes of one staging buffer (128 rows * rowb_out)
  uint32_t out_box_bytes;
  int nslot;          // staging slots per epilogue group (tma_epi)
  // residual prefetch (tma_epi with a residual, nslot >= 2 * blocks per
  // tile): a group's slots form two sets used by alternate tiles; right
  // after a tile's store is committed the group issues the residual loads of
  // its next tile into the other set, so their HBM latency overlaps this
  // tile's store drain and the next accumulator wait
  int res_pf;
  // halo mode (stride-1 convs): tiles span the padded output width
  // BW = OW + S - 1; a pipeline slice is one (kernel row r, channel block)
  // input band, loaded once; the S horizontal taps read it through
  // descriptors shifted by s rows; B holds the S weight slices of the pair.
  int halo;
  int R;
  int halo_baseoff;   // set the UMMA matrix base offset for shifted views
  // split-K: work unit u = (tile u / splits, split u % splits) covers k-stages
  // [split * kps, min(kstages, (split + 1) * kps)); with splits > 1 every
  // unit stores its raw fp32 accumulator to ws[u][chunk16][row][16] and,
  // after all splits of the tile arrived, reduces and finishes 1/splits of it.
  int splits, kps, num_units;
  // CTA pair (cta_group::2): the two CTAs of a cluster own the two 128-row
  // halves of a 256-row M tile and the two halves of its N tile; the leader
  // (rank 0) issues M=256 MMAs reading both CTAs' shared memory, so every
  // weight byte fetched serves 256 output pixels.  Group g -> N tile
  // g % tiles_k, M tiles 2 * (g / tiles_k) + rank (a missing odd tile is a
  // dummy: loads out of bounds, stores clipped).
  int pair, tiles_m, num_groups;
  // BN-ReLU prologue (DenseNet pre-activation fused into a 1x1 conv): warps
  // 10-17 rewrite every landed activation slice in shared memory as
  // relu(x * pro_scale[c] + pro_shift[c]) before the MMA may read it (the
  // MMA waits on xfull barriers); the epilogue keeps warps 2-9
  const float* pro_scale;
  const float* pro_shift;
  int pro, pro_relu;
  // weight-stationary: every CTA's tiles share one N block (grid % tiles_k
  // == 0), whose whole weight image (b_region bytes) is loaded into shared
  // memory once; the stage ring then carries only activations.  Halo tiles
  // load one band per channel block covering all R rows (kernel row r = the
  // band view shifted by r*BW rows), so a stage feeds R*S taps.
  int wst;
  uint32_t b_region;
  int static_w;     // NEO_FLAG_STATIC_WEIGHTS: weight image fetched before griddepcontrol.wait
  int dbg;          // NEOB200_DBG timing experiments (1: no epilogue work, 2: no A loads,
                    // 8: per-CTA MMA-loop clocks -> neo_dbg_clk)
  float* ws;        // partials
  int* counters;    // per-tile arrival counters (zero between launches)
  // last-tile sharing (TMA epilogue, single-CTA tiles, unsplit): the CTA's
  // final tile is drained by two epilogue groups, each taking half of its
  // output channel blocks -- nothing else is left for the idle group to do,
  // and the last epilogue is the launch's tail
  int share_last;
  int epi_warps;      // epilogue warps of this launch: 16, or 8 in half-SM mode (320 threads)
  int dbg_slot;     // NEOB200_DBG & 256: per-launch timeline slot (g_tl)
};

__device__ __forceinline__ void decode_tile(const ConvTCParams& p, int t, int& n0, int& oh0,
                                            int& ow0, int& k0) {
  // unsigned, three divisions (every epilogue thread decodes every tile:
  // signed div/mod pairs were ~7% of the kernel's instructions)
  const uint32_t ut = (uint32_t)t, tk = (uint32_t)p.tiles_k, tw = (uint32_t)p.tiles_w,
                 th = (uint32_t)p.tiles_h;
  const uint32_t mt = ut / tk;
  const uint32_t kt = ut - mt * tk;
  const uint32_t q2 = mt / tw;
  const uint32_t wi = mt - q2 * tw;
  const uint32_t ni = q2 / th;
  const uint32_t hi = q2 - ni * th;
  n0 = (int)ni * p.BNI;
  oh0 = hi * p.BH;
  ow0 = wi * p.BWo;
  k0 = kt * p.BN;
}

// i-th work unit of this CTA, or -1 when done
__device__ __forceinline__ int cta_unit(const ConvTCParams& p, int i, int rank) {
  if (!p.pair) {
    const int u = (int)blockIdx.x + i * (int)gridDim.x;
    return u < p.num_units ? u : -1;
  }
  const int g = (int)blockIdx.x / 2 + i * ((int)gridDim.x / 2);
  if (g >= p.num_groups) return -1;
  const int kt = g % p.tiles_k;
  const int tm = (g / p.tiles_k) * 2 + rank;
  return tm * p.tiles_k + kt;
}

struct EpiAccess {
  size_t out_base, res_base;  // element offsets of channel block 0 for this pixel
  size_t plane;               // OH*OW*y elements per channel block
};

__device__ __forceinline__ float epi_apply(const ConvTCParams& p, float v, int k) {
  if (p.scale) v = fmaf(v, __ldg(p.scale + k), p.shift ? __ldg(p.shift + k) : 0.f);
  else if (p.shift) v = v + __ldg(p.shift + k);
  if (p.bias) v = v + __ldg(p.bias + k);
  return v;
}

__device__ __forceinline__ float epi_finish(const ConvTCParams& p, float v) {
  if (p.relu) v = fmaxf(v, 0.f);
  if (p.round_tf32) v = neo_round_tf32(v);
  return v;
}

// 16 accumulator columns [kbase, kbase+16) of one output pixel
__device__ __forceinline__ void epi_chunk(const ConvTCParams& p, const uint32_t (&v)[16],
                                          int kbase, const EpiAccess& ea) {
  float f[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) f[j] = __uint_as_float(v[j]);

  if ((p.y & 15) == 0 && kbase + 16 <= p.K) {
    // whole chunk inside one output channel block: vector path
    const int kb = kbase / p.y, j0 = kbase % p.y;
#pragma unroll
    for (int j = 0; j < 16; ++j) f[j] = epi_apply(p, f[j], kbase + j);
    if (p.out_f32) {
      if (p.res) {
        const float4* r4 = reinterpret_cast<const float4*>(
            static_cast<const float*>(p.res) + ea.res_base + (size_t)kb * ea.plane + j0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float4 rv = __ldg(r4 + q);
          f[4 * q + 0] += rv.x;
          f[4 * q + 1] += rv.y;
          f[4 * q + 2] += rv.z;
          f[4 * q + 3] += rv.w;
        }
      }
      float4* o4 = reinterpret_cast<float4*>(static_cast<float*>(p.out) + ea.out_base +
                                             (size_t)kb * ea.plane + j0);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        o4[q] = make_float4(epi_finish(p, f[4 * q]), epi_finish(p, f[4 * q + 1]),
                            epi_finish(p, f[4 * q + 2]), epi_finish(p, f[4 * q + 3]));
    } else {
      if (p.res) {
        const uint4* r4 = reinterpret_cast<const uint4*>(
            static_cast<const __nv_bfloat16*>(p.res) + ea.res_base + (size_t)kb * ea.plane + j0);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          uint4 rv = __ldg(r4 + q);
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&rv);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float2 t = __bfloat1622float2(h2[e]);
            f[8 * q + 2 * e] += t.x;
            f[8 * q + 2 * e + 1] += t.y;
          }
        }
      }
      uint4 packed[2];
      __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(packed);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        h2[e] = __floats2bfloat162_rn(epi_finish(p, f[2 * e]), epi_finish(p, f[2 * e + 1]));
      uint4* o4 = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + ea.out_base +
                                           (size_t)kb * ea.plane + j0);
      o4[0] = packed[0];
      o4[1] = packed[1];
    }
    return;
  }
  // generic path: any y, partial chunk at the end of K (fully unrolled so
  // f[] stays in registers)
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int k = kbase + j;
    if (k >= p.K) continue;
    const int kb = k / p.y, jj = k % p.y;
    float val = epi_apply(p, f[j], k);
    const size_t o = ea.out_base + (size_t)kb * ea.plane + jj;
    if (p.out_f32) {
      if (p.res) val += static_cast<const float*>(p.res)[ea.res_base + (size_t)kb * ea.plane + jj];
      static_cast<float*>(p.out)[o] = epi_finish(p, val);
    } else {
      if (p.res)
        val += __bfloat162float(
            static_cast<const __nv_bfloat16*>(p.res)[ea.res_base + (size_t)kb * ea.plane + jj]);
      static_cast<__nv_bfloat16*>(p.out)[o] = __float2bfloat16_rn(epi_finish(p, val));
    }
  }
}

// Epilogue of one output channel block (y columns) staged through shared
// memory: TMEM -> registers -> (+ residual from the smem tile the TMA load
// brought in) -> swizzled smem row -> TMA store of the whole block.
// Per-column epilogue vectors of a 16-column chunk, loaded as broadcast
// float4s (every thread of the warp reads the same addresses); absent vectors
// become the identity so the per-element math is branch-free:
//   v = fma(v, scale, shift) ; v += bias ; v += residual ; v = max(v, floor)
// (floor = 0 for relu, -inf otherwise) -- the reference order of
// kernels.py:185-197 with one rounding per reference operation.
// The tile's per-column epilogue vectors live in shared memory (staged once
// per tile by the epilogue group, identity values for absent vectors), so the
// per-element math is branch-free and no global load sits on its path:
//   v = fma(v, scale, shift) ; v += bias ; v += residual ; v = max(v, floor)
// (floor = 0 for relu, -inf otherwise) -- the reference order of
// kernels.py:185-197 with one rounding per reference operation.
constexpr int kParamFloats = 3 * 256;   // scale | shift | bias for BN <= 256

// One output channel block (y columns) of one pixel row: TMEM -> registers ->
// epilogue -> swizzled smem row (which already holds the residual block when
// HAS_RES).  OUT selects f32 / bf16 / e4m3 storage (qs = 1 / output scale
// for e4m3).
template <int OUT, bool HAS_RES, bool AFFINE>
__device__ __forceinline__ void epi_block_tma(const ConvTCParams& p, uint32_t tcol, int col0,
                                              int m, uint8_t* sbuf_gen, const float* par,
                                              float relu_floor, bool round, int c_begin,
                                              int c_step, float qs) {
  constexpr bool OUT_F32 = OUT == kOutF32;
  const int nchunk = p.y / 16;  // 16-column TMEM loads
  constexpr int kChunks16 = OUT_F32 ? 4 : OUT == kOutBF16 ? 2 : 1;   // 16-byte pieces per 16 values
  // swz_offset(m, chunk, rowb) hoisted: the row's base and its XOR pattern
  // are fixed per thread (chunk * 16 < rowb keeps o >> 7 == base >> 7)
  const uint32_t srow = (uint32_t)m * (uint32_t)p.rowb_out;
  const uint32_t smask = p.rowb_out == 128 ? 7u : p.rowb_out == 64 ? 3u : p.rowb_out == 32 ? 1u : 0u;
  const uint32_t sxr = (srow >> 7) & smask;
  // one chunk: 16 accumulator columns of row m -> scale/shift/bias
  // (+ residual from the slot) -> relu -> the swizzled staging slot
  auto finish = [&](const uint32_t (&v)[16], int c) {
    const int col = col0 + c * 16;
    constexpr int kPer = 16 / kChunks16;   // values per 16-byte staging piece
#pragma unroll
    for (int q = 0; q < kChunks16; ++q) {
      // parameters of this piece only (keeps the live register set small)
      float f[kPer];
#pragma unroll
      for (int j4 = 0; j4 < kPer / 4; ++j4) {
        const int cc = col + q * kPer + 4 * j4;
        const float4 bi = *reinterpret_cast<const float4*>(par + 512 + cc);
        const float* vv = reinterpret_cast<const float*>(v) + q * kPer + 4 * j4;
        // packed f32x2 FMA / add (FFMA2 / FADD2): the same IEEE RN operations
        // as the scalar forms, half the instructions
        const float2 v01 = make_float2(vv[0], vv[1]), v23 = make_float2(vv[2], vv[3]);
        const float2 b01 = make_float2(bi.x, bi.y), b23 = make_float2(bi.z, bi.w);
        float2 r01, r23;
        if constexpr (AFFINE) {
          const float4 sc = *reinterpret_cast<const float4*>(par + cc);
          const float4 sh = *reinterpret_cast<const float4*>(par + 256 + cc);
          r01 = __fadd2_rn(__ffma2_rn(v01, make_float2(sc.x, sc.y), make_float2(sh.x, sh.y)), b01);
          r23 = __fadd2_rn(__ffma2_rn(v23, make_float2(sc.z, sc.w), make_float2(sh.z, sh.w)), b23);
        } else {
          // identity scale/shift: fma(v, 1, 0) == v, so this is the same value
          r01 = __fadd2_rn(v01, b01);
          r23 = __fadd2_rn(v23, b23);
        }
        f[4 * j4 + 0] = r01.x;
        f[4 * j4 + 1] = r01.y;
        f[4 * j4 + 2] = r23.x;
        f[4 * j4 + 3] = r23.y;
      }
      const uint32_t off = srow + ((((uint32_t)(c * kChunks16 + q)) ^ sxr) << 4);
      uint4* slot = reinterpret_cast<uint4*>(sbuf_gen + off);
      if constexpr (OUT_F32) {
        float o[4];
        float4 rv = HAS_RES ? *reinterpret_cast<float4*>(slot) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float r4[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float t = f[j];
          if constexpr (HAS_RES) t += r4[j];
          t = fmaxf(t, relu_floor);
          o[j] = round ? neo_round_tf32(t) : t;
        }
        *reinterpret_cast<float4*>(slot) = make_float4(o[0], o[1], o[2], o[3]);
      } else if constexpr (OUT == kOutFP8) {
        // e4m3 storage: residual bytes widened exactly (e4m3 -> f16 -> f32)
        // and scaled (fma: one rounding, the scales are powers of two), the
        // relu floor, then the output scale and ONE rounding to e4m3
        if constexpr (HAS_RES) {
          const uint4 rv = *slot;
          const uint32_t* r = reinterpret_cast<const uint32_t*>(&rv);
          const float rs = p.res_scale;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const __nv_fp8x2_storage_t pr = (__nv_fp8x2_storage_t)(r[j >> 1] >> (16 * (j & 1)));
            const float2 rf = __half22float2(__half2(__nv_cvt_fp8x2_to_halfraw2(pr, __NV_E4M3)));
            f[2 * j] = fmaf(rf.x, rs, f[2 * j]);
            f[2 * j + 1] = fmaf(rf.y, rs, f[2 * j + 1]);
          }
        }
        uint4 packed;
        uint32_t* h = reinterpret_cast<uint32_t*>(&packed);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 a = make_float2(fmaxf(f[4 * j], relu_floor) * qs,
                                       fmaxf(f[4 * j + 1], relu_floor) * qs);
          const float2 b = make_float2(fmaxf(f[4 * j + 2], relu_floor) * qs,
                                       fmaxf(f[4 * j + 3], relu_floor) * qs);
          h[j] = (uint32_t)__nv_cvt_float2_to_fp8x2(a, __NV_SATFINITE, __NV_E4M3) |
                 ((uint32_t)__nv_cvt_float2_to_fp8x2(b, __NV_SATFINITE, __NV_E4M3) << 16);
        }
        *slot = packed;
      } else {
        // bf16 output in the reference order (kernels.py:185-197): the
        // residual (bf16 -> f32 is exact) is added to the f32 conv result,
        // then ONE rounding to bf16 with the relu fused into the conversion
        // (rounding keeps the sign, so relu(rn(v)) == rn(relu(v)))
        uint4 packed;
        uint32_t* h = reinterpret_cast<uint32_t*>(&packed);
        const bool relu = relu_floor == 0.f;
        if constexpr (HAS_RES) {
          const uint4 rv = *slot;
          const uint32_t* r = reinterpret_cast<const uint32_t*>(&rv);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 rf = make_float2(__uint_as_float(r[j] << 16), __uint_as_float(r[j] & 0xFFFF0000u));
            const float2 s = __fadd2_rn(make_float2(f[2 * j], f[2 * j + 1]), rf);
            f[2 * j] = s.x;
            f[2 * j + 1] = s.y;
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (relu)
            asm("cvt.rn.relu.bf16x2.f32 %0, %2, %1;" : "=r"(h[j]) : "f"(f[2 * j]), "f"(f[2 * j + 1]));
          else
            asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(h[j]) : "f"(f[2 * j]), "f"(f[2 * j + 1]));
        }
        *slot = packed;
      }
    }
  };
#pragma unroll 1
  for (int c = c_begin; c < nchunk; c += c_step) {
    uint32_t v[16];
    tmem_ld16(tcol + c * 16, v);
    tmem_ld_wait_regs(v);
    finish(v, c);
  }
}

// Split-K fixup of one unit's share: (chunk16, row) pairs
// [sp*share, (sp+1)*share) of tile t, each summed over the splits in order
// and finished by the direct epilogue.  Kept out of line so the main
// kernel's register allocation is not shaped by this cold path.
__device__ __noinline__ void splitk_fixup(const ConvTCParams& p, int t, int sp, int n0, int oh0,
                                          int ow0, int k0, int gtid, int gthreads) {
  const int nch = p.BN / 16;
  const int pairs = nch * kTileM;
  const int share = (pairs + p.splits - 1) / p.splits;
  const int pend = min(pairs, (sp + 1) * share);
  const float4* tile_ws = reinterpret_cast<const float4*>(p.ws) +
                          (size_t)t * p.splits * nch * kTileM * 4;
  const size_t sstride = (size_t)nch * kTileM * 4;
  const size_t plane = (size_t)p.OH * p.OW * p.y;
  for (int pi = sp * share + gtid; pi < pend; pi += gthreads) {
    const int c = pi / kTileM, mr = pi % kTileM;
    const int kb0 = k0 + c * 16;
    const int wl = mr % p.BW, hl = (mr / p.BW) % p.BH, nl = mr / (p.BW * p.BH);
    const int ow = ow0 + wl, oh = oh0 + hl, n = n0 + nl;
    if (kb0 >= p.K || mr >= p.BW * p.BH * p.BNI || wl >= p.BWo || ow >= p.OW || oh >= p.OH ||
        n >= p.N)
      continue;
    const float4* src = tile_ws + ((size_t)c * kTileM + mr) * 4;
    float f[16];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 a = __ldcg(src + j);
      f[4 * j] = a.x;
      f[4 * j + 1] = a.y;
      f[4 * j + 2] = a.z;
      f[4 * j + 3] = a.w;
    }
    for (int s2 = 1; s2 < p.splits; ++s2) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float4 a = __ldcg(src + s2 * sstride + j);
        f[4 * j] += a.x;
        f[4 * j + 1] += a.y;
        f[4 * j + 2] += a.z;
        f[4 * j + 3] += a.w;
      }
    }
    uint32_t v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(f[j]);
    EpiAccess ea;
    ea.plane = plane;
    const size_t pix = ((size_t)oh * p.OW + ow) * p.y;
    ea.out_base = (size_t)n * p.out_cb_total * plane + (size_t)p.out_cb_off * plane + pix;
    ea.res_base = (size_t)n * p.res_cb_total * plane + (size_t)p.res_cb_off * plane + pix;
    epi_chunk(p, v, kb0, ea);
  }
}

#ifdef NEO_TRACE
// debug builds only: CTA 0 logs (event, tile, globaltimer) records, one
// region per warp indexed by a shared-memory counter (no global atomics on
// the traced path); counts are published at kernel exit
constexpr int kTraceWarps = 18, kTracePerWarp = 2048;
__device__ unsigned long long g_trace[kTraceWarps * kTracePerWarp];
__device__ unsigned int g_trace_cnt[kTraceWarps];
__device__ __forceinline__ void trace(int ev, int t, unsigned* cnt) {
  if (blockIdx.x != 0) return;
  unsigned long long ns;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
  const int w = threadIdx.x >> 5;
  const unsigned int i = atomicAdd_block(cnt + w, 1u);
  if (i < (unsigned)kTracePerWarp)
    g_trace[w * kTracePerWarp + i] = ((unsigned long long)ev << 56) |
                                     ((unsigned long long)(t & 0xFFFF) << 40) | (ns & 0xFFFFFFFFFFull);
}
#define TRACE(ev, t) trace(ev, t, s_trace_cnt)
#else
#define TRACE(ev, t)
#endif

// NEOB200_DBG & 8: per-CTA (MMA-loop cycles, ns) for clock checks
__device__ unsigned long long g_dbg_clk[8 * 1024];
// NEOB200_DBG & 256: per-launch, per-CTA globaltimer stamps (in-graph
// timelines: entry, past griddepcontrol.wait, first MMA, last commit, exit)
constexpr int kTlSlots = 64, kTlCtas = 160, kTlEv = 5;
__device__ unsigned long long g_tl[kTlSlots * kTlCtas * kTlEv];
__device__ __forceinline__ void tl_stamp(const ConvTCParams& p, int ev) {
  unsigned long long ns;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
  if (blockIdx.x < kTlCtas) g_tl[((p.dbg_slot % kTlSlots) * kTlCtas + blockIdx.x) * kTlEv + ev] = ns;
}

// MMA issue: descriptors are formed by adding small offsets (in 16-byte
// units) to per-stage bases, with the K steps of a slice unrolled at compile
// time, so the single issuing thread spends a handful of uniform-datapath
// instructions per tcgen05.mma instead of rebuilding descriptors (measured
// on B200: ~175 cycles per MMA with per-MMA descriptor arithmetic, 64 cycles
// -- the M=128 N=128 K=16 execution time -- with constant offsets).
// Descriptor arithmetic stays on the low 32-bit word (14-bit start-address
// field, byte offset >> 4; smem addresses never carry out of it); the high
// word (SBO, swizzle, version) is fixed per launch.  The two halves are
// joined inside the asm, so the issuing loop only does 32-bit uniform adds
// (64-bit loop-carried descriptors were kept in vector registers and moved
// to uniform registers before every MMA, stalling the issue).
template <int KIND, bool PAIR>
__device__ __forceinline__ void mma_issue(uint32_t d, uint32_t alo, uint32_t ahi, uint32_t blo,
                                          uint32_t bhi, uint32_t idesc, uint32_t acc) {
#define NEO_MMA_LO(CG, KIND)                                                                 \
  asm volatile("{\n\t.reg .pred p;\n\t.reg .b64 ad, bd;\n\t"                              \
               "setp.ne.b32 p, %6, 0;\n\t"                                                  \
               "mov.b64 ad, {%1, %2};\n\t"                                                  \
               "mov.b64 bd, {%3, %4};\n\t"                                                  \
               "tcgen05.mma.cta_group::" CG ".kind::" KIND " [%0], ad, bd, %5, p;\n\t}"      \
               ::"r"(d), "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(acc)     \
               : "memory")
  if constexpr (PAIR) {
    if constexpr (KIND == kKindTF32) NEO_MMA_LO("2", "tf32");
    else if constexpr (KIND == kKindFP8) NEO_MMA_LO("2", "f8f6f4");
    else NEO_MMA_LO("2", "f16");
  } else {
    if constexpr (KIND == kKindTF32) NEO_MMA_LO("1", "tf32");
    else if constexpr (KIND == kKindFP8) NEO_MMA_LO("1", "f8f6f4");
    else NEO_MMA_LO("1", "f16");
  }
#undef NEO_MMA_LO
}
// n slices (slice j at alo + j*a_step, blo + j*b_step), KPR K steps of 32
// bytes (+2 in descriptor units) each; acc0 = accumulate flag of the first MMA
template <int KIND, bool PAIR, int KPR>
__device__ __forceinline__ void mma_slices(uint32_t d, uint32_t alo, uint32_t ahi, uint32_t blo,
                                           uint32_t bhi, uint32_t a_step, uint32_t b_step, int n,
                                           uint32_t idesc, uint32_t acc0) {
  for (int j = 0; j < n; ++j) {
#pragma unroll
    for (int kk = 0; kk < KPR; ++kk)
      mma_issue<KIND, PAIR>(d, alo + 2u * kk, ahi, blo + 2u * kk, bhi, idesc, kk == 0 ? acc0 : 1u);
    acc0 = 1u;
    alo += a_step;
    blo += b_step;
  }
}

// MMA issue modes of mma_tiles
enum { kMmaK4 = 0, kMmaK2, kMmaK1, kMmaNarrow, kMmaHalo, kMmaHaloWst, kMmaHalo64, kMmaHaloWst64,
       kMmaHalo32, kMmaHaloWst32 };

// The MMA issuer's tile loop.  Barrier map as in conv_tc_kernel.  Stage and
// accumulator indices advance by counters; MODE fixes the operand layout:
//   K4/K2/K1  SWIZZLE_128/64/32 K-major slices (4/2/1 K steps of 16 per slice)
//   Narrow    16-byte rows, no swizzle, one K step spans two slices (LBO)
//   Halo      one band per (r, channel block), S taps = shifted views
//   HaloWst   weight-stationary halo: one band per channel block, R*S taps,
//             weights at b_sub * (cb*R + r) in the resident image
//   Halo64 / HaloWst64  the same over 64-byte rows (SWIZZLE_64B: e4m3 maps of
//             64 channels, bf16 of 32); a tap shift is one 64-byte row
template <int KIND, bool PAIR, int MODE>
__device__ __forceinline__ void mma_tiles(const ConvTCParams& p, int rank, uint32_t tmem_base,
                                          uint32_t sA, uint32_t sB, uint32_t sBar) {
  // A/B format codes: kind::tf32 TF32 = 2, kind::f16 BF16 = 1, kind::f8f6f4 E4M3 = 0
  const uint32_t idesc = umma_idesc(KIND == kKindTF32 ? 2u : KIND == kKindFP8 ? 0u : 1u,
                                    PAIR ? 2 * kTileM : kTileM, p.BN);
  constexpr bool halo64 = MODE == kMmaHalo64 || MODE == kMmaHaloWst64;
  constexpr bool halo32 = MODE == kMmaHalo32 || MODE == kMmaHaloWst32;
  const bool halo_mode = MODE == kMmaHalo || MODE == kMmaHaloWst || halo64 || halo32;
  // halo row: 128 bytes (SW128, 4 K steps per row), 64 (SW64, 2) or 32 (SW32, 1)
  constexpr uint32_t hrowb = halo32 ? 32u : halo64 ? 64u : 128u;
  constexpr uint32_t hrow_u = hrowb / 16u;             // one row in descriptor units
  constexpr int HKPR = (int)(hrowb / 32u);
  constexpr uint32_t hsbo = 8u * hrowb;                // 8-row core-matrix group
  constexpr uint32_t hlay = halo32 ? 6u : halo64 ? 4u : 2u;   // UMMA SWIZZLE_32B / 64B / 128B
  const uint64_t adesc0 = MODE == kMmaNarrow ? umma_smem_desc(sA, p.a_sub, 128, 0)
                          : halo_mode ? umma_smem_desc(sA, 16, hsbo, hlay)
                                      : umma_smem_desc(sA, 16, 8 * p.rowb, p.swz);
  const uint64_t bdesc0 = MODE == kMmaNarrow ? umma_smem_desc(sB, p.b_sub, 128, 0)
                          : halo_mode ? umma_smem_desc(sB, 16, hsbo, hlay)
                                      : umma_smem_desc(sB, 16, 8 * p.rowb, p.swz);
  const uint32_t a0lo = (uint32_t)adesc0, ahi = (uint32_t)(adesc0 >> 32);
  const uint32_t b0lo = (uint32_t)bdesc0, bhi = (uint32_t)(bdesc0 >> 32);
  const uint32_t a_stage_u = p.a_stage >> 4, b_stage_u = p.b_stage >> 4;
  const uint32_t a_sub_u = p.a_sub >> 4, b_sub_u = p.b_sub >> 4;
  const uint32_t b_tap_u = (uint32_t)(PAIR ? p.BN / 2 : p.BN) * hrow_u;   // halo: weight tap stride
  const uint32_t band_r_u = (uint32_t)p.BW * hrow_u;                      // wst halo: kernel row stride
  const uint32_t full0 = p.pro ? sBar + 384u : sBar;                 // xfull (prologue) or full
  const int nst = p.stages, ng = p.ngroups, G = p.G, S = p.S, R = p.R;
  const int kst = p.kstages;
  const bool split = p.splits > 1;
  const bool wst = p.wst != 0;
  int stage = 0, acc = 0;
  uint32_t phase = 0, acc_phase = 0;
  const bool prof = (p.dbg & 16) != 0;
  long long c_te = 0, c_fu = 0, c_mma = 0, c_com = 0, c_x;
  for (int it = 0;; ++it) {
    const int u = cta_unit(p, it, rank);
    if (u < 0) break;
    int ks0 = 0, ks1 = kst;
    if (split) {
      const int t = u / p.splits;
      ks0 = (u - t * p.splits) * p.kps;
      ks1 = min(kst, ks0 + p.kps);
    }
    if (prof) c_x = clock64();
    mbar_wait(sBar + 160u + 8u * acc, acc_phase ^ 1u);     // accumulator drained
    tc_fence_after();
    if (prof) c_te += clock64() - c_x;
    const uint32_t d_tmem = tmem_base + acc * p.BN;
    uint32_t ad = a0lo + (uint32_t)stage * a_stage_u;
    uint32_t bd = b0lo + (uint32_t)(wst && !halo_mode ? ks0 : stage) * b_stage_u;
    for (int ks = ks0; ks < ks1; ++ks) {
      if (prof) c_x = clock64();
      mbar_wait(full0 + 8u * stage, phase);
      tc_fence_after();
      if (prof) {
        const long long c = clock64();
        c_fu += c - c_x;
        c_x = c;
      }
      const uint32_t acc0 = ks != ks0 ? 1u : 0u;
      if constexpr (MODE == kMmaHaloWst || MODE == kMmaHaloWst64 || MODE == kMmaHaloWst32) {
        const uint32_t bw = b0lo + (uint32_t)ks * R * b_sub_u;
        for (int r = 0; r < R; ++r)
          mma_slices<KIND, PAIR, HKPR>(d_tmem, ad + r * band_r_u, ahi, bw + r * b_sub_u, bhi,
                                       hrow_u, b_tap_u, S, idesc, (acc0 | (uint32_t)r) ? 1u : 0u);
      } else if constexpr (MODE == kMmaHalo || MODE == kMmaHalo64 || MODE == kMmaHalo32) {
        for (int g = 0; g < G; ++g)
          mma_slices<KIND, PAIR, HKPR>(d_tmem, ad + g * a_sub_u, ahi, bd + g * b_sub_u, bhi,
                                       hrow_u, b_tap_u, S, idesc, (acc0 | (uint32_t)g) ? 1u : 0u);
      } else if constexpr (MODE == kMmaNarrow) {
        const int ksteps = G / 2;
        for (int k = 0; k < ksteps; ++k)
          mma_issue<KIND, PAIR>(d_tmem, ad + 2u * k * a_sub_u, ahi, bd + 2u * k * b_sub_u, bhi,
                                idesc, k == 0 ? acc0 : 1u);
      } else {
        constexpr int KPR = MODE == kMmaK4 ? 4 : MODE == kMmaK2 ? 2 : 1;
        mma_slices<KIND, PAIR, KPR>(d_tmem, ad, ahi, bd, bhi, a_sub_u, b_sub_u, G, idesc, acc0);
      }
      if (prof) {
        const long long c = clock64();
        c_mma += c - c_x;
        c_x = c;
      }
      if constexpr (PAIR) umma_commit2_mc(sBar + 64u + 8u * stage, 3);
      else umma_commit(sBar + 64u + 8u * stage);
      if (prof) c_com += clock64() - c_x;
      if (++stage == nst) {
        stage = 0;
        phase ^= 1u;
        ad = a0lo;
        bd = wst && !halo_mode ? bd + b_stage_u : b0lo;
      } else {
        ad += a_stage_u;
        bd += b_stage_u;
      }
    }
    if constexpr (PAIR) umma_commit2_mc(sBar + 128u + 8u * acc, 3);
    else umma_commit(sBar + 128u + 8u * acc);
    if (++acc == ng) {
      acc = 0;
      acc_phase ^= 1u;
    }
  }
  if (prof) {
    g_dbg_clk[2048 + 4 * blockIdx.x] = c_te;
    g_dbg_clk[2048 + 4 * blockIdx.x + 1] = c_fu;
    g_dbg_clk[2048 + 4 * blockIdx.x + 2] = c_mma;
    g_dbg_clk[2048 + 4 * blockIdx.x + 3] = c_com;
  }
}

// PAIR: CTA-pair (cta_group::2) instantiation, launched as 2-CTA clusters;
// kernels containing cta_group::2 instructions cannot run unclustered, so
// single-CTA tiles use the PAIR=false instantiation
template <int KIND, bool PAIR>
__global__ void __launch_bounds__(kThreads, 1) conv_tc_kernel(const __grid_constant__ ConvTCParams p) {
  constexpr bool TF32 = KIND == kKindTF32;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  long long dbg_t_entry = 0;
  if (p.dbg & 64) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(dbg_t_entry));
  if ((p.dbg & 256) && threadIdx.x == 0) tl_stamp(p, 0);
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t pad = (1024u - (sraw & 1023u)) & 1023u;
  const uint32_t sA = sraw + pad;
  const uint32_t sB = sA + p.stages * p.a_stage;
  const uint32_t sO = sB + p.b_region;   // ngroups x nslot staging slots
  const uint32_t sBar = sO + p.ngroups * p.nslot * p.stage_out;
  uint8_t* gen_base = smem_raw + pad;
  uint8_t* bar_gen = gen_base + (sBar - sA);
  auto full_bar = [&](int i) { return sBar + 8u * i; };
  auto empty_bar = [&](int i) { return sBar + 64u + 8u * i; };
  auto tfull_bar = [&](int a) { return sBar + 128u + 8u * a; };
  auto tempty_bar = [&](int a) { return sBar + 160u + 8u * a; };
  auto res_bar = [&](int g, int b) { return sBar + 192u + 16u * g + 8u * b; };
  const uint32_t tslot = sBar + 256u;
  auto xfull_bar = [&](int i) { return sBar + 384u + 8u * i; };   // prologue: slice rewritten
  const uint32_t wbar = sBar + 320u;                                // weight-stationary image
  volatile uint32_t* tslot_gen = reinterpret_cast<volatile uint32_t*>(bar_gen + 256);
  float* par_gen = reinterpret_cast<float*>(bar_gen + 512);   // ngroups x kParamFloats

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int epi_warps = p.pro ? kEpiWarps - kProWarps : p.epi_warps;   // warps 2 .. 2+epi_warps-1
  const int rank = PAIR ? (int)cluster_ctarank() : 0;
  const bool leader_cta = rank == 0;
#ifdef NEO_TRACE
  __shared__ unsigned s_trace_cnt[32];
  if (threadIdx.x < 32) s_trace_cnt[threadIdx.x] = 0;
  __syncthreads();
#endif
  if (threadIdx.x == 0) TRACE(60, 0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&p.tmA);
    tma_prefetch_desc(&p.tmB);
    if (p.tma_epi) {
      tma_prefetch_desc(&p.tmO);
      if (p.res) tma_prefetch_desc(&p.tmR);
      if (p.k_split) tma_prefetch_desc(&p.tmO2);
    }
    for (int i = 0; i < p.stages; ++i) {
      mbar_init(full_bar(i), 1);
      mbar_init(empty_bar(i), 1);
      mbar_init(xfull_bar(i), kProWarps);
    }
    mbar_init(wbar, 1);
    for (int a = 0; a < p.ngroups; ++a) {
      mbar_init(tfull_bar(a), 1);
      // pair: the leader's MMA waits for both CTAs' epilogue warps
      mbar_init(tempty_bar(a), (PAIR ? 2 : 1) * (epi_warps / p.ngroups));
      mbar_init(res_bar(a, 0), 1);
      mbar_init(res_bar(a, 1), 1);
    }
    fence_mbar_init();
  }
  if constexpr (PAIR) cluster_sync_all();   // peer barriers initialised before any remote arrive
  if (warp == 1) {
    if constexpr (PAIR) {
      tmem_alloc2(tslot, p.tmem_cols);
      tmem_relinquish2();
    } else {
      tmem_alloc(tslot, p.tmem_cols);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tslot_gen;
  if (threadIdx.x == 0) TRACE(61, 0);
  // PDL: barrier init, TMEM allocation and descriptor prefetch above overlap
  // the previous kernel's tail.  Each role waits for the previous kernel
  // before it touches global memory the previous kernels may write; the
  // producer first issues a static resident weight image (weights are not
  // written by the step), and the MMA warp never touches global memory.
  neo_pdl_trigger();
  if (warp != 0 && warp != 1) neo_pdl_wait();
  long long dbg_t_pdl = 0;
  if (p.dbg & 64) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(dbg_t_pdl));
  if ((p.dbg & 256) && threadIdx.x == 64) tl_stamp(p, 1);     // an epilogue warp, past the wait

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int stage = 0;
      uint32_t phase = 0;
      // pair: the peer's loads complete on the leader's full barriers
      const uint32_t fbar_base = PAIR ? mapa_shared(full_bar(0), 0) : full_bar(0);
      const int bofs = PAIR ? rank * (p.BN / 2) : 0;   // weight rows this CTA fetches
      if (!(p.wst && p.static_w)) neo_pdl_wait();
      if (p.wst) {
        // the CTA's N block (grid % tiles_k == 0) -> its whole weight image
        const int wk0 = ((int)blockIdx.x % p.tiles_k) * p.BN;
        mbar_arrive_expect_tx(wbar, p.b_region);
        if (p.halo) {
          for (int co = 0; co < p.Cb; ++co)
            for (int r = 0; r < p.R; ++r)
              tma_load_4d(sB + (uint32_t)(co * p.R + r) * p.b_sub, &p.tmB, wbar, 0, wk0, co,
                          r * p.S);
        } else {
          for (int ks = 0; ks < p.kstages; ++ks)
            tma_load_3d(sB + (uint32_t)ks * p.b_stage, &p.tmB, wbar, 0, wk0, ks * p.G);
        }
        if (p.static_w) neo_pdl_wait();   // activations come from the previous kernel
      }
      for (int i = 0;; ++i) {
        const int u = cta_unit(p, i, rank);
        if (u < 0) break;
        const int t = p.splits == 1 ? u : u / p.splits;
        const int ks0 = p.splits == 1 ? 0 : (u - t * p.splits) * p.kps;
        const int ks1 = p.splits == 1 ? p.kstages : min(p.kstages, ks0 + p.kps);
        int n0, oh0, ow0, k0;
        decode_tile(p, t, n0, oh0, ow0, k0);
        const int iw0 = ow0 * p.stride_w - p.pad_w;
        const int ih0 = oh0 * p.stride_h - p.pad_h;
        if (p.halo && p.wst) {
          // one band per channel block: rows ih0 .. ih0 + BH + R - 2
          for (int ks = ks0; ks < ks1; ++ks) {
            TRACE(1, t);
            mbar_wait(empty_bar(stage), phase ^ 1u);
            TRACE(2, t);
            if (p.dbg & 2) {
              mbar_arrive(full_bar(stage));
            } else {
              mbar_arrive_expect_tx(full_bar(stage), p.tx_bytes);
              tma_load_5d(sA + stage * p.a_stage, &p.tmA, full_bar(stage), 0, iw0, ih0, ks, n0);
            }
            if (++stage == p.stages) {
              stage = 0;
              phase ^= 1u;
            }
          }
          continue;
        }
        if (p.halo) {
          for (int ks = ks0; ks < ks1; ++ks) {
            TRACE(1, t);
            mbar_wait(empty_bar(stage), phase ^ 1u);
            TRACE(2, t);
            const uint32_t fb = fbar_base + 8u * stage;
            if (!PAIR && (p.dbg & 4)) {      // timing experiment: no operand loads
              mbar_arrive(full_bar(stage));
              if (++stage == p.stages) {
                stage = 0;
                phase ^= 1u;
              }
              continue;
            }
            if (leader_cta) mbar_arrive_expect_tx(full_bar(stage), p.tx_bytes);
            const uint32_t a_dst = sA + stage * p.a_stage;
            const uint32_t b_dst = sB + stage * p.b_stage;
            for (int g = 0; g < p.G; ++g) {
              const int pi = ks * p.G + g;        // (r, channel block) pair
              int co = p.Cb, r = 0;               // padding pair -> zeros
              if (pi < p.nslices) {
                co = pi % p.Cb;
                r = pi / p.Cb;
              }
              if (!PAIR || leader_cta) {
                tma_load_5d(a_dst + g * p.a_sub, &p.tmA, fb, 0, iw0, ih0 + r, co, n0);
                tma_load_4d(b_dst + g * p.b_sub, &p.tmB, fb, 0, k0 + bofs, co, r * p.S);
              } else if constexpr (PAIR) {
                tma_load_5d_pair(a_dst + g * p.a_sub, &p.tmA, fb, 0, iw0, ih0 + r, co, n0);
                tma_load_4d_pair(b_dst + g * p.b_sub, &p.tmB, fb, 0, k0 + bofs, co, r * p.S);
              }
            }
            if (++stage == p.stages) {
              stage = 0;
              phase ^= 1u;
            }
          }
          continue;
        }
        // slice = (r, s, channel block), channel block fastest; walked with
        // counters (no divisions on the single producer thread)
        int sl = ks0 * p.G;
        int co = sl % p.Cb, sc = (sl / p.Cb) % p.S, rc = sl / (p.Cb * p.S);
        for (int ks = ks0; ks < ks1; ++ks) {
          TRACE(1, t);
          mbar_wait(empty_bar(stage), phase ^ 1u);
          TRACE(2, t);
          const uint32_t fb = fbar_base + 8u * stage;
          if (!PAIR && (p.dbg & 4)) {        // timing experiment: no operand loads
            mbar_arrive(full_bar(stage));
            if (++stage == p.stages) {
              stage = 0;
              phase ^= 1u;
            }
            continue;
          }
          if (leader_cta) mbar_arrive_expect_tx(full_bar(stage), p.tx_bytes);
          const uint32_t a_dst = sA + stage * p.a_stage;
          for (int g = 0; g < p.G; ++g, ++sl) {
            const int cx = sl < p.nslices ? iw0 + sc : 0;     // stage padding slice:
            const int cy = sl < p.nslices ? ih0 + rc : 0;     // fully out of bounds -> zeros
            const int cc = sl < p.nslices ? co : p.Cb;
            if (!PAIR || leader_cta) tma_load_5d(a_dst + g * p.a_sub, &p.tmA, fb, 0, cx, cy, cc, n0);
            else if constexpr (PAIR) tma_load_5d_pair(a_dst + g * p.a_sub, &p.tmA, fb, 0, cx, cy, cc, n0);
            if (sl < p.nslices) {
              if (++co == p.Cb) {
                co = 0;
                if (++sc == p.S) {
                  sc = 0;
                  ++rc;
                }
              }
            }
          }
          if (p.wst) {
          } else if (!PAIR || leader_cta) {
            tma_load_3d(sB + stage * p.b_stage, &p.tmB, fb, 0, k0 + bofs, ks * p.G);
          } else if constexpr (PAIR) {
            tma_load_3d_pair(sB + stage * p.b_stage, &p.tmB, fb, 0, k0 + bofs, ks * p.G);
          }
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader_cta) {
      // ---------------- MMA issuer (pair: the leader issues M=256) ----------
      // one tile-loop instantiation per operand layout: the single issuing
      // thread must keep the tensor pipe's short queue (~2 MMAs) fed, so the
      // loop carries no per-stage mode branches and no integer divisions
      long long dbg_c0 = 0, dbg_t0 = 0;
      if (p.wst) mbar_wait(wbar, 0);
      if (p.dbg & 8) {
        dbg_c0 = clock64();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(dbg_t0));
      }
      if (p.dbg & 256) tl_stamp(p, 2);
      const int mode = p.halo ? (p.rowb == 32   ? (p.wst ? kMmaHaloWst32 : kMmaHalo32)
                                 : p.rowb == 64 ? (p.wst ? kMmaHaloWst64 : kMmaHalo64)
                                                : (p.wst ? kMmaHaloWst : kMmaHalo))
                       : p.rowb == 16 ? kMmaNarrow
                       : p.rowb >= 128 ? kMmaK4
                       : p.rowb == 64 ? kMmaK2 : kMmaK1;
      switch (mode) {
        case kMmaK4: mma_tiles<KIND, PAIR, kMmaK4>(p, rank, tmem_base, sA, sB, sBar); break;
        case kMmaK2: mma_tiles<KIND, PAIR, kMmaK2>(p, rank, tmem_base, sA, sB, sBar); break;
        case kMmaK1: mma_tiles<KIND, PAIR, kMmaK1>(p, rank, tmem_base, sA, sB, sBar); break;
        case kMmaNarrow: mma_tiles<KIND, PAIR, kMmaNarrow>(p, rank, tmem_base, sA, sB, sBar); break;
        case kMmaHalo: mma_tiles<KIND, PAIR, kMmaHalo>(p, rank, tmem_base, sA, sB, sBar); break;
        case kMmaHalo64: mma_tiles<KIND, PAIR, kMmaHalo64>(p, rank, tmem_base, sA, sB, sBar); break;
        case kMmaHaloWst64: mma_tiles<KIND, PAIR, kMmaHaloWst64>(p, rank, tmem_base, sA, sB, sBar); break;
        case kMmaHalo32: mma_tiles<KIND, PAIR, kMmaHalo32>(p, rank, tmem_base, sA, sB, sBar); break;
        case kMmaHaloWst32: mma_tiles<KIND, PAIR, kMmaHaloWst32>(p, rank, tmem_base, sA, sB, sBar); break;
        default: mma_tiles<KIND, PAIR, kMmaHaloWst>(p, rank, tmem_base, sA, sB, sBar); break;
      }
      if (p.dbg & 256) tl_stamp(p, 3);
      if (p.dbg & 8) {
        long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        g_dbg_clk[2 * blockIdx.x] = (unsigned long long)(clock64() - dbg_c0);
        g_dbg_clk[2 * blockIdx.x + 1] = (unsigned long long)(t1 - dbg_t0);
        g_dbg_clk[7000 + 2 * blockIdx.x] = dbg_t0;
        g_dbg_clk[7000 + 2 * blockIdx.x + 1] = t1;
      }
    }
  } else if (p.pro && warp >= 2 + epi_warps) {
    // ---------------- prologue warps: walk the stage ring behind the
    // producer; rewrite each landed slice in place, hand it to the MMA
    const int ptid = (warp - 2 - epi_warps) * 32 + lane;
    const int chunks_row = p.rowb / 16;               // 16-byte chunks per row
    const int per_slice = kTileM * chunks_row;
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0;; ++it) {
      const int u = cta_unit(p, it, rank);
      if (u < 0) break;
      const int t = u / p.splits;
      const int ks0 = (u - t * p.splits) * p.kps;
      const int ks1 = min(p.kstages, ks0 + p.kps);
      for (int ks = ks0; ks < ks1; ++ks) {
        mbar_wait(full_bar(stage), phase);
        uint8_t* a_gen = gen_base + stage * p.a_stage;
        for (int g = 0; g < p.G; ++g) {
          const int sl = ks * p.G + g;                // 1x1: slice = channel block
          if (sl >= p.nslices) continue;              // padding slice: zeros x zero weights
          const int cbase = (sl % p.Cb) * (p.rowb / (TF32 ? 4 : 2));
          uint8_t* slice = a_gen + g * p.a_sub;
          if constexpr (!TF32) {
            // bf16: a thread always rewrites the same 16-byte chunk column
            // of the slice (256 threads, chunks_row | 256), so its 8
            // channels' scale / shift are loaded once per slice; multiply
            // and add as the reference's two rounded ops (executor.py:
            // 180-181), relu, one bf16 conversion per pair -- the rewrite
            // must keep pace with the MMAs
            const int ch = ptid & (chunks_row - 1);
            const int c0 = cbase + ch * 8;
            const float4 s0 = __ldg(reinterpret_cast<const float4*>(p.pro_scale + c0));
            const float4 s1 = __ldg(reinterpret_cast<const float4*>(p.pro_scale + c0 + 4));
            const float4 t0 = __ldg(reinterpret_cast<const float4*>(p.pro_shift + c0));
            const float4 t1 = __ldg(reinterpret_cast<const float4*>(p.pro_shift + c0 + 4));
            const float2 sc2[4] = {make_float2(s0.x, s0.y), make_float2(s0.z, s0.w),
                                   make_float2(s1.x, s1.y), make_float2(s1.z, s1.w)};
            const float2 sh2[4] = {make_float2(t0.x, t0.y), make_float2(t0.z, t0.w),
                                   make_float2(t1.x, t1.y), make_float2(t1.z, t1.w)};
            const int row_step = (kProWarps * 32) / chunks_row;
            for (int row = ptid / chunks_row; row < kTileM; row += row_step) {
              uint4* ptr = reinterpret_cast<uint4*>(slice + swz_offset(row, ch, p.rowb));
              uint4 v = *ptr;
              uint32_t* h = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 x2 = make_float2(__uint_as_float(h[e] << 16),
                                              __uint_as_float(h[e] & 0xFFFF0000u));
                // scalar _rn ops: nvcc contracts __fmul2_rn + __fadd2_rn into
                // one FFMA2 (one rounding), which would break the reference's
                // two-rounding BN and the bit-identity with the unfused path
                float2 y2 = make_float2(__fadd_rn(__fmul_rn(x2.x, sc2[e].x), sh2[e].x),
                                        __fadd_rn(__fmul_rn(x2.y, sc2[e].y), sh2[e].y));
                if (p.pro_relu) {          // fmaxf like the unfused BN-ReLU (bit-identical)
                  y2.x = fmaxf(y2.x, 0.f);
                  y2.y = fmaxf(y2.y, 0.f);
                }
                asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(h[e]) : "f"(y2.x), "f"(y2.y));
              }
              *ptr = v;
            }
            continue;
          }
          for (int idx = ptid; idx < per_slice; idx += kProWarps * 32) {
            const int row = idx / chunks_row, ch = idx - row * chunks_row;
            uint4* ptr = reinterpret_cast<uint4*>(slice + swz_offset(row, ch, p.rowb));
            uint4 v = *ptr;
            float* f = reinterpret_cast<float*>(&v);
            const int c0 = cbase + ch * 4;
            const float4 sc = __ldg(reinterpret_cast<const float4*>(p.pro_scale + c0));
            const float4 sh = __ldg(reinterpret_cast<const float4*>(p.pro_shift + c0));
            const float scv[4] = {sc.x, sc.y, sc.z, sc.w}, shv[4] = {sh.x, sh.y, sh.z, sh.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float y = __fadd_rn(__fmul_rn(f[e], scv[e]), shv[e]);
              if (p.pro_relu) y = fmaxf(y, 0.f);
              f[e] = neo_round_tf32(y);
            }
            *ptr = v;
          }
        }
        fence_proxy_async_smem();      // generic-proxy writes -> tensor-core reads
        __syncwarp();
        if (lane == 0) mbar_arrive(xfull_bar(stage));
        if (++stage == p.stages) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
  } else {
    // ---------------- epilogue: two groups of 4 warps, group g takes the
    // tiles whose accumulator lives in TMEM stage g (alternate tiles), so
    // both groups drain in parallel with the MMA of the next tile.
    const int gwarps = epi_warps / p.ngroups;      // 8 or 4 (4 in prologue mode)
    const int gthreads = gwarps * 32;
    const int grp = (warp - 2) / gwarps;
    const int nsub = gwarps / 4;                    // warps per lane quarter: 2 or 1
    const int half = ((warp - 2) >> 2) % nsub;      // which channel blocks of a tile
    const int q = warp & 3;                 // TMEM lane quarter of this warp
    const int m = q * 32 + lane;            // accumulator row = tile pixel
    // halo strips: accumulator row m = (tile row h, band column w) with a
    // pitch of BW band columns; only w < BWo belongs to the strip, and its
    // staging row is compacted to h * BWo + w (the store / residual boxes are
    // BWo columns wide).  Rows of band columns past the strip are parked in
    // the staging rows behind the box (BWo*BH + h*(S-1) + w - BWo < BW*BH <=
    // 128): they are computed like any other row and never stored, so the
    // per-piece epilogue loop carries no predicate
    int ms = m;
    if (p.BWo != p.BW) {
      const int hh = m / p.BW, ww = m - hh * p.BW;
      ms = ww < p.BWo ? hh * p.BWo + ww
                      : min(kTileM - 1, p.BWo * p.BH + hh * (p.BW - p.BWo) + (ww - p.BWo));
    }
    const bool leader = (warp == 2 + gwarps * grp) && lane == 0;
    const uint32_t bar_id = 1 + grp;
    const size_t plane = (size_t)p.OH * p.OW * p.y;
    uint32_t res_phase = 0u;                // phase of this group's residual barrier
    int par_k0 = -1;                        // N block whose parameters are staged
    const bool affine = p.scale != nullptr || p.shift != nullptr;
    const bool eprof = (p.dbg & 32) != 0 && (warp == 2 + gwarps * grp) && lane == 0;
    long long e_pre = 0, e_tf = 0, e_res = 0, e_cmp = 0, e_st = 0, e_x = 0;
    auto etick = [&](long long& acc_c) {
      if (eprof) {
        const long long c = clock64();
        acc_c += c - e_x;
        e_x = c;
      }
    };
    // pair: accumulator releases go to the leader CTA's tempty barriers
    const uint32_t tempty_base = PAIR ? mapa_shared(tempty_bar(0), 0) : tempty_bar(0);
    const uint32_t ng_log2 = (uint32_t)(__ffs(p.ngroups) - 1);
    // last-tile sharing: the owner group of the CTA's last unit drains the
    // first half of its channel blocks, the next group the second half
    const int last_it = (p.share_last && (int)blockIdx.x < p.num_units)
                            ? (p.num_units - 1 - (int)blockIdx.x) / (int)gridDim.x : -1;
    const int owner_grp = last_it >= 0 ? (last_it & (p.ngroups - 1)) : -1;
    const int helper_grp = last_it >= 0 ? ((owner_grp + 1) & (p.ngroups - 1)) : -1;
    for (int it = grp;; it += p.ngroups) {
      int u = cta_unit(p, it, rank);
      int acc = grp;
      uint32_t acc_phase = ((uint32_t)it >> ng_log2) & 1u;   // ngroups is 2 or 4
      bool helping = false;
      if (u < 0) {
        if (grp != helper_grp || last_it < 0) break;
        helping = true;                   // join the owner group's last tile
        u = cta_unit(p, last_it, rank);
        acc = owner_grp;
        acc_phase = ((uint32_t)last_it >> ng_log2) & 1u;
      }
      const bool owning_last = !helping && it == last_it;
      const int t = p.splits == 1 ? u : (int)((uint32_t)u / (uint32_t)p.splits);
      int n0, oh0, ow0, k0;
      decode_tile(p, t, n0, oh0, ow0, k0);
      const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16) + acc * p.BN;
      const int ncols = min(p.BN, p.K - k0);
      if (p.splits > 1) {
        // split-K: every unit of a tile stores its raw accumulator to
        // ws[u][chunk16][row][16] and releases TMEM; once all splits of the
        // tile arrived (per-tile counter; the host keeps every unit of a split
        // launch co-resident), each unit reduces its 1/splits share of the
        // tile's (chunk, row) pairs in split order -- deterministic -- and runs
        // the direct epilogue on it.
        mbar_wait(tfull_bar(acc), acc_phase);
        tc_fence_after();
        const int nch = p.BN / 16;
        float4* dst = reinterpret_cast<float4*>(p.ws) + ((size_t)u * nch * kTileM + m) * 4;
        for (int c = half; c < nch; c += nsub) {
          uint32_t v[16];
          tmem_ld16(trow + c * 16, v);
          tmem_ld_wait();
          float4* d = dst + (size_t)c * kTileM * 4;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            __stcg(d + j, make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                      __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3])));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (PAIR) mbar_arrive_cluster(tempty_base + 8u * acc);
          else mbar_arrive(tempty_bar(acc));
        }
        __threadfence();
        named_bar_sync(bar_id, gthreads);
        if (leader) {
          TRACE(40, t);
          atomicAdd(p.counters + t, 1);
          spin_until_geq(p.counters + t, p.splits);
          TRACE(41, t);
        }
        named_bar_sync(bar_id, gthreads);
        __threadfence();
        splitk_fixup(p, t, u - t * p.splits, n0, oh0, ow0, k0, ((warp - 2) % gwarps) * 32 + lane,
                     gthreads);
        // second arrival: the unit arriving last (every unit is past its
        // wait) re-zeroes the counter for the next launch
        named_bar_sync(bar_id, gthreads);
        if (leader) TRACE(42, t);
        if (leader && atomicAdd(p.counters + t, 1) == 2 * p.splits - 1) p.counters[t] = 0;
        continue;
      }
      if (p.tma_epi && (p.dbg & 1)) {
        // timing experiment (NEOB200_DBG & 1): drain nothing -- wait for the
        // accumulator and release it at once (no residual loads, no stores)
        if (helping) break;
        mbar_wait(tfull_bar(acc), acc_phase);
        tc_fence_after();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (PAIR) mbar_arrive_cluster(tempty_base + 8u * acc);
          else mbar_arrive(tempty_bar(acc));
        }
        continue;
      }
      if (p.tma_epi) {
        // staged epilogue: the tile's output channel blocks go through up to
        // p.nslot swizzled smem slots; residual blocks are fetched by TMA
        // into the same slots before the accumulator is waited for, then
        // results overwrite them and leave with TMA bulk stores.
        const bool has_res = p.res != nullptr;
        const int nblk = ncols / p.y;
        const bool pf = p.res_pf != 0;
        int blk_lo = 0, blk_hi = nblk;
        if (helping || owning_last) {
          const int hb = (nblk + 1) >> 1;
          if (nblk < 2) {
            if (helping) break;           // nothing to share
          } else if (helping) {
            blk_lo = hb;
          } else {
            blk_hi = hb;
          }
        }
        const int lt = (int)((uint32_t)it >> ng_log2);   // this group's tile counter
        const int set = pf ? (lt & 1) : 0;        // prefetch: alternate slot sets
        const uint32_t sgrp = sO + (grp * p.nslot + set * (p.nslot / 2)) * p.stage_out;
        uint8_t* sgrp_gen = gen_base + (sgrp - sA);
        const uint32_t rbar = res_bar(grp, set);
        auto load_res = [&](uint32_t dst, uint32_t bar, int b0, int cnt, int tow0, int toh0, int tk0,
                            int tn0) {
          mbar_arrive_expect_tx(bar, cnt * p.out_box_bytes);
          for (int i = 0; i < cnt; ++i)
            tma_load_5d(dst + i * p.stage_out, &p.tmR, bar, 0, tow0, toh0,
                        p.res_cb_off + (tk0 + (b0 + i) * p.y) / p.y, tn0);
        };
        auto issue_res = [&](int b0, int cnt) {
          if (!leader) return;
          bulk_wait_read<0>();              // previous stores left the slots
          if (has_res) load_res(sgrp, rbar, b0, cnt, ow0, oh0, k0, n0);
        };
        if (leader) TRACE(20 + grp, t);
        if (eprof) e_x = clock64();
        if (!pf || helping) issue_res(blk_lo, min(blk_hi - blk_lo, pf ? p.nslot / 2 : p.nslot));
        else if (lt == 0 && leader) load_res(sgrp, rbar, 0, nblk, ow0, oh0, k0, n0);
        if (k0 != par_k0) {
          // stage this tile's channel vectors (identity where absent); a
          // group keeps them while its tiles stay in one N block
          par_k0 = k0;
          float* par = par_gen + grp * kParamFloats;
          const int j = ((warp - 2) % gwarps) * 32 + lane;
          const int k = k0 + j;
          const bool in = j < p.BN && k < p.K;
          par[j] = (in && p.scale) ? __ldg(p.scale + k) : 1.f;
          par[256 + j] = (in && p.shift) ? __ldg(p.shift + k) : 0.f;
          par[512 + j] = (in && p.bias) ? __ldg(p.bias + k) : 0.f;
        }
        if (leader) TRACE(22 + grp, t);
        named_bar_sync(bar_id, gthreads);
        if (leader) TRACE(24 + grp, t);
        etick(e_pre);
        mbar_wait(tfull_bar(acc), acc_phase);
        if (leader) TRACE(26 + grp, t);
        tc_fence_after();
        etick(e_tf);

        const int slots = pf ? p.nslot / 2 : p.nslot;
        for (int b0 = blk_lo; b0 < blk_hi; b0 += slots) {
          const int cnt = min(slots, blk_hi - b0);
          if (b0 > blk_lo) {
            issue_res(b0, cnt);
            named_bar_sync(bar_id, gthreads);
          }
          if (has_res) {
            mbar_wait(rbar, pf ? ((uint32_t)(lt >> 1) & 1u) : (res_phase & 1u));
            res_phase ^= 1u;
          }
          etick(e_res);
          if (leader) TRACE(28 + grp, t);
          const bool sec = p.k_split > 0 && k0 >= p.k_split;   // second output's tile
          const float floor_v = (sec ? p.relu2 : p.relu) ? 0.f : -INFINITY;
          const float qs = sec ? p.out2_qscale : p.out_qscale;
          const bool rnd = p.round_tf32 != 0;
          // the two warps of a lane quarter split the chunk's work: whole
          // blocks when there are several, 16-column pieces of one block else
          const bool by_block = nsub == 1 || cnt >= 2;
          const int bstep = nsub == 1 ? 1 : (cnt >= 2 ? 2 : 1);
          const int cbeg = by_block ? 0 : half, cstep = by_block ? 1 : 2;
          const float* par = par_gen + grp * kParamFloats;
          for (int i = (nsub == 2 && cnt >= 2 ? half : 0); i < cnt; i += bstep) {
            const uint32_t tcol = trow + (b0 + i) * p.y;
            const int col0 = (b0 + i) * p.y;
            uint8_t* sg = sgrp_gen + i * p.stage_out;
#define NEO_EPI(OUT, RES, AFF) \
  epi_block_tma<OUT, RES, AFF>(p, tcol, col0, ms, sg, par, floor_v, rnd, cbeg, cstep, qs)
#define NEO_EPI_OUT(OUT)                       \
  if (affine) {                                \
    if (has_res) NEO_EPI(OUT, true, true);     \
    else NEO_EPI(OUT, false, true);            \
  } else {                                     \
    if (has_res) NEO_EPI(OUT, true, false);    \
    else NEO_EPI(OUT, false, false);           \
  }
            if (p.out_kind == kOutF32) {
              NEO_EPI_OUT(kOutF32)
            } else if ((KIND == kKindFP8 || KIND == kKindBF16Q) && p.out_kind == kOutFP8) {
              NEO_EPI_OUT(kOutFP8)
            } else {
              NEO_EPI_OUT(kOutBF16)
            }
#undef NEO_EPI_OUT
#undef NEO_EPI
          }
          if (b0 + cnt >= blk_hi && !helping) {   // accumulator read: release TMEM
            // (a shared last tile is released by its owner alone: the MMA
            // thread never waits on that accumulator again)
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if constexpr (PAIR) mbar_arrive_cluster(tempty_base + 8u * acc);
              else mbar_arrive(tempty_bar(acc));
            }
          }
          etick(e_cmp);
          if (leader) TRACE(30 + grp, t);
          fence_proxy_async_smem();
          named_bar_sync(bar_id, gthreads);
          if (leader) TRACE(32 + grp, t);
          if (leader) {
            const bool sec = p.k_split > 0 && k0 >= p.k_split;
            const CUtensorMap* tmo = sec ? &p.tmO2 : &p.tmO;
            const int cb0 = sec ? p.out2_cb_off + (k0 - p.k_split) / p.y : p.out_cb_off + k0 / p.y;
            for (int i = 0; i < cnt; ++i)
              tma_store_5d(tmo, sgrp + i * p.stage_out, 0, ow0, oh0, cb0 + b0 + i, n0);
            bulk_commit();
            if (pf && !helping) {
              // the group's next tile: its residual goes into the other set
              // once the store issued from that set one tile ago has read it
              const int un = cta_unit(p, it + p.ngroups, rank);
              if (un >= 0) {
                int nn0, noh0, now0, nk0;
                decode_tile(p, un / p.splits, nn0, noh0, now0, nk0);
                bulk_wait_read<1>();
                const int nset = set ^ 1;
                load_res(sO + (grp * p.nslot + nset * (p.nslot / 2)) * p.stage_out,
                         res_bar(grp, nset), 0, min(p.K - nk0, p.BN) / p.y, now0, noh0, nk0,
                         nn0);
              }
            }
          }
          etick(e_st);
        }
        if (helping) break;
        continue;
      } else {
        if (helping) break;                // (sharing needs the TMA epilogue)
        mbar_wait(tfull_bar(acc), acc_phase);
        tc_fence_after();
        const int wl = m % p.BW, hl = (m / p.BW) % p.BH, nl = m / (p.BW * p.BH);
        const int ow = ow0 + wl, oh = oh0 + hl, n = n0 + nl;
        const bool valid = (m < p.BW * p.BH * p.BNI) && wl < p.BWo && ow < p.OW && oh < p.OH &&
                           n < p.N;
        EpiAccess ea;
        ea.plane = plane;
        const size_t pix = ((size_t)oh * p.OW + ow) * p.y;
        ea.out_base = (size_t)n * p.out_cb_total * plane + (size_t)p.out_cb_off * plane + pix;
        ea.res_base = (size_t)n * p.res_cb_total * plane + (size_t)p.res_cb_off * plane + pix;
        for (int c0 = 16 * half; c0 < ncols; c0 += 16 * nsub) {
          uint32_t v[16];
          tmem_ld16(trow + c0, v);
          tmem_ld_wait();
          if (valid) epi_chunk(p, v, k0 + c0, ea);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
          if constexpr (PAIR) mbar_arrive_cluster(tempty_base + 8u * acc);
          else mbar_arrive(tempty_bar(acc));
        }
    }
    // the staging slots must outlive the stores' reads; the writes themselves
    // complete with the grid (dependent kernels wait on grid completion)
    if (leader) bulk_wait_read<0>();
    if (leader) TRACE(64, 0);
    if (eprof) {
      unsigned long long* d = g_dbg_clk + 4096 + (blockIdx.x * 4 + grp) * 5;
      d[0] = e_pre;
      d[1] = e_tf;
      d[2] = e_res;
      d[3] = e_cmp;
      d[4] = e_st;
    }
  }

  __syncthreads();
  if (threadIdx.x == 0) TRACE(62, 0);
  if ((p.dbg & 256) && threadIdx.x == 0) tl_stamp(p, 4);
  if ((p.dbg & 64) && threadIdx.x == 0) {
    // per-CTA timeline: entry, past griddepcontrol.wait, all roles done
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_dbg_clk[6144 + 3 * blockIdx.x] = dbg_t_entry;
    g_dbg_clk[6144 + 3 * blockIdx.x + 1] = dbg_t_pdl;
    g_dbg_clk[6144 + 3 * blockIdx.x + 2] = t;
  }
#ifdef NEO_TRACE
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x < kTraceWarps)
    g_trace_cnt[threadIdx.x] = min(s_trace_cnt[threadIdx.x], (unsigned)kTracePerWarp);
#endif
  if constexpr (PAIR) cluster_sync_all();   // the peer's TMEM is written by the leader's MMAs
  if (warp == 1) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc2(tmem_base, p.tmem_cols);
    else tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

// ---------------------------------------------------------------------------
// host side

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
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

int sm_count_of_current_device() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = v > 0 ? v : 148;
  }
  return cache[dev];
}

int swizzle_code_umma(int rowb) {
  switch (rowb) {
    case 32: return 6;
    case 64: return 4;
    case 128: return 2;
    default: return 0;
  }
}
CUtensorMapSwizzle swizzle_code_tma(int rowb) {
  switch (rowb) {
    case 32: return CU_TENSOR_MAP_SWIZZLE_32B;
    case 64: return CU_TENSOR_MAP_SWIZZLE_64B;
    case 128: return CU_TENSOR_MAP_SWIZZLE_128B;
    default: return CU_TENSOR_MAP_SWIZZLE_NONE;
  }
}

int64_t conv_out_dim(int64_t in, int64_t k, int st, int pad) { return (in + 2 * pad - k) / st + 1; }

// Half-SM mode (NEOB200_HALF=1): every conv CTA takes at most half an SM --
// 320 threads (8 epilogue warps), <= 113 KB of shared memory, <= 256 TMEM
// columns -- so two CTAs are co-resident per SM: CTAs of the next launch
// (PDL) or of a second stream's launch set up and run beside this one's
// fill / drain phases.
bool half_sm_mode() {
  static const bool on = getenv("NEOB200_HALF") && atoi(getenv("NEOB200_HALF")) > 0;
  return on;
}
int64_t smem_budget() { return half_sm_mode() ? 113 * 1024 : kSmemBudget; }

struct Geometry {
  int BW, BH, BNI;
};

// M-tile geometry maximising useful rows of the 128-row MMA tile.
// ``local``: tiles of ONE image only (tile_img = 1).  On odd maps at batch
// 128 the unrestricted pick is one pixel x 128 images (all 128 rows useful),
// which is fine for 1x1 convs and small maps but loses 22-29% on windowed
// convs over large maps (Inception-v3's 147x147 / 73x73 3x3 layers,
// tools/geo_sweep.py): every tap's A box is 128 rows scattered over 128
// images instead of a few contiguous row segments.
Geometry pick_geometry(int64_t N, int64_t OH, int64_t OW, bool local = false) {
  Geometry best{1, 1, 1};
  double best_eff = -1.0;
  const int bw_max = (int)std::min<int64_t>(OW, kTileM);
  for (int bw = 1; bw <= bw_max; ++bw) {
    const int bh_max = (int)std::min<int64_t>(OH, kTileM / bw);
    for (int bh = 1; bh <= bh_max; ++bh) {
      const int bni_max = local ? 1 : (int)std::min<int64_t>(N, kTileM / (bw * bh));
      for (int bni = 1; bni <= bni_max; ++bni) {
        const double tiles =
            (double)neo_ceil_div(OW, bw) * neo_ceil_div(OH, bh) * neo_ceil_div(N, bni);
        const double eff = (double)N * OH * OW / (tiles * kTileM);
        const bool better = eff > best_eff + 1e-9 ||
                            (eff > best_eff - 1e-9 &&
                             (bw > best.BW || (bw == best.BW && bw * bh * bni > best.BW * best.BH * best.BNI)));
        if (better) {
          best_eff = eff;
          best = {bw, bh, bni};
        }
      }
    }
  }
  return best;
}

int pick_tile_n(int64_t K) {
  if (half_sm_mode()) {                  // 2 accumulators in 256 TMEM columns
    if (K <= 128) return (int)neo_ceil_div(K, 16) * 16;
    return 128;
  }
  if (K <= 256) return (int)neo_ceil_div(K, 16) * 16;
  int best = 256;
  int64_t best_waste = neo_ceil_div(K, 256) * 256 - K;
  for (int bn : {192, 128}) {
    int64_t waste = neo_ceil_div(K, bn) * bn - K;
    if (waste < best_waste) {
      best_waste = waste;
      best = bn;
    }
  }
  return best;
}

int pick_slices_per_stage(int64_t nslices, int rowb, int bn) {
  const int gmax = std::max(1, 256 / rowb);
  int best = (rowb == 16) ? 2 : 1;
  double best_cost = 1e30;
  for (int g = 1; g <= gmax; ++g) {
    if (rowb == 16 && (g & 1)) continue;
    const int64_t stage_bytes = (int64_t)g * (kTileM + bn) * rowb;
    if (stage_bytes > 60 * 1024 && g > ((rowb == 16) ? 2 : 1)) continue;
    const int64_t ks = neo_ceil_div(nslices, g);
    const double cost = (double)(ks * g) * rowb + (double)ks * 48.0;
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = g;
    }
  }
  return best;
}

// operand element bytes of a tensor-core mode
int mode_elem_size(int mode) {
  return mode == NEO_MODE_BF16 ? 2 : mode == NEO_MODE_FP8 ? 1 : 4;
}

}  // namespace

// exported for layout.cu / the ABI
int64_t neo_conv_umma_slices(int mode, int64_t c, int64_t r, int64_t s, int x,
                             int slices_per_stage) {
  // stage padding past nslices is served by TMA out-of-bounds zero fill, so
  // the image needs exactly R*S*ceil(C/x) slices whatever slices_per_stage is
  (void)mode;
  (void)slices_per_stage;
  if (x <= 0) return -1;
  return r * s * neo_ceil_div(c, x);
}

// epilogue groups = TMEM accumulator stages: four for short reductions
// (<= 8 slices: the tile time is the epilogue's, and four tiles draining in
// parallel hide its latency) when four N tiles fit the 512 TMEM columns,
// else two (long K loops want the shared memory for pipeline stages)
static int epi_groups(const neo_conv_params* p, int tile_n) {
  if (p->pro_scale) return 2;            // prologue mode: 8 epilogue warps, 2 groups
  if (half_sm_mode()) return 2;          // 8 epilogue warps, 2 x 128 TMEM columns
  static const int forced = getenv("NEOB200_EPI_GROUPS") ? atoi(getenv("NEOB200_EPI_GROUPS")) : 0;
  if (forced == 2 || (forced == 4 && tile_n <= 128)) return forced;
  const int64_t slices = p->r * p->s * neo_ceil_div(p->c, std::max(1, p->ic_bn));
  return tile_n <= 128 && slices <= 8 ? 4 : 2;
}

// Row bytes of one output channel block for the TMA-store epilogue, or 0 when
// the direct-store path must run: the block must be a 32/64/128-byte row of
// whole 16-column chunks and every N tile must hold whole channel blocks.
static int epi_rowb_out(const neo_conv_params* p, int tile_n) {
  const int out_es = (int)neo_dtype_size(p->out_dtype);
  const int y = p->oc_bn;
  const int rowb_out = y * out_es;
  // 16-byte rows (unswizzled staging): e4m3 blocks of 16 channels only (the
  // direct epilogue has no e4m3 store)
  const bool rows_ok = rowb_out == 32 || rowb_out == 64 || rowb_out == 128 ||
                       (rowb_out == 16 && p->out_dtype == NEO_FP8);
  const bool ok = y % 16 == 0 && rows_ok && tile_n % y == 0 && !getenv("NEOB200_DIRECT_EPILOGUE");
  return ok ? rowb_out : 0;
}

// stride-1 convs with a horizontal window, 128- or 64-byte rows (SW128 /
// SW64 shifted views: the swizzle follows absolute shared-memory address
// bits, so a view shifted by whole rows reads what TMA wrote) and a padded
// width that fits the 128-row M tile
static bool halo_format_ok(const neo_conv_params* p, int rowb) {
  static const bool disabled = getenv("NEOB200_NO_HALO") != nullptr;
  static const bool no64 = getenv("NEOB200_NO_HALO64") != nullptr;
  static const bool no32 = getenv("NEOB200_NO_HALO32") != nullptr;
  return !disabled && p->stride_h == 1 && p->stride_w == 1 && p->s > 1 &&
         (rowb == 128 || (rowb == 64 && !no64) || (rowb == 32 && !no32));
}
static bool halo_eligible(const neo_conv_params* p, int rowb, int64_t OW) {
  return halo_format_ok(p, rowb) && OW + p->s - 1 <= kTileM;
}
// Halo STRIPS (NEO_FLAG_HALO_STRIPS): maps wider than one 128-row tile
// (VGG's 224 / 112 maps, SSD's 128, Inception's 147) are cut into column
// strips of BWo output columns; a tile's band is BW = BWo + S - 1 input
// columns of BH (+ R - 1) rows, the S taps are the same shifted views, and the
// epilogue drops the S - 1 band columns past the strip (compacted staging
// rows, BWo-wide store / residual boxes).  Without strips those layers run
// plain tiles that fetch every tap's box separately (R*S-fold A traffic).
static bool halo_strips_on() {
  static const bool off = getenv("NEOB200_NO_HALO_STRIPS") != nullptr;
  return !off;
}
struct StripGeom { int BWo, BH; double eff; };
static StripGeom pick_strips(int64_t OH, int64_t OW, int S) {
  StripGeom best{0, 0, 0.0};
  const int ns0 = (int)neo_ceil_div(OW, kTileM - (S - 1));
  for (int ns = ns0; ns <= ns0 + 24; ++ns) {
    const int bwo = (int)neo_ceil_div(OW, ns);
    if (bwo < 8) break;
    const int bw = bwo + S - 1;
    const int bh = (int)std::min<int64_t>(OH, kTileM / bw);
    if (bh < 1) continue;
    const double eff = (double)OW * OH / ((double)neo_ceil_div(OW, bwo) * neo_ceil_div(OH, bh) * kTileM);
    // most useful rows; ties -> taller tiles (a band carries R - 1 extra rows)
    if (eff > best.eff + 1e-9 || (eff > best.eff - 1e-9 && bh > best.BH)) best = {bwo, bh, eff};
  }
  return best;
}
// halo bands are whole 1024-byte swizzle periods (8 rows of 128 B, 16 of
// 64 B): TMA's SWIZZLE_64B pattern is laid out on 1024-byte boundaries, and
// a 64-byte-row band of an odd number of 512-byte atoms misplaced every
// following stage / the weight image (measured: e4m3 64->128 3x3 tiles)
static int halo_row_align(const neo_conv_params* p) {
  const int es = p->mode == NEO_MODE_BF16 ? 2 : p->mode == NEO_MODE_FP8 ? 1 : 4;
  return std::max(8, 1024 / std::max(16, p->ic_bn * es));
}
static int halo_a_rows(const neo_conv_params* p) {
  const int al = halo_row_align(p);
  return (int)neo_ceil_div(kTileM + p->s - 1, al) * al;
}
// CTA-pair (cta_group::2) tiles: explicit cta_pair (2 on, 1 off) or
// NEOB200_PAIR=1; needs an unsplit reduction, at least two M tiles and an N
// tile whose halves are whole 16-row pieces
static bool use_pair(const neo_conv_params* p, int tile_n, int64_t m_tiles) {
  static const bool env_on = getenv("NEOB200_PAIR") && atoi(getenv("NEOB200_PAIR")) > 0;
  const bool want = p->cta_pair == 2 || (p->cta_pair == 0 && env_on);
  return want && p->split_k <= 1 && m_tiles >= 2 && tile_n % 32 == 0;
}
// weight rows one CTA holds per slice
static int b_rows(const neo_conv_params* p, int tile_n, int64_t m_tiles) {
  return use_pair(p, tile_n, m_tiles) ? tile_n / 2 : tile_n;
}
static int64_t halo_pair_bytes(const neo_conv_params* p, int rowb, int64_t m_tiles) {
  return (int64_t)halo_a_rows(p) * rowb + (int64_t)p->s * b_rows(p, p->tile_n, m_tiles) * rowb;
}

// weight-stationary (see ConvTCParams::wst): single-CTA tiles, unsplit
// reduction, no prologue; the resident image and the activation stage sizes
static bool wst_allowed(const neo_conv_params* p, int tile_n, int64_t m_tiles) {
  static const bool disabled = getenv("NEOB200_NO_WST") != nullptr;
  return !disabled && !p->pro_scale && p->split_k <= 1 && !use_pair(p, tile_n, m_tiles);
}
static int64_t wst_w_bytes(const neo_conv_params* p, bool halo, int rowb, int G, int tile_n) {
  const int64_t Cb = neo_ceil_div(p->c, p->ic_bn);
  if (halo) return p->r * p->s * Cb * (int64_t)tile_n * rowb;
  return neo_ceil_div(p->r * p->s * Cb, G) * G * (int64_t)tile_n * rowb;
}
// halo band: 128 rows read from the largest shift (R-1)*BW + S-1
static int wst_band_rows(const neo_conv_params* p, int BW) {
  const int al = halo_row_align(p);
  return (int)neo_ceil_div(kTileM + (p->r - 1) * BW + p->s - 1, al) * al;
}

int neo_conv_default_tiles(neo_conv_params* p) {
  NEO_CHECK_ARG(p != nullptr, NEO_ERR_INVALID_ARG, "null params");
  NEO_CHECK_ARG(p->struct_size == (int)sizeof(neo_conv_params), NEO_ERR_INVALID_ARG,
                "neo_conv_params.struct_size %d != %d", p->struct_size,
                (int)sizeof(neo_conv_params));
  if (p->mode == NEO_MODE_FP32) return NEO_OK;
  const int es = mode_elem_size(p->mode);
  const int rowb = p->ic_bn * es;
  const int64_t OH = conv_out_dim(p->h, p->r, p->stride_h, p->pad_h);
  const int64_t OW = conv_out_dim(p->w_in, p->s, p->stride_w, p->pad_w);
  NEO_CHECK_ARG(OH >= 1 && OW >= 1, NEO_ERR_SHAPE_MISMATCH, "conv has empty output");
  if (half_sm_mode() && p->tile_n > 128) p->tile_n = 128;   // 2 accumulators in 256 TMEM columns
  const bool auto_geom = p->tile_w <= 0 || p->tile_h <= 0 || p->tile_img <= 0;
  const bool auto_tn = p->tile_n <= 0;
  Geometry g0{0, 0, 0};
  if (auto_geom) {
    Geometry g = pick_geometry(p->n, OH, OW);
    if (g.BNI > 1 && g.BW * g.BH < 16 && p->r * p->s > 1 && OW >= 64 &&
        (p->mode != NEO_MODE_FP8 || rowb >= 64)) {
      // image-scattered tile on a large windowed map: keep the tile's pixels
      // in one image when that still fills >= 85% of the MMA rows (e4m3 maps
      // of <= 32 channels -- 16/32-byte rows -- measured 4-10% faster
      // scattered, so they keep the unrestricted pick)
      const Geometry gl = pick_geometry(p->n, OH, OW, true);
      const double eff_l = (double)OW * OH /
                           ((double)neo_ceil_div(OW, gl.BW) * neo_ceil_div(OH, gl.BH) * kTileM);
      if (eff_l >= 0.85) g = gl;
    }
    g0 = g;
    p->tile_w = g.BW;
    p->tile_h = g.BH;
    p->tile_img = g.BNI;
    // halo strips only where the full padded width does not fit one tile:
    // forcing them onto 112 / 56 / 28-wide maps (taller bands, fewer band
    // rows per output) measured 0-3% slower than full-width halo tiles
    const bool strips_ok = halo_strips_on() && halo_format_ok(p, rowb) && p->tile_n <= 0 &&
                           p->slices_per_stage <= 0 && p->stages <= 0 && p->split_k <= 1 &&
                           p->cta_pair != 2 && !p->pro_scale;
    // 32-byte rows (SW32 shifted views: bf16 maps of 16 channels, Inception's
    // 48 / 80-channel tensors) joined the halo mainloop after the schedule DB
    // was tuned, so they only take it when no explicit tile parameter (tuned
    // for plain tiles) comes with the launch
    if (halo_eligible(p, rowb, OW) && (rowb != 32 || strips_ok)) {
      // halo tiles: full padded width, as many output rows as fit in 128
      const int bwp = (int)(OW + p->s - 1);
      const int bh = (int)std::min<int64_t>(OH, kTileM / bwp);
      const double eff_h = (double)OW * OH / ((double)neo_ceil_div(OH, bh) * kTileM);
      // a width that fills little of the 128 rows (71 of 128 at 73 padded
      // columns) is better cut into strips; at equal fill full-width tiles
      // measured 0-3% faster
      const StripGeom sg = strips_ok ? pick_strips(OH, OW, (int)p->s) : StripGeom{0, 0, 0.0};
      if (sg.BWo > 0 && sg.BWo < OW && sg.eff >= eff_h + 0.08) {
        p->tile_w = sg.BWo + (int)p->s - 1;
        p->tile_h = sg.BH;
        p->tile_img = 1;
        p->flags |= NEO_FLAG_HALO_STRIPS;
      } else {
        const double eff_s = (double)OW * OH * p->n /
                             ((double)neo_ceil_div(OW, g.BW) * neo_ceil_div(OH, g.BH) *
                              neo_ceil_div(p->n, g.BNI) * kTileM);
        // the band reuse cuts A traffic ~S-fold, which outweighs idle rows
        if (eff_h >= 0.35 * eff_s) {
          p->tile_w = bwp;
          p->tile_h = bh;
          p->tile_img = 1;
        }
      }
    } else if (strips_ok && OW + p->s - 1 > kTileM) {
      // wide map, nothing but the geometry left to the kernel: halo strips
      // (explicit tile parameters were tuned for plain tiles and keep them)
      const StripGeom sg = pick_strips(OH, OW, (int)p->s);
      if (sg.BWo > 0 && sg.eff >= 0.7) {
        p->tile_w = sg.BWo + (int)p->s - 1;
        p->tile_h = sg.BH;
        p->tile_img = 1;
        p->flags |= NEO_FLAG_HALO_STRIPS;
      }
    }
  }
  const bool strips = (p->flags & NEO_FLAG_HALO_STRIPS) != 0;
  bool halo = p->tile_w > OW || strips;   // halo geometry: wider than the output, or strips
  int64_t m_tiles = neo_ceil_div(OW, strips ? p->tile_w - (p->s - 1) : p->tile_w) *
                    neo_ceil_div(OH, p->tile_h) * neo_ceil_div(p->n, p->tile_img);
  const int64_t budget = smem_budget() - 2048 - kMaxGroups * kParamFloats * 4;
  auto staging_of = [&](int tn) -> int64_t {
    const int rbo = epi_rowb_out(p, tn);
    return rbo ? (int64_t)epi_groups(p, tn) * kTileM * rbo * (tn / std::max(1, p->oc_bn)) : 0;
  };
  if (p->tile_n <= 0) {
    // widest N tile that still gives every SM at least one tile (halo
    // stages carry S weight slices, so their N tile stops at 128)
    // short reductions are epilogue-bound: cap at 128 so four epilogue
    // groups (TMEM stages) can drain tiles in parallel
    const int64_t red_slices = p->r * p->s * neo_ceil_div(p->c, std::max(1, p->ic_bn));
    const int widest = (halo || red_slices <= 8 || p->pro_scale) ? std::min(128, pick_tile_n(p->k))
                                                                 : pick_tile_n(p->k);
    p->tile_n = widest;
    // the TMA-store epilogue needs whole output channel blocks per N tile
    const int min_bn = (p->oc_bn % 16 == 0 && p->oc_bn <= widest) ? p->oc_bn : 16;
    for (int bn : {256, 128, 64}) {
      if (bn > widest || bn < min_bn) continue;
      p->tile_n = bn;
      if (m_tiles * neo_ceil_div(p->k, bn) >= sm_count_of_current_device()) break;
    }
    if (p->tile_n > widest) p->tile_n = widest;
  }
  if (halo) {
    // a halo stage carries S weight slices: two stages must fit beside the
    // epilogue staging (wide kernels such as 1x7 shrink the N tile first,
    // then fall back to plain tiles)
    auto fits = [&]() {
      return 2 * halo_pair_bytes(p, rowb, m_tiles) + staging_of(p->tile_n) <= budget;
    };
    // (never below one output channel block: the TMA-store epilogue -- the
    // only e4m3 store -- needs whole blocks per N tile)
    const int floor_tn = (p->oc_bn % 16 == 0 && p->oc_bn > 32) ? p->oc_bn : 32;
    while (!fits() && auto_tn && p->tile_n > floor_tn) p->tile_n /= 2;
    if (!fits() && auto_geom) {
      p->tile_w = g0.BW;
      p->tile_h = g0.BH;
      p->tile_img = g0.BNI;
      p->flags &= ~NEO_FLAG_HALO_STRIPS;
      halo = false;
      m_tiles = neo_ceil_div(OW, p->tile_w) * neo_ceil_div(OH, p->tile_h) *
                neo_ceil_div(p->n, p->tile_img);
      if (auto_tn) {
        p->tile_n = pick_tile_n(p->k);
        const int min_bn = (p->oc_bn % 16 == 0 && p->oc_bn <= p->tile_n) ? p->oc_bn : 16;
        for (int bn : {256, 128, 64}) {
          if (bn > pick_tile_n(p->k) || bn < min_bn) continue;
          p->tile_n = bn;
          if (m_tiles * neo_ceil_div(p->k, bn) >= sm_count_of_current_device()) break;
        }
      }
    }
  }
  const int64_t nslices = halo ? p->r * neo_ceil_div(p->c, p->ic_bn)
                               : p->r * p->s * neo_ceil_div(p->c, p->ic_bn);
  // pipeline: keep the full epilogue staging (every output block of a tile
  // in smem, so residual loads are issued before the accumulator is ready)
  // and as many stages as fit, shrinking slices per stage if needed
  const int64_t staging = staging_of(p->tile_n);
  // split-K when the (M, N) tiles leave most SMs idle: single-slice stages
  // give the splits fine granularity
  const int sms = sm_count_of_current_device();
  const int64_t base_units = m_tiles * neo_ceil_div(p->k, p->tile_n);
  // automatic split-K is opt-in (NEOB200_AUTO_SPLITK): measured on B200 the
  // partial-sum exchange still costs more than the idle SMs it recovers for
  // most under-filled layers, so split_k is a tuner / caller choice
  static const bool auto_split = getenv("NEOB200_AUTO_SPLITK") != nullptr;
  const bool underfilled = p->split_k <= 0 && base_units * 2 <= sms && auto_split;
  if (underfilled && p->slices_per_stage <= 0) p->slices_per_stage = rowb == 16 ? 2 : 1;
  // weight-stationary when the whole N block's weights fit beside the
  // staging and >= 3 activation stages (2 when explicitly asked for)
  bool wst = false;
  if (p->weight_stationary != 1 && !underfilled && wst_allowed(p, p->tile_n, m_tiles)) {
    const int g = p->slices_per_stage > 0 ? p->slices_per_stage
                                          : (halo ? 1 : pick_slices_per_stage(nslices, rowb, p->tile_n));
    const int64_t wb = wst_w_bytes(p, halo, rowb, g, p->tile_n);
    const int64_t ast = halo ? (int64_t)wst_band_rows(p, p->tile_w) * rowb : (int64_t)g * kTileM * rowb;
    const int64_t kst = halo ? neo_ceil_div(p->c, p->ic_bn) : neo_ceil_div(nslices, g);
    const int64_t want = std::min<int64_t>(6, std::max<int64_t>(3, kst + 2));
    // an explicit depth may squeeze the epilogue staging to one slot per group
    const int rbo = epi_rowb_out(p, p->tile_n);
    const int64_t min_staging = rbo ? (int64_t)epi_groups(p, p->tile_n) * kTileM * rbo : 0;
    const int64_t fit = (budget - (p->stages > 0 ? min_staging : staging) - wb) / ast;
    if ((!halo || g == 1) && fit >= std::max(p->stages, p->weight_stationary == 2 ? 2 : 3)) {
      wst = true;
      p->slices_per_stage = g;
      if (p->stages <= 0) p->stages = (int)std::min<int64_t>({want, fit, kMaxStages});
      p->split_k = 1;
    }
  }
  p->weight_stationary = wst ? 2 : 1;
  if (!wst && (p->slices_per_stage <= 0 || p->stages <= 0)) {
    int g = p->slices_per_stage > 0 ? p->slices_per_stage
                                    : (halo ? 1 : pick_slices_per_stage(nslices, rowb, p->tile_n));
    const int gmin = rowb == 16 ? 2 : 1;
    for (;;) {
      const int64_t stage = halo ? (int64_t)g * halo_pair_bytes(p, rowb, m_tiles)
                                 : (int64_t)g * (kTileM + b_rows(p, p->tile_n, m_tiles)) * rowb;
      const int64_t kst = neo_ceil_div(nslices, g);
      const int64_t want = kst <= 1 ? 2 : std::min<int64_t>(6, kst + 1);
      const int64_t fit = (budget - staging) / stage;
      if (fit >= std::min<int64_t>(want, 3) || g <= gmin || p->slices_per_stage > 0) {
        p->slices_per_stage = g;
        if (p->stages <= 0) {
          // else shrink the staging, but keep one slot per epilogue group so
          // the TMA-store epilogue survives (the direct path is far slower)
          const int rbo = epi_rowb_out(p, p->tile_n);
          const int64_t min_staging =
              rbo ? (int64_t)epi_groups(p, p->tile_n) * kTileM * rbo : 0;
          const int64_t room = fit >= 2 ? fit : (budget - min_staging) / stage;
          p->stages = (int)std::max<int64_t>(2, std::min<int64_t>(want, room));
        }
        break;
      }
      g = std::max(gmin, g / 2);
    }
  }
  if (p->split_k <= 0) {
    int64_t split = 1;
    if (underfilled) {
      const int64_t kst = neo_ceil_div(nslices, p->slices_per_stage);
      split = std::min<int64_t>({sms / std::max<int64_t>(1, base_units), kst / 4, 32});
      if (split < 2) split = 1;
    }
    p->split_k = (int)split;
  }
  return NEO_OK;
}

namespace {
struct SplitPlan {
  int splits, kps;
  int64_t ws_bytes;
};
SplitPlan split_plan(const neo_conv_params* p, int64_t kstages, int64_t num_tiles) {
  SplitPlan sp{1, (int)kstages, 0};
  const int64_t want = std::max(1, std::min<int>(p->split_k, (int)kstages));
  // every unit of a split launch must be resident at once (units wait for
  // their tile's other splits): at most one unit per SM
  const int64_t cap = std::max<int64_t>(1, sm_count_of_current_device() / std::max<int64_t>(1, num_tiles));
  const int64_t want_c = std::min<int64_t>(want, cap);
  if (want_c > 1) {
    sp.kps = (int)neo_ceil_div(kstages, want_c);
    sp.splits = (int)neo_ceil_div(kstages, sp.kps);
    sp.ws_bytes = sp.splits > 1 ? neo_ceil_div(num_tiles * 4, 256) * 256 +
                                      num_tiles * sp.splits * (int64_t)p->tile_n * kTileM * 4
                                : 0;
  }
  return sp;
}
int64_t conv_kstages(const neo_conv_params* p, bool halo) {
  const int64_t Cb = neo_ceil_div(p->c, p->ic_bn);
  const int64_t nslices = halo ? p->r * Cb : p->r * p->s * Cb;
  return neo_ceil_div(nslices, p->slices_per_stage);
}
int64_t conv_num_tiles(const neo_conv_params* p) {
  const int64_t OH = conv_out_dim(p->h, p->r, p->stride_h, p->pad_h);
  const int64_t OW = conv_out_dim(p->w_in, p->s, p->stride_w, p->pad_w);
  const int64_t bwo = (p->flags & NEO_FLAG_HALO_STRIPS) ? p->tile_w - (p->s - 1) : p->tile_w;
  return neo_ceil_div(OW, bwo) * neo_ceil_div(OH, p->tile_h) *
         neo_ceil_div(p->n, p->tile_img) * neo_ceil_div(p->k, p->tile_n);
}
}  // namespace

// bytes of split-K workspace the launch of *p needs (0: no split)
int neo_conv_workspace_bytes(const neo_conv_params* pin, int64_t* bytes) {
  NEO_CHECK_ARG(pin != nullptr && bytes != nullptr, NEO_ERR_INVALID_ARG, "null argument");
  NEO_CHECK_ARG(pin->struct_size == (int)sizeof(neo_conv_params), NEO_ERR_INVALID_ARG,
                "neo_conv_params.struct_size %d != %d", pin->struct_size,
                (int)sizeof(neo_conv_params));
  *bytes = 0;
  if (pin->mode == NEO_MODE_FP32) return NEO_OK;
  neo_conv_params pc = *pin;
  const int st = neo_conv_default_tiles(&pc);
  if (st != NEO_OK) return st;
  const int64_t OW = conv_out_dim(pc.w_in, pc.s, pc.stride_w, pc.pad_w);
  const bool halo = pc.tile_w > OW || (pc.flags & NEO_FLAG_HALO_STRIPS);
  *bytes = split_plan(&pc, conv_kstages(&pc, halo), conv_num_tiles(&pc)).ws_bytes;
  return NEO_OK;
}

int neo_conv_tc_launch(const neo_conv_params* pin, cudaStream_t stream) {
  neo_conv_params pc = *pin;
  int st = neo_conv_default_tiles(&pc);
  if (st != NEO_OK) return st;
  const neo_conv_params* p = &pc;
  const bool tf32 = p->mode == NEO_MODE_TF32;
  const bool fp8 = p->mode == NEO_MODE_FP8;
  const int kind = tf32 ? kKindTF32 : fp8 ? kKindFP8
                   : p->out_dtype == NEO_FP8 ? kKindBF16Q : kKindBF16;
  const int es = mode_elem_size(p->mode);
  const int x = p->ic_bn;
  const int rowb = x * es;
  NEO_CHECK_ARG(rowb == 16 || rowb == 32 || rowb == 64 || rowb == 128, NEO_ERR_UNSUPPORTED,
                "tensor-core conv needs ic_bn*sizeof in {16,32,64,128} bytes (ic_bn=%d, %s)", x,
                tf32 ? "tf32" : fp8 ? "fp8" : "bf16");
  NEO_CHECK_ARG(p->out_dtype == NEO_F32 || !tf32, NEO_ERR_UNSUPPORTED, "tf32 mode writes f32");
  // e4m3 outputs: NEO_MODE_FP8 convs, or a bf16 conv entering an fp8 chain
  // (e.g. a 3-channel image stem folded to bf16); residuals stay e4m3
  NEO_CHECK_ARG(p->out_dtype != NEO_FP8 || !tf32, NEO_ERR_UNSUPPORTED,
                "e4m3 outputs come from NEO_MODE_FP8 or NEO_MODE_BF16 convs");
  NEO_CHECK_ARG(p->out_dtype == NEO_F32 || p->out_dtype == NEO_BF16 || p->out_dtype == NEO_FP8,
                NEO_ERR_INVALID_ARG, "bad out_dtype %d", p->out_dtype);
  if (fp8) {
    // e4m3 tiles: unsplit reductions, no smem prologue (the split-K fixup
    // and the BN-ReLU rewrite only know bf16 / f32 operands)
    NEO_CHECK_ARG(p->pro_scale == nullptr, NEO_ERR_UNSUPPORTED, "no BN-ReLU prologue in fp8 mode");
    NEO_CHECK_ARG(p->split_k <= 1, NEO_ERR_SCHEDULE_INVALID, "no split-K in fp8 mode");
  }
  const int64_t OH = conv_out_dim(p->h, p->r, p->stride_h, p->pad_h);
  const int64_t OW = conv_out_dim(p->w_in, p->s, p->stride_w, p->pad_w);
  const int BW = p->tile_w, BH = p->tile_h, BNI = p->tile_img, BN = p->tile_n;
  NEO_CHECK_ARG(BW * BH * BNI <= kTileM && BW >= 1 && BH >= 1 && BNI >= 1, NEO_ERR_SCHEDULE_INVALID,
                "M tile %dx%dx%d exceeds 128 pixels", BW, BH, BNI);
  NEO_CHECK_ARG(BN % 16 == 0 && BN >= 16 && BN <= 256, NEO_ERR_SCHEDULE_INVALID,
                "tile_n=%d must be a multiple of 16 in [16,256]", BN);
  NEO_CHECK_ARG(BW * p->stride_w <= 256 && BH * p->stride_h <= 256 && p->stride_w <= 8 &&
                    p->stride_h <= 8,
                NEO_ERR_UNSUPPORTED, "TMA box too large for stride");
  const int G = p->slices_per_stage;
  NEO_CHECK_ARG(G >= 1 && (rowb != 16 || G % 2 == 0), NEO_ERR_SCHEDULE_INVALID,
                "slices_per_stage=%d invalid for %d-byte rows", G, rowb);
  NEO_CHECK_ARG(p->stages >= 2 && p->stages <= kMaxStages, NEO_ERR_SCHEDULE_INVALID,
                "stages=%d outside [2,%d] (stage too large for shared memory?)", p->stages,
                kMaxStages);

  const int64_t Cb = neo_ceil_div(p->c, x);
  const int64_t cbt = p->x_cb_total > 0 ? p->x_cb_total : Cb;
  const bool strips = (p->flags & NEO_FLAG_HALO_STRIPS) != 0;
  const bool halo = BW > OW || strips;
  const bool wst = p->weight_stationary == 2;
  const int BWo = strips ? BW - (int)(p->s - 1) : BW;   // output columns per tile
  NEO_CHECK_ARG(!halo || (strips ? halo_format_ok(p, rowb) : halo_eligible(p, rowb, OW)),
                NEO_ERR_SCHEDULE_INVALID,
                "tile_w=%d wider than the output needs a stride-1, 128-byte-row conv", BW);
  NEO_CHECK_ARG(!halo || strips || (BW == OW + p->s - 1 && BNI == 1), NEO_ERR_SCHEDULE_INVALID,
                "halo tiles must span the padded width OW+S-1 of one image");
  NEO_CHECK_ARG(!strips || (BWo >= 1 && BNI == 1 && p->split_k <= 1 && p->cta_pair != 2 &&
                            !p->pro_scale),
                NEO_ERR_SCHEDULE_INVALID,
                "halo strips: one image per tile, no split-K / CTA pair / prologue");
  const int64_t nslices = halo ? (wst ? Cb : p->r * Cb) : p->r * p->s * Cb;
  NEO_CHECK_ARG(!(wst && halo && G != 1), NEO_ERR_SCHEDULE_INVALID,
                "weight-stationary halo tiles take one channel block per stage");
  const int64_t kstages = neo_ceil_div(nslices, G);

  if (p->pro_scale) {
    // BN-ReLU prologue: 1x1, unpadded, whole channel blocks, N tile <= 128
    NEO_CHECK_ARG(p->pro_shift != nullptr, NEO_ERR_INVALID_ARG, "prologue needs scale and shift");
    NEO_CHECK_ARG(p->r == 1 && p->s == 1 && p->pad_h == 0 && p->pad_w == 0 && p->c % x == 0,
                  NEO_ERR_UNSUPPORTED,
                  "BN-ReLU prologue needs an unpadded 1x1 conv over whole channel blocks");
    NEO_CHECK_ARG(BN <= 128 && p->cta_pair != 2, NEO_ERR_SCHEDULE_INVALID,
                  "BN-ReLU prologue runs single-CTA tiles with tile_n <= 128 (tile_n=%d)", BN);
  }
  const int64_t tiles_m_all = neo_ceil_div(OW, BWo) * neo_ceil_div(OH, BH) * neo_ceil_div(p->n, BNI);
  const bool pair = !p->pro_scale && use_pair(p, BN, tiles_m_all);
  NEO_CHECK_ARG(!wst || wst_allowed(p, BN, tiles_m_all), NEO_ERR_SCHEDULE_INVALID,
                "weight-stationary tiles need single-CTA tiles, no split-K, no prologue");
  NEO_CHECK_ARG(!(p->cta_pair == 2 && !pair), NEO_ERR_SCHEDULE_INVALID,
                "cta_pair not possible here (split_k=%d, tile_n=%d, %lld M tiles)", p->split_k,
                BN, (long long)tiles_m_all);
  const int bro = pair ? BN / 2 : BN;       // weight rows this CTA loads per slice

  ConvTCParams kp;
  memset(&kp, 0, sizeof(kp));
  auto encode = get_encode_fn();
  NEO_CHECK_ARG(encode != nullptr, NEO_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const CUtensorMapDataType dt = tf32  ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : fp8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                       : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  {
    const char* base = static_cast<const char*>(p->x) + (size_t)p->x_cb_offset * p->h * p->w_in * rowb;
    cuuint64_t dims[5] = {(cuuint64_t)x, (cuuint64_t)p->w_in, (cuuint64_t)p->h, (cuuint64_t)Cb,
                          (cuuint64_t)p->n};
    cuuint64_t strides[4] = {(cuuint64_t)rowb, (cuuint64_t)p->w_in * rowb,
                             (cuuint64_t)p->h * p->w_in * rowb,
                             (cuuint64_t)cbt * p->h * p->w_in * rowb};
    cuuint32_t box[5] = {(cuuint32_t)x, (cuuint32_t)(BW * p->stride_w),
                         (cuuint32_t)(BH * p->stride_h + (halo && wst ? p->r - 1 : 0)), 1u,
                         (cuuint32_t)BNI};
    // halo: box = BH rows of the padded width (stride 1), i.e. BH*BW pixels
    cuuint32_t estr[5] = {1u, (cuuint32_t)p->stride_w, (cuuint32_t)p->stride_h, 1u, 1u};
    CUresult r = encode(&kp.tmA, dt, 5, const_cast<char*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_code_tma(rowb),
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    NEO_CHECK_ARG(r == CUDA_SUCCESS, NEO_ERR_CUDA, "tensor map A encode failed (%d)", (int)r);
  }
  if (halo) {
    // weight image viewed as (x, K, Cb, R*S); one box = the S taps of (r, cb)
    cuuint64_t dims[4] = {(cuuint64_t)x, (cuuint64_t)p->k, (cuuint64_t)Cb,
                          (cuuint64_t)(p->r * p->s)};
    cuuint64_t strides[3] = {(cuuint64_t)rowb, (cuuint64_t)p->k * rowb,
                             (cuuint64_t)Cb * p->k * rowb};
    cuuint32_t box[4] = {(cuuint32_t)x, (cuuint32_t)bro, 1u, (cuuint32_t)p->s};
    cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
    CUresult r = encode(&kp.tmB, dt, 4, const_cast<void*>(p->w), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_code_tma(rowb),
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    NEO_CHECK_ARG(r == CUDA_SUCCESS, NEO_ERR_CUDA, "tensor map B encode failed (%d)", (int)r);
  } else {
    // slices past nslices (stage padding) are out of bounds -> zero filled
    cuuint64_t dims[3] = {(cuuint64_t)x, (cuuint64_t)p->k, (cuuint64_t)nslices};
    cuuint64_t strides[2] = {(cuuint64_t)rowb, (cuuint64_t)p->k * rowb};
    cuuint32_t box[3] = {(cuuint32_t)x, (cuuint32_t)bro, (cuuint32_t)G};
    cuuint32_t estr[3] = {1u, 1u, 1u};
    CUresult r = encode(&kp.tmB, dt, 3, const_cast<void*>(p->w), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_code_tma(rowb),
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    NEO_CHECK_ARG(r == CUDA_SUCCESS, NEO_ERR_CUDA, "tensor map B encode failed (%d)", (int)r);
  }
  kp.N = (int)p->n;
  kp.OH = (int)OH;
  kp.OW = (int)OW;
  kp.K = (int)p->k;
  kp.BW = BW;
  kp.BWo = BWo;
  kp.BH = BH;
  kp.BNI = BNI;
  kp.BN = BN;
  kp.tiles_w = (int)neo_ceil_div(OW, BWo);
  kp.tiles_h = (int)neo_ceil_div(OH, BH);
  kp.tiles_k = (int)neo_ceil_div(p->k, BN);
  const int64_t tiles_n = neo_ceil_div(p->n, BNI);
  const int64_t num_tiles = (int64_t)kp.tiles_w * kp.tiles_h * tiles_n * kp.tiles_k;
  NEO_CHECK_ARG(num_tiles < (1ll << 31), NEO_ERR_UNSUPPORTED, "too many tiles");
  kp.num_tiles = (int)num_tiles;
  {
    SplitPlan sp = split_plan(p, kstages, num_tiles);
    if (sp.splits > 1 && (p->workspace == nullptr || p->workspace_bytes < sp.ws_bytes)) {
      NEO_CHECK_ARG(pin->split_k <= 1, NEO_ERR_INVALID_ARG,
                    "split_k=%d needs a %lld-byte workspace", pin->split_k,
                    (long long)sp.ws_bytes);
      sp = SplitPlan{1, (int)kstages, 0};   // automatic split without workspace: none
    }
    kp.splits = sp.splits;
    kp.kps = sp.kps;
    kp.counters = static_cast<int*>(p->workspace);
    kp.ws = sp.splits > 1 ? reinterpret_cast<float*>(static_cast<char*>(p->workspace) +
                                                     neo_ceil_div(num_tiles * 4, 256) * 256)
                          : nullptr;
    NEO_CHECK_ARG(num_tiles * sp.splits < (1ll << 31), NEO_ERR_UNSUPPORTED, "too many units");
    kp.num_units = (int)(num_tiles * sp.splits);
    NEO_CHECK_ARG(!wst || sp.splits == 1, NEO_ERR_SCHEDULE_INVALID,
                  "weight-stationary tiles need an unsplit reduction");
    NEO_CHECK_ARG(!pair || sp.splits == 1, NEO_ERR_SCHEDULE_INVALID,
                  "CTA-pair tiles need an unsplit reduction");
    kp.pair = pair ? 1 : 0;
    kp.tiles_m = (int)tiles_m_all;
    kp.num_groups = pair ? (int)(kp.tiles_k * neo_ceil_div(tiles_m_all, 2)) : kp.num_units;
  }
  kp.G = G;
  kp.kstages = (int)kstages;
  kp.Cb = (int)Cb;
  kp.S = (int)p->s;
  kp.nslices = (int)nslices;
  kp.stride_h = p->stride_h;
  kp.stride_w = p->stride_w;
  kp.pad_h = p->pad_h;
  kp.pad_w = p->pad_w;
  kp.rowb = rowb;
  kp.swz = swizzle_code_umma(rowb);
  kp.stages = p->stages;
  kp.halo = halo ? 1 : 0;
  kp.R = (int)p->r;
  {
    static const char* bo = getenv("NEOB200_HALO_BASEOFF");
    kp.halo_baseoff = bo ? atoi(bo) : 0;  // swizzle follows absolute address bits
  }
  if (halo && wst) {
    kp.a_sub = (uint32_t)(wst_band_rows(p, BW) * rowb);
    kp.b_sub = (uint32_t)(p->s * BN * rowb);
    kp.tx_bytes = (uint32_t)((BH + p->r - 1) * BW * rowb);
  } else if (halo) {
    kp.a_sub = (uint32_t)(halo_a_rows(p) * rowb);
    kp.b_sub = (uint32_t)(p->s * bro * rowb);
    kp.tx_bytes = (uint32_t)((pair ? 2 : 1) * G * (BW * BH * rowb + p->s * bro * rowb));
  } else {
    kp.a_sub = (uint32_t)(kTileM * rowb);
    kp.b_sub = (uint32_t)(bro * rowb);
    kp.tx_bytes = (uint32_t)((pair ? 2 : 1) * G * (BW * BH * BNI * rowb + (wst ? 0 : bro * rowb)));
  }
  kp.a_stage = kp.a_sub * G;
  kp.b_stage = kp.b_sub * G;
  kp.wst = wst ? 1 : 0;
  kp.static_w = (p->flags & NEO_FLAG_STATIC_WEIGHTS) ? 1 : 0;
  {
    static const char* dbg = getenv("NEOB200_DBG");
    kp.dbg = dbg ? atoi(dbg) : 0;
    static int slot = 0;
    if (kp.dbg & 256) kp.dbg_slot = slot++;
  }
  kp.b_region = wst ? (halo ? (uint32_t)(p->r * Cb) * kp.b_sub : (uint32_t)kstages * kp.b_stage)
                    : (uint32_t)p->stages * kp.b_stage;
  kp.ngroups = epi_groups(p, BN);
  uint32_t cols = 32;
  while (cols < (uint32_t)(kp.ngroups * BN)) cols <<= 1;
  kp.tmem_cols = cols;
  NEO_CHECK_ARG(!half_sm_mode() || cols <= 256, NEO_ERR_SCHEDULE_INVALID,
                "half-SM mode: tile_n=%d needs %u TMEM columns (> 256)", BN, cols);
  kp.epi_warps = half_sm_mode() && !p->pro_scale ? 8 : kEpiWarps;
  const int threads = half_sm_mode() && !p->pro_scale ? 32 * (2 + 8) : kThreads;
  kp.scale = p->scale;
  kp.shift = p->shift;
  kp.bias = p->bias;
  kp.res = p->residual;
  kp.out = p->out;
  kp.y = p->oc_bn;
  const int64_t kbt = neo_ceil_div(p->k_split > 0 ? p->k_split : p->k, p->oc_bn);
  kp.out_cb_off = p->out_cb_offset;
  kp.out_cb_total = p->out_cb_total > 0 ? p->out_cb_total : (int)kbt;
  kp.res_cb_off = p->res_cb_offset;
  kp.res_cb_total = p->res_cb_total > 0 ? p->res_cb_total : (int)kbt;
  kp.relu = p->relu;
  if (p->k_split > 0) {
    // two outputs: channels [0, k_split) -> out, [k_split, k) -> out2
    NEO_CHECK_ARG(p->out2 != nullptr && p->k_split < p->k && p->k_split % BN == 0 &&
                      p->k_split % p->oc_bn == 0 && (p->k - p->k_split) % p->oc_bn == 0,
                  NEO_ERR_SCHEDULE_INVALID,
                  "second output needs k_split (%lld) a multiple of the N tile (%d) below K",
                  (long long)p->k_split, BN);
    NEO_CHECK_ARG(!p->residual && !pair && !p->pro_scale && kp.splits == 1, NEO_ERR_UNSUPPORTED,
                  "two-output convs take no residual, CTA pair, prologue or split-K");
    NEO_CHECK_ARG(p->out2_cb_total >= 1 &&
                      p->out2_cb_offset + (p->k - p->k_split) / p->oc_bn <= p->out2_cb_total,
                  NEO_ERR_SHAPE_MISMATCH, "second output window out of range");
    kp.k_split = (int)p->k_split;
    kp.relu2 = p->relu2;
    kp.out2_cb_off = p->out2_cb_offset;
  }
  kp.out_f32 = p->out_dtype == NEO_F32;
  kp.out_kind = p->out_dtype == NEO_F32 ? kOutF32 : p->out_dtype == NEO_FP8 ? kOutFP8 : kOutBF16;
  {
    auto inv = [](float sc) { return sc > 0.f ? (float)(1.0 / (double)sc) : 1.f; };
    kp.res_scale = p->res_scale > 0.f ? p->res_scale : 1.f;
    kp.out_qscale = inv(p->out_scale);
    kp.out2_qscale = inv(p->out2_scale);
  }
  kp.round_tf32 = (p->flags & NEO_FLAG_ROUND_TF32) ? 1 : 0;
  kp.pro = p->pro_scale != nullptr;
  kp.pro_scale = p->pro_scale;
  kp.pro_shift = p->pro_shift;
  kp.pro_relu = p->pro_relu;

  // TMA-store epilogue: output / residual tensor maps over (y, OW, OH, Kb_total, N)
  const int rb_out = epi_rowb_out(p, BN);
  {
    const int64_t left = smem_budget() - 2048 - kMaxGroups * kParamFloats * 4 -
                         (int64_t)p->stages * kp.a_stage - kp.b_region;
    const int64_t slots = rb_out ? left / ((int64_t)kp.ngroups * kTileM * rb_out) : 0;
    const int64_t per_tile = BN / std::max(1, p->oc_bn);
    static const bool no_pf = getenv("NEOB200_NO_RES_PREFETCH") != nullptr;
    kp.res_pf = (!no_pf && p->residual && !pair && kp.splits == 1 && slots >= 2 * per_tile && per_tile >= 1 &&
                 p->k % BN == 0) ? 1 : 0;
    kp.nslot = (int)std::min<int64_t>(slots, (kp.res_pf ? 2 : 1) * per_tile);
  }
  kp.tma_epi = rb_out > 0 && kp.nslot >= 1;
  NEO_CHECK_ARG(kp.tma_epi || p->out_dtype != NEO_FP8, NEO_ERR_UNSUPPORTED,
                "e4m3 outputs need the TMA-store epilogue (oc_bn rows of 32/64/128 bytes, "
                "whole channel blocks per N tile)");
  {
    static const bool no_share = getenv("NEOB200_NO_SHARE_LAST") != nullptr;
    kp.share_last = (!no_share && kp.tma_epi && kp.splits == 1 && !pair && !p->pro_scale &&
                     kp.ngroups >= 2) ? 1 : 0;
  }
  NEO_CHECK_ARG(kp.tma_epi || !kp.k_split, NEO_ERR_UNSUPPORTED,
                "two-output convs need the TMA-store epilogue (oc_bn rows of 32/64/128 bytes)");
  if (kp.tma_epi) {
    const int y = p->oc_bn;
    kp.rowb_out = rb_out;
    kp.stage_out = (uint32_t)(kTileM * kp.rowb_out);
    kp.out_box_bytes = (uint32_t)(BWo * BH * BNI * kp.rowb_out);
    const CUtensorMapDataType odt = kp.out_f32                  ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                    : kp.out_kind == kOutFP8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                                             : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    cuuint32_t box[5] = {(cuuint32_t)y, (cuuint32_t)BWo, (cuuint32_t)BH, 1u, (cuuint32_t)BNI};
    cuuint32_t estr[5] = {1u, 1u, 1u, 1u, 1u};
    auto encode_fm = [&](CUtensorMap* map, const void* base, int64_t cb_total) {
      cuuint64_t dims[5] = {(cuuint64_t)y, (cuuint64_t)OW, (cuuint64_t)OH, (cuuint64_t)cb_total,
                            (cuuint64_t)p->n};
      cuuint64_t strides[4] = {(cuuint64_t)kp.rowb_out, (cuuint64_t)OW * kp.rowb_out,
                               (cuuint64_t)OH * OW * kp.rowb_out,
                               (cuuint64_t)cb_total * OH * OW * kp.rowb_out};
      return encode(map, odt, 5, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_code_tma(kp.rowb_out),
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    CUresult r = encode_fm(&kp.tmO, p->out, kp.out_cb_total);
    NEO_CHECK_ARG(r == CUDA_SUCCESS, NEO_ERR_CUDA, "tensor map O encode failed (%d)", (int)r);
    if (kp.k_split) {
      r = encode_fm(&kp.tmO2, p->out2, p->out2_cb_total);
      NEO_CHECK_ARG(r == CUDA_SUCCESS, NEO_ERR_CUDA, "tensor map O2 encode failed (%d)", (int)r);
    }
    if (p->residual) {
      r = encode_fm(&kp.tmR, p->residual, kp.res_cb_total);
      NEO_CHECK_ARG(r == CUDA_SUCCESS, NEO_ERR_CUDA, "tensor map R encode failed (%d)", (int)r);
    }
  } else {
    kp.nslot = 0;
    kp.rowb_out = 0;
    kp.stage_out = 0;
    kp.out_box_bytes = 0;
  }

  const size_t smem = 1024 + (size_t)p->stages * kp.a_stage + kp.b_region +
                     (size_t)kp.ngroups * kp.nslot * kp.stage_out + 512 +
                     (size_t)kp.ngroups * kParamFloats * 4;
  NEO_CHECK_ARG(smem <= (size_t)smem_budget(), NEO_ERR_SCHEDULE_INVALID,
                "conv tile needs %zu bytes of shared memory", smem);
  static const int half_ctas = getenv("NEOB200_HALF_CTAS") ? atoi(getenv("NEOB200_HALF_CTAS")) : 1;
  const int sms = sm_count_of_current_device() * (half_sm_mode() ? half_ctas : 1);
  // weight-stationary: grid % tiles_k == 0 keeps each CTA on one N block
  const int grid = pair  ? (int)std::min<int64_t>(kp.num_groups, sms / 2) * 2
                   : wst ? (int)(std::min<int64_t>(kp.num_units, sms) / kp.tiles_k * kp.tiles_k)
                         : (int)std::min<int64_t>(kp.num_units, sms);
  // opt in to the large dynamic shared memory once per (device, kernel); the
  // attribute call is kept out of later launches so they can be graph-captured
  static bool attr_set[64][8] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  using KFn = void (*)(ConvTCParams);
  static const KFn kfn[4][2] = {
      {conv_tc_kernel<kKindBF16, false>, conv_tc_kernel<kKindBF16, true>},
      {conv_tc_kernel<kKindTF32, false>, conv_tc_kernel<kKindTF32, true>},
      {conv_tc_kernel<kKindFP8, false>, conv_tc_kernel<kKindFP8, true>},
      {conv_tc_kernel<kKindBF16Q, false>, conv_tc_kernel<kKindBF16Q, true>}};
  const KFn fn = kfn[kind][pair ? 1 : 0];
  bool& done = attr_set[dev & 63][kind * 2 + (pair ? 1 : 0)];
  if (!done) {
    NEO_CUDA_TRY(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kSmemBudget));
    if (half_sm_mode())
      NEO_CUDA_TRY(cudaFuncSetAttribute((const void*)fn,
                                        cudaFuncAttributePreferredSharedMemoryCarveout,
                                        cudaSharedmemCarveoutMaxShared));
    done = true;
  }
  if (pair) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = neo_pdl_enabled() ? 2 : 1;
    NEO_CUDA_TRY(cudaLaunchKernelEx(&cfg, fn, kp));
  } else {
    neo_launch(fn, grid, threads, smem, stream, kp);
  }
  NEO_LAUNCH_CHECK();
  return NEO_OK;
}

#ifdef NEO_TRACE
// records of the last traced launch (CTA 0), all warps concatenated
extern "C" int neo_trace_dump(unsigned long long* host, int max_n) {
  unsigned int cnt[kTraceWarps];
  cudaMemcpyFromSymbol(cnt, g_trace_cnt, sizeof(cnt));
  int n = 0;
  for (int w = 0; w < kTraceWarps; ++w) {
    const int take = std::min<int>((int)cnt[w], max_n - n);
    if (take <= 0) continue;
    cudaMemcpyFromSymbol(host + n, g_trace, take * sizeof(unsigned long long),
                         (size_t)w * kTracePerWarp * sizeof(unsigned long long));
    n += take;
  }
  unsigned int zero[kTraceWarps] = {};
  cudaMemcpyToSymbol(g_trace_cnt, zero, sizeof(zero));
  return n;
}
#endif

// debug: NEOB200_DBG&256 timelines, [slot][cta][event] globaltimer ns
extern "C" __attribute__((visibility("default"))) int neo_dbg_timeline(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_tl, n * sizeof(unsigned long long));
}

// debug: per-CTA (MMA-loop cycles, ns) of the last NEOB200_DBG&8 launch
extern "C" __attribute__((visibility("default"))) int neo_dbg_clk(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_dbg_clk, n * sizeof(unsigned long long));
}
