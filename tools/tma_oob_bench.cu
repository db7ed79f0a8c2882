// Does TMA slow down on boxes that are partly out of bounds (the conv's
// implicit zero padding)?  One producer lane issues 5-D boxes shaped like
// the conv's A tiles into a ring of stages; one consumer lane frees them.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../paper_1809_02697_b200/csrc -I../include tma_oob_bench.cu -lcuda -o tma_oob_bench
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>

#include "neo_common.cuh"

struct Args {
  CUtensorMap map;
  CUtensorMap mapB;     // conv-like weight box (x, K, Cb, taps)
  int withB, b_bytes;
  int iters, stages, box_bytes, off, N, Cb;
  int rank, rows_per_box, total_rows;   // rank 2/3: flat views
};

__global__ void __launch_bounds__(64, 1) k5(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t stage_bytes = ((a.box_bytes + 1023) & ~1023) + (a.withB ? ((a.b_bytes + 1023) & ~1023) : 0);
  const uint32_t bars = base + a.stages * stage_bytes;
  auto full = [&](int s) { return bars + 8u * s; };
  auto empty = [&](int s) { return bars + 128u + 8u * s; };
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int stage = 0;
    uint32_t phase = 0;
    int cb = 0, n = blockIdx.x % a.N;
    for (int it = 0; it < a.iters; ++it) {
      mbar_wait(empty(stage), phase ^ 1u);
      mbar_arrive_expect_tx(full(stage), a.box_bytes + (a.withB ? a.b_bytes : 0));
      if (a.withB)
        tma_load_4d(base + stage * stage_bytes + ((a.box_bytes + 1023) & ~1023), &a.mapB,
                    full(stage), 0, 0, cb, 0);
      if (a.rank == 5) {
        tma_load_5d(base + stage * stage_bytes, &a.map, full(stage), 0, a.off, a.off, cb, n);
      } else if (a.rank == 3) {
        tma_load_3d(base + stage * stage_bytes, &a.map, full(stage), 0, 0, cb + n * a.Cb);
      } else {
        const int row = ((it * 977) % (a.total_rows / a.rows_per_box)) * a.rows_per_box;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3}], [%4];" ::"r"(base + stage * stage_bytes),
            "l"(reinterpret_cast<uint64_t>(&a.map)), "r"(0), "r"(row), "r"(full(stage))
            : "memory");
      }
      if (++cb == a.Cb) {
        cb = 0;
        if (++n == a.N) n = 0;
      }
      if (++stage == a.stages) {
        stage = 0;
        phase ^= 1u;
      }
    }
  } else if (threadIdx.x == 32) {
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0; it < a.iters; ++it) {
      mbar_wait(full(stage), phase);
      mbar_arrive(empty(stage));
      if (++stage == a.stages) {
        stage = 0;
        phase ^= 1u;
      }
    }
  }
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q);
  const int N = 32, Cb = 4, x = 64;
  struct Cfg { int H, W, bh, bw, off, grid; const char* name; };
  Cfg cfgs[] = {
    {7, 7, 7, 7, 0, 1, "7x7 box in bounds"},
    {7, 7, 7, 9, 0, 1, "7x9 box, 2 cols OOB right"},
    {7, 7, 9, 9, -1, 1, "9x9 box, 1-px halo all sides"},
    {14, 14, 8, 16, 0, 1, "8x16 box, 2 cols OOB"},
    {14, 14, 8, 14, 0, 1, "8x14 box in bounds"},
    {14, 14, 8, 16, -1, 1, "8x16 box at (-1,-1)"},
    {56, 56, 2, 58, -1, 1, "2x58 box at (-1,-1)"},
    {56, 56, 2, 56, 0, 1, "2x56 box in bounds"},
    {7, 7, 7, 7, 0, 148, "7x7 in bounds, 148 CTAs"},
    {7, 7, 9, 9, -1, 148, "9x9 halo, 148 CTAs"},
  };
  void* src = nullptr;
  cudaMalloc(&src, (size_t)N * Cb * 56 * 56 * x * 2);
  cudaMemset(src, 0, (size_t)N * Cb * 56 * 56 * x * 2);
  cudaFuncSetAttribute(k5, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  // flat views: rank 3 (x, H*W, Cb*N) box {x, 128, 1}; rank 2 (x, rows) box {x, 128}
  for (int rank : {3, 2}) {
    for (int grid : {1, 148}) {
      Args a{};
      a.iters = 2048;
      a.stages = 6;
      a.N = N;
      a.Cb = Cb;
      a.rank = rank;
      a.rows_per_box = 128;
      const int H = 56, W = 56;
      a.total_rows = N * Cb * H * W;
      a.box_bytes = 128 * x * 2;
      if (rank == 3) {
        cuuint64_t dims[3] = {(cuuint64_t)x, (cuuint64_t)(H * W), (cuuint64_t)(Cb * N)};
        cuuint64_t strides[2] = {(cuuint64_t)x * 2, (cuuint64_t)H * W * x * 2};
        cuuint32_t box[3] = {(cuuint32_t)x, 128, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        encode(&a.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, src, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      } else {
        cuuint64_t dims[2] = {(cuuint64_t)x, (cuuint64_t)a.total_rows};
        cuuint64_t strides[1] = {(cuuint64_t)x * 2};
        cuuint32_t box[2] = {(cuuint32_t)x, 128};
        cuuint32_t estr[2] = {1, 1};
        encode(&a.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      }
      const size_t smem = a.stages * ((a.box_bytes + 1023) & ~1023) + 2048;
      k5<<<grid, 64, smem>>>(a);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k5<<<grid, 64, smem>>>(a);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("rank-%d box {64,128} (16 KB)       grid %3d: %7.1f ns per box, %6.1f GB/s per CTA  %s\n",
             rank, grid, ms * 1e6 / a.iters, (double)a.box_bytes * a.iters / (ms * 1e-3) / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  for (auto c : cfgs) {
    Args a{};
    a.rank = 5;
    a.iters = 2048;
    a.stages = 6;
    a.N = N;
    a.Cb = Cb;
    a.off = c.off;
    a.box_bytes = c.bh * c.bw * x * 2;
    cuuint64_t dims[5] = {(cuuint64_t)x, (cuuint64_t)c.W, (cuuint64_t)c.H, (cuuint64_t)Cb,
                          (cuuint64_t)N};
    cuuint64_t strides[4] = {(cuuint64_t)x * 2, (cuuint64_t)c.W * x * 2,
                             (cuuint64_t)c.H * c.W * x * 2, (cuuint64_t)Cb * c.H * c.W * x * 2};
    cuuint32_t box[5] = {(cuuint32_t)x, (cuuint32_t)c.bw, (cuuint32_t)c.bh, 1, 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    encode(&a.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, src, dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const size_t smem = a.stages * ((a.box_bytes + 1023) & ~1023) + 2048;
    k5<<<c.grid, 64, smem>>>(a);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k5<<<c.grid, 64, smem>>>(a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-32s grid %3d: %7.1f ns per box, %6.1f GB/s per CTA  %s\n", c.name, c.grid,
           ms * 1e6 / a.iters, (double)a.box_bytes * a.iters / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  // the conv's halo stage: one 5-D band box + one 4-D weight box (3 taps x
  // 128 rows) per stage, issued by one thread, 2 or 4 stages in flight
  void* wsrc = nullptr;
  cudaMalloc(&wsrc, 9ull * 4 * 256 * 128);
  for (int stages : {2, 4}) {
    for (int grid : {1, 148}) {
      Args a{};
      a.iters = 2048;
      a.stages = stages;
      a.N = N;
      a.Cb = Cb;
      a.rank = 5;
      a.off = -1;
      a.withB = 1;
      const int H = 14, W = 14, bh = 8, bw = 16;
      a.box_bytes = bh * bw * x * 2;
      a.b_bytes = 3 * 128 * 128;
      cuuint64_t dims[5] = {(cuuint64_t)x, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)Cb,
                            (cuuint64_t)N};
      cuuint64_t strides[4] = {(cuuint64_t)x * 2, (cuuint64_t)W * x * 2,
                               (cuuint64_t)H * W * x * 2, (cuuint64_t)Cb * H * W * x * 2};
      cuuint32_t box[5] = {(cuuint32_t)x, (cuuint32_t)bw, (cuuint32_t)bh, 1, 1};
      cuuint32_t estr[5] = {1, 1, 1, 1, 1};
      encode(&a.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, src, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      cuuint64_t bd[4] = {(cuuint64_t)x, 256, (cuuint64_t)Cb, 9};
      cuuint64_t bs[3] = {(cuuint64_t)x * 2, 256ull * x * 2, 256ull * Cb * x * 2};
      cuuint32_t bb[4] = {(cuuint32_t)x, 128, 1, 3};
      cuuint32_t be[4] = {1, 1, 1, 1};
      encode(&a.mapB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, wsrc, bd, bs, bb, be,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const size_t smem = a.stages * (((a.box_bytes + 1023) & ~1023) + ((a.b_bytes + 1023) & ~1023)) + 2048;
      k5<<<grid, 64, smem>>>(a);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k5<<<grid, 64, smem>>>(a);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("conv halo stage (A 16KB + B 48KB), %d stages, grid %3d: %7.1f ns per stage  %s\n",
             stages, grid, ms * 1e6 / a.iters, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
