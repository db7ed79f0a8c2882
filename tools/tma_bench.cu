// TMA streaming microbenchmark: per-SM throughput of cp.async.bulk.tensor
// loads for the box shapes the conv kernel issues (rows of `rowb` bytes,
// `rows` rows per box, `boxes` boxes per stage, `stages` stages in flight).
// One producer lane issues, one consumer lane waits on the full barrier and
// frees the stage at once (no compute), so the result is the load path alone.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../paper_1809_02697_b200/csrc -I../include tma_bench.cu -lcuda -o tma_bench
//   ./tma_bench
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>

#include "neo_common.cuh"

struct Args {
  CUtensorMap map;  // 2-D: (row elems, total rows)
  const CUtensorMap* gmap;  // same descriptor in global memory (mode 2)
  int mode;                 // 0 param, 1 param + prefetch, 2 global + prefetch
  int rows, boxes, stages, iters, rowb;
  long long total_rows;
};

__global__ void __launch_bounds__(96, 1) tma_stream(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t stage_bytes = (uint32_t)(a.rows * a.rowb * a.boxes);
  const uint32_t bars = base + a.stages * stage_bytes;
  auto full = [&](int s) { return bars + 8u * s; };
  auto empty = [&](int s) { return bars + 64u + 8u * s; };
  const CUtensorMap* mp = a.mode == 2 ? a.gmap : &a.map;
  if (threadIdx.x == 0 && a.mode >= 1)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(mp)) : "memory");
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const long long nboxrows = a.total_rows / a.rows;
  if (a.mode == 4 && (threadIdx.x == 0 || threadIdx.x == 32 * 2)) {
    // two producer warps (warp 0 and warp 2), each issuing half of each stage
    int stage = 0;
    uint32_t phase = 0;
    const int half = threadIdx.x == 0 ? 0 : 1;
    for (int it = 0; it < a.iters; ++it) {
      mbar_wait(empty(stage), phase ^ 1u);
      if (half == 0) mbar_arrive_expect_tx(full(stage), stage_bytes);
      for (int b = half; b < a.boxes; b += 2) {
        const long long box = (long long)blockIdx.x * 977 + (long long)it * a.boxes + b;
        const int row = (int)((box & (nboxrows - 1)) * a.rows);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3}], [%4];" ::"r"(base + stage * stage_bytes + b * a.rows * a.rowb),
            "l"(reinterpret_cast<uint64_t>(mp)), "r"(0), "r"(row), "r"(full(stage))
            : "memory");
      }
      if (++stage == a.stages) {
        stage = 0;
        phase ^= 1u;
      }
    }
  } else if (a.mode == 3 && threadIdx.x < 32) {
    // boxes of a stage issued by different lanes of the producer warp
    int stage = 0;
    uint32_t phase = 0;
    const int lane = threadIdx.x;
    for (int it = 0; it < a.iters; ++it) {
      if (lane == 0) {
        mbar_wait(empty(stage), phase ^ 1u);
        mbar_arrive_expect_tx(full(stage), stage_bytes);
      }
      __syncwarp();
      if (lane < a.boxes) {
        const long long box = (long long)blockIdx.x * 977 + (long long)it * a.boxes + lane;
        const int row = (int)((box & (nboxrows - 1)) * a.rows);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3}], [%4];" ::"r"(base + stage * stage_bytes + lane * a.rows * a.rowb),
            "l"(reinterpret_cast<uint64_t>(mp)), "r"(0), "r"(row), "r"(full(stage))
            : "memory");
      }
      if (++stage == a.stages) {
        stage = 0;
        phase ^= 1u;
      }
    }
  } else if (threadIdx.x == 0) {
    int stage = 0;
    uint32_t phase = 0;
    long long box = (long long)blockIdx.x * 977;
    for (int it = 0; it < a.iters; ++it) {
      mbar_wait(empty(stage), phase ^ 1u);
      mbar_arrive_expect_tx(full(stage), stage_bytes);
      for (int b = 0; b < a.boxes; ++b) {
        const int row = (int)((box++ & (nboxrows - 1)) * a.rows);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3}], [%4];" ::"r"(base + stage * stage_bytes + b * a.rows * a.rowb),
            "l"(reinterpret_cast<uint64_t>(mp)), "r"(0), "r"(row), "r"(full(stage))
            : "memory");
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

int main(int argc, char** argv) {
  const long long src_mb = argc > 1 ? atoll(argv[1]) : 512;
  const int grid = argc > 2 ? atoi(argv[2]) : 1;   // CTAs (one per SM), e.g. 148
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q);
  const long long bytes = src_mb << 20;   // default 512 MB source (beyond L2)
  void* src = nullptr;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  printf("mode rowb rows boxes stages grid | stageKB | GB/s/SM  total TB/s\n");
  struct Cfg { int rowb, rows, boxes, stages, grid, mode; };
  std::vector<Cfg> cfgs;
  CUtensorMap* gmap = nullptr;
  cudaMalloc(&gmap, sizeof(CUtensorMap));
  for (int mode : {1, 3, 4})
    for (int boxes : {2, 4, 8})
      cfgs.push_back({128, 32, boxes, 4, grid, mode});
  for (int mode : {1, 3, 4})
    for (int rows : {64, 128, 256})
      for (int stages : {3, 6})
        cfgs.push_back({128, rows, 2, stages, grid, mode});
  for (auto c : cfgs) {
    Args a{};
    a.mode = c.mode;
    a.gmap = gmap;
    a.rows = c.rows;
    a.boxes = c.boxes;
    a.stages = c.stages;
    a.rowb = c.rowb;
    a.total_rows = bytes / c.rowb;
    const long long stage_bytes = (long long)c.rows * c.rowb * c.boxes;
    if (c.stages * stage_bytes + 2048 > 227 * 1024) continue;
    a.iters = (int)std::max<long long>(64, (64ll << 20) / stage_bytes / std::min(c.grid, 8));
    cuuint64_t dims[2] = {(cuuint64_t)(c.rowb / 2), (cuuint64_t)a.total_rows};
    cuuint64_t strides[1] = {(cuuint64_t)c.rowb};
    cuuint32_t box[2] = {(cuuint32_t)(c.rowb / 2), (cuuint32_t)c.rows};
    cuuint32_t estr[2] = {1, 1};
    CUtensorMapSwizzle swz = c.rowb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    encode(&a.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemcpy(gmap, &a.map, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    const size_t smem = c.stages * stage_bytes + 2048;
    tma_stream<<<c.grid, 96, smem>>>(a);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    tma_stream<<<c.grid, 96, smem>>>(a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double moved = (double)stage_bytes * a.iters * c.grid;
    printf("%4d %4d %4d %5d %6d %4d | %7.1f | %7.1f  %7.2f   %s\n", c.mode, c.rowb, c.rows, c.boxes,
           c.stages, c.grid, stage_bytes / 1024.0, moved / (ms * 1e-3) / 1e9 / c.grid,
           moved / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
