// tcgen05.mma issue throughput vs N (M = 128, K = 16 bf16, operands in
// shared memory, SW128 K-major): one thread issues `iters` MMAs back to back
// into one TMEM accumulator, commits, waits; cycles per MMA are reported
// beside the ideal 128*N*16 / 4096 MAC-per-clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../paper_1809_02697_b200/csrc -I../include mma_bench.cu -o mma_bench
#include <cstdio>
#include <cstdlib>

#include "neo_common.cuh"

__global__ void __launch_bounds__(576, 1) mma_kernel(int n, int iters, int kstride, int nacc, unsigned long long* out, int fill) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t sA = base, sB = base + 64 * 1024;
  const uint32_t bar = base + 160 * 1024;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 8, 1);
    mbar_init(bar + 16, 1);
    fence_mbar_init();
  }
  if (fill) {
    // pseudo-random operand bits (bf16 values of moderate magnitude)
    uint32_t* w = reinterpret_cast<uint32_t*>(smem + (base - smem_u32(smem)));
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) {
      uint32_t h = (uint32_t)i * 2654435761u;
      h ^= h >> 13;
      h *= 0x5bd1e995u;
      w[i] = (h & 0x807f807fu) | 0x3c003c00u;
    }
  }
  __syncthreads();
  if (warp == 0) {
    tmem_alloc(smem_u32(&tslot), 128);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc(1u, 128, n);
    const uint64_t ad0 = umma_smem_desc(sA, 16, 1024, 2), bd0 = umma_smem_desc(sB, 16, 1024, 2);
    const long long t0 = clock64();
    if (nacc >= 100) {
      // halo-tap pattern of the weight-stationary 3x3 kernel: tap (r, s) reads
      // A shifted by r*58 + s rows (nacc 100) or unshifted (nacc 101) and
      // weight slice (r, s); 9 taps x 4 K steps per "tile"
      // 102: + A band rotating over 3 stage buffers (31 KB apart) per tile
      // 103: + tcgen05.commit to an mbarrier after every tile
      // 104: + accumulator alternating between two 64-column TMEM stages
      const uint32_t sh = nacc == 101 ? 0u : 1u;
      int tile = 0;
      for (int i = 0; i < iters; i += 36, ++tile) {
        const uint64_t aband = ad0 + (nacc >= 102 ? (uint64_t)((tile % 3) * 31744 / 16) : 0);
        const uint32_t dt = tmem + (nacc >= 104 ? (uint32_t)((tile & 1) * n) : 0u);
        for (int r = 0; r < 3; ++r) {
          const uint64_t ar = aband + sh * (uint64_t)(r * 58 * 8);
          const uint64_t br = bd0 + (uint64_t)(r * 3 * n * 8);
          for (int s2 = 0; s2 < 3; ++s2) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              umma_ss<false>(dt, ar + sh * (uint64_t)(s2 * 8) + 2u * kk,
                             br + (uint64_t)(s2 * n * 8) + 2u * kk, idesc,
                             (nacc >= 105 && (r | s2 | kk) == 0) ? 0u : 1u);
          }
        }
        if (nacc >= 103) umma_commit(bar + 8);
        if (nacc >= 106) umma_commit(bar + 16);
      }
    } else if (nacc <= 0) {
      // unrolled: constant descriptor offsets, no per-MMA register work;
      // nacc < 0: A view shifted by -nacc 128-byte rows (halo taps)
      const uint64_t ash = ad0 + (uint64_t)(-nacc * 8);
      for (int i = 0; i < iters; i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          umma_ss<false>(tmem, ash + (uint64_t)((j & 3) * 2), bd0 + (uint64_t)((j & 3) * 2), idesc,
                         1u);
      }
    } else {
      for (int i = 0; i < iters; ++i) {
        const uint32_t off = (uint32_t)((i % kstride) * 32) >> 4;   // walk the K chunks
        const int a = i % nacc;
        umma_ss<false>(tmem + a * n, ad0 + off, bd0 + off, idesc, i >= nacc);
      }
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}

int main(int argc, char** argv) {
  const int grid_arg = argc > 1 ? atoi(argv[1]) : 1;
  const int fill = argc > 2 ? atoi(argv[2]) : 0;
  const int nthreads = argc > 3 ? atoi(argv[3]) : 128;
  const int smem_kb = argc > 4 ? atoi(argv[4]) : 170;
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024);
  for (int nacc : {106}) {
    for (int n : {32, 64, 128, 256}) {
      if (n > 256 || (nacc >= 100 && n > 64)) continue;
      const int iters = nacc >= 100 ? 36 * 128 : 4096, grid = grid_arg;
      mma_kernel<<<grid, nthreads, smem_kb * 1024>>>(n, iters, 4, nacc, d, fill);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      mma_kernel<<<grid, nthreads, smem_kb * 1024>>>(n, iters, 4, nacc, d, fill);
      cudaEventRecord(e1);
      cudaDeviceSynchronize();
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("  kernel %.1f us, %.1f ns/MMA -> ", ms * 1e3, ms * 1e6 / iters);
      unsigned long long h[1];
      cudaMemcpy(h, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      printf("A row shift %d N=%3d: %7.1f cycles/MMA (ideal %5.1f at 4096 MAC/clk)  %s\n", -nacc,
             n, (double)h[0] / iters, 128.0 * n * 16 / 4096, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
