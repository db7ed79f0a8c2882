// tcgen05.mma issue throughput vs N (M = 128, K = 16 bf16, operands in
// shared memory, SW128 K-major): one thread issues `iters` MMAs back to back
// into one TMEM accumulator, commits, waits; cycles per MMA are reported
// beside the ideal 128*N*16 / 4096 MAC-per-clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../paper_1809_02697_b200/csrc -I../include mma_bench.cu -o mma_bench
#include <cstdio>

#include "neo_common.cuh"

__global__ void __launch_bounds__(128, 1) mma_kernel(int n, int iters, int kstride, int nacc, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t sA = base, sB = base + 64 * 1024;
  const uint32_t bar = base + 160 * 1024;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(smem_u32(&tslot), 512);
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
    if (nacc <= 0) {
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
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int nacc : {0, -1, -2, -4, -8}) {
    for (int n : {32, 64, 128, 256}) {
      if (n > 256) continue;
      const int iters = 4096, grid = 1;
      mma_kernel<<<grid, 128, 170 * 1024>>>(n, iters, 4, nacc, d);
      mma_kernel<<<grid, 128, 170 * 1024>>>(n, iters, 4, nacc, d);
      cudaDeviceSynchronize();
      unsigned long long h[1];
      cudaMemcpy(h, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      printf("A row shift %d N=%3d: %7.1f cycles/MMA (ideal %5.1f at 4096 MAC/clk)  %s\n", -nacc,
             n, (double)h[0] / iters, 128.0 * n * 16 / 4096, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
