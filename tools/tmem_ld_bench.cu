// TMEM load latency with and without concurrent tcgen05.mma traffic: warp 0
// lane 0 issues back-to-back M=128 MMAs into TMEM columns [256, 256+N); warps
// 4-7 (one per lane quarter) time tcgen05.ld.32x32b.x16 + wait::ld on
// columns [0, 128).  mma=0 runs the loads alone.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../paper_1809_02697_b200/csrc -I../include tmem_ld_bench.cu -o tmem_ld_bench
#include <cstdio>

#include "neo_common.cuh"

__global__ void __launch_bounds__(256, 1) tl(int n, int mma, int loads, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t sA = base, sB = base + 64 * 1024, bar = base + 160 * 1024;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    stop = 0;
  }
  if (warp == 0) {
    tmem_alloc(smem_u32(&tslot), 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0 && lane == 0 && mma) {
    const uint32_t idesc = umma_idesc(1u, 128, n);
    const uint64_t ad0 = umma_smem_desc(sA, 16, 1024, 2), bd0 = umma_smem_desc(sB, 16, 1024, 2);
    for (int i = 0; i < 20000 && !stop; ++i)
      umma_ss<false>(tmem + 256, ad0 + (uint64_t)((i & 3) * 2), bd0 + (uint64_t)((i & 3) * 2),
                     idesc, 1u);
    umma_commit(bar);
    mbar_wait(bar, 0);
  }
  if (warp >= 4) {
    const uint32_t q = (uint32_t)(warp & 3);
    long long tot = 0;
    uint32_t acc = 0;
    for (int i = 0; i < loads; ++i) {
      uint32_t v[16];
      const long long t0 = clock64();
      tmem_ld16(tmem + (q * 32 << 16) + (uint32_t)((i & 7) * 16), v);
      tmem_ld_wait_regs(v);
      tot += clock64() - t0;
#pragma unroll
      for (int j = 0; j < 16; ++j) acc += v[j];
    }
    if (lane == 0) out[warp - 4] = tot / loads;
    if (acc == 0x12345678u) out[8] = acc;
    if (warp == 4 && lane == 0) stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16 * sizeof(long long));
  cudaFuncSetAttribute(tl, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int n : {64, 128, 256})
    for (int mma : {0, 1}) {
      tl<<<1, 256, 170 * 1024>>>(n, mma, 2000, d);
      long long h[4];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("N=%3d mma=%d: tmem ld16+wait %lld %lld %lld %lld cycles  %s\n", n, mma, h[0], h[1],
             h[2], h[3], cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
