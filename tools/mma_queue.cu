// tcgen05.mma issue-queue probe: one thread issues K MMAs (M=128, N given,
// K=16 bf16, SW128 operands) back to back after an idle tensor pipe and
// records the cycles spent issuing (the issue blocks once the queue is full)
// and until their completion (commit + mbarrier wait).  Issue cycles flat in
// K = queue depth; completion(1) = pipeline latency; slope = per-MMA time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../paper_1809_02697_b200/csrc -I../include mma_queue.cu -o mma_queue
#include <cstdio>
#include <cstdlib>

#include "neo_common.cuh"

__global__ void __launch_bounds__(128, 1) probe(int n, int k, long long* out) {
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
    tmem_alloc(smem_u32(&tslot), 256);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc(1u, 128, n);
    const uint64_t ad0 = umma_smem_desc(sA, 16, 1024, 2), bd0 = umma_smem_desc(sB, 16, 1024, 2);
    uint32_t phase = 0;
    for (int rep = 0; rep < 3; ++rep) {   // rep 0 warms up
      const long long t0 = clock64();
      for (int i = 0; i < k; ++i)
        umma_ss<false>(tmem, ad0 + (uint64_t)((i & 3) * 2), bd0 + (uint64_t)((i & 3) * 2), idesc, 1u);
      const long long t1 = clock64();
      umma_commit(bar);
      mbar_wait(bar, phase);
      phase ^= 1u;
      const long long t2 = clock64();
      out[0] = t1 - t0;
      out[1] = t2 - t0;
      // idle gap so the next rep starts from an empty pipe
      const long long g = clock64();
      while (clock64() - g < 20000) {
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}


// grouped issue: groups of 4 MMAs (one 64-channel slice), per group:
// mode 0 nothing, 1 commit to an mbarrier, 2 + try_wait on a completed
// barrier, 3 + tcgen05 fence::after_thread_sync, 4 + integer division
__global__ void __launch_bounds__(128, 1) grouped(int n, int groups, int mode, int divisor, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t sA = base, sB = base + 64 * 1024;
  const uint32_t bar = base + 160 * 1024, done = bar + 8, cbar = bar + 16;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(done, 1);
    mbar_init(cbar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(smem_u32(&tslot), 256);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    mbar_arrive(done);   // phase 0 completes: try_wait(done, 0) succeeds at once
    const uint32_t idesc = umma_idesc(1u, 128, n);
    const uint64_t ad0 = umma_smem_desc(sA, 16, 1024, 2), bd0 = umma_smem_desc(sB, 16, 1024, 2);
    int acc = 0;
    const long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      if (mode >= 2) mbar_wait(done, 0);
      if (mode >= 3) tc_fence_after();
      if (mode >= 4) acc += g / divisor;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        // 32-bit low-word descriptor arithmetic (as in conv_tc.cu mma_issue)
        const uint32_t alo = (uint32_t)ad0 + 2u * kk, blo = (uint32_t)bd0 + 2u * kk;
        asm volatile("{\n\t.reg .pred p;\n\t.reg .b64 ad, bd;\n\tsetp.ne.b32 p, %6, 0;\n\t"
                     "mov.b64 ad, {%1, %2};\n\tmov.b64 bd, {%3, %4};\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], ad, bd, %5, p;\n\t}"
                     ::"r"(tmem), "r"(alo), "r"((uint32_t)(ad0 >> 32)), "r"(blo),
                     "r"((uint32_t)(bd0 >> 32)), "r"(idesc), "r"(1u) : "memory");
      }
      if (mode >= 1) umma_commit(cbar);
      if (mode >= 5) umma_commit(cbar);
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    out[0] = clock64() - t0;
    out[1] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 2 * sizeof(long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int n : {64, 128, 256}) {
    for (int k : {1, 2, 4, 6, 8, 12, 16, 24, 32, 48, 64, 128}) {
      probe<<<1, 128, 170 * 1024>>>(n, k, d);
      long long h[2];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("N=%3d K=%4d: issue %6lld cycles, complete %6lld cycles (%.1f/MMA)  %s\n", n, k, h[0],
             h[1], (double)h[1] / k, cudaGetErrorString(cudaGetLastError()));
    }
  }
  cudaFuncSetAttribute(grouped, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int n : {64, 128, 256})
    for (int mode = 0; mode <= 5; ++mode) {
      grouped<<<1, 128, 170 * 1024>>>(n, 256, mode, 7, d);
      grouped<<<1, 128, 170 * 1024>>>(n, 256, mode, 7, d);
      long long h[2];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("grouped N=%3d mode %d: %.1f cycles/MMA  %s\n", n, mode, (double)h[0] / 1024,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
