// Full-chip tcgen05.mma rate: every SM (grid = 148 CTAs) runs one thread
// issuing groups of MMAs (M=128, N given, one 64-channel bf16 slice = 4 K16
// steps, or one 128-channel e4m3 slice = 4 K32 steps) back to back with a
// commit per group, as the conv kernel's issuing loop does; reports cycles
// per MMA (max over CTAs) and the clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../paper_1809_02697_b200/csrc -I../include mma_fullchip.cu -o mma_fullchip
#include <cstdio>
#include <cstdlib>

#include "neo_common.cuh"

template <bool FP8>
__global__ void __launch_bounds__(128, 1) grouped(int n, int groups, int shift, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t sA = base, sB = base + 64 * 1024;
  const uint32_t bar = base + 160 * 1024, cbar = bar + 16;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
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
    const uint32_t idesc = umma_idesc(FP8 ? 0u : 1u, 128, n);
    // shift: A view starts `shift` 128-byte rows into the atom (halo views)
    const uint64_t ad0 = umma_smem_desc(sA + 128u * shift, 16, 1024, 2),
                   bd0 = umma_smem_desc(sB, 16, 1024, 2);
    const long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t alo = (uint32_t)ad0 + 2u * kk, blo = (uint32_t)bd0 + 2u * kk;
        if (FP8)
          asm volatile("{\n\t.reg .pred p;\n\t.reg .b64 ad, bd;\n\tsetp.ne.b32 p, %6, 0;\n\t"
                       "mov.b64 ad, {%1, %2};\n\tmov.b64 bd, {%3, %4};\n\t"
                       "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], ad, bd, %5, p;\n\t}"
                       ::"r"(tmem), "r"(alo), "r"((uint32_t)(ad0 >> 32)), "r"(blo),
                       "r"((uint32_t)(bd0 >> 32)), "r"(idesc), "r"(1u) : "memory");
        else
          asm volatile("{\n\t.reg .pred p;\n\t.reg .b64 ad, bd;\n\tsetp.ne.b32 p, %6, 0;\n\t"
                       "mov.b64 ad, {%1, %2};\n\tmov.b64 bd, {%3, %4};\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], ad, bd, %5, p;\n\t}"
                       ::"r"(tmem), "r"(alo), "r"((uint32_t)(ad0 >> 32)), "r"(blo),
                       "r"((uint32_t)(bd0 >> 32)), "r"(idesc), "r"(1u) : "memory");
      }
      umma_commit(cbar);
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    out[blockIdx.x] = clock64() - t0;
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
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(grouped<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(grouped<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int fp8 = 0; fp8 < 2; ++fp8)
    for (int grid : {1, 148})
      for (int n : {64, 128, 256})
        for (int shift : {0, 3}) {
          const int groups = 2048;
          cudaEvent_t a, b;
          cudaEventCreate(&a);
          cudaEventCreate(&b);
          for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (fp8) grouped<true><<<grid, 128, 170 * 1024>>>(n, groups, shift, d);
            else grouped<false><<<grid, 128, 170 * 1024>>>(n, groups, shift, d);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
          }
          float ms = 0;
          cudaEventElapsedTime(&ms, a, b);
          long long h[148];
          cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
          long long mx = 0;
          for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
          const double mmas = 4.0 * groups;
          const double flop = 2.0 * 128 * n * (fp8 ? 32 : 16) * mmas * grid;
          printf("%s grid=%3d N=%3d shift=%d: %.1f cycles/MMA, %.2f GHz, %.0f TFLOP/s  %s\n",
                 fp8 ? "fp8 " : "bf16", grid, n, shift, mx / mmas, mx / (ms * 1e6), flop / (ms * 1e9),
                 cudaGetErrorString(cudaGetLastError()));
        }
  return 0;
}
