// Probe: tcgen05.mma kind::f16 with the A operand in tensor memory ("TS"),
// written row-per-lane by tcgen05.st (two bf16 per 32-bit column), B in
// shared memory (K-major SWIZZLE_64B, 64-byte rows = 32 bf16).  Checks
// D = A * B^T against the host for M=128, N=64, K=32.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../paper_1809_02697_b200/csrc -I../include mma_ts_test.cu -o mma_ts_test
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "neo_common.cuh"

constexpr int M = 128, N = 64, K = 32;

__global__ void __launch_bounds__(128, 1) probe(const __nv_bfloat16* A, const __nv_bfloat16* B,
                                                float* D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  uint8_t* gbase = smem + (base - smem_u32(smem));
  const uint32_t sB = base, bar = base + 8192;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // B: N rows x 64 bytes, SW64 swizzle
  for (int i = threadIdx.x; i < N * 4; i += 128) {
    const int n = i >> 2, c = i & 3;
    const uint4 v = reinterpret_cast<const uint4*>(B + n * K)[c];
    *reinterpret_cast<uint4*>(gbase + swz_offset(n, c, 64)) = v;
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(smem_u32(&tslot), 128);
    tmem_relinquish();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  // A: row m = lane of warp m/32; 32 bf16 = 16 columns at column 64
  {
    const int m = warp * 32 + lane;
    uint32_t r[16];
    const uint32_t* src = reinterpret_cast<const uint32_t*>(A + m * K);
#pragma unroll
    for (int j = 0; j < 16; ++j) r[j] = src[j];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + 64u;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
        "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc(1u, M, N);
    const uint64_t bd = umma_smem_desc(sB, 16, 512, 4);
    for (int kk = 0; kk < K / 16; ++kk) {
      const uint32_t a = tmem + 64u + 8u * kk;
      const uint64_t b = bd + (uint64_t)(2 * kk);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                   ::"r"(tmem), "r"(a), "l"(b), "r"(idesc), "r"(kk) : "memory");
    }
    umma_commit(bar);
  }
  mbar_wait(bar, 0);
  tc_fence_after();
  {
    uint32_t v[16];
    const int m = warp * 32 + lane;
    for (int c = 0; c < N; c += 16) {
      tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
      tmem_ld_wait();
      for (int j = 0; j < 16; ++j) D[m * N + c + j] = __uint_as_float(v[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}

int main() {
  std::vector<__nv_bfloat16> a(M * K), b(N * K);
  std::vector<float> af(M * K), bf(N * K);
  srand(1);
  for (int i = 0; i < M * K; ++i) { float v = (rand() % 17 - 8) / 8.f; a[i] = __float2bfloat16(v); af[i] = __bfloat162float(a[i]); }
  for (int i = 0; i < N * K; ++i) { float v = (rand() % 13 - 6) / 4.f; b[i] = __float2bfloat16(v); bf[i] = __bfloat162float(b[i]); }
  __nv_bfloat16 *dA, *dB; float* dD;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, N * K * 2); cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, a.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, b.data(), N * K * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<<<1, 128, 32 * 1024>>>(dA, dB, dD);
  std::vector<float> d(M * N);
  cudaError_t e = cudaMemcpy(d.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  int bad = 0; double maxerr = 0;
  for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
    double s = 0; for (int k = 0; k < K; ++k) s += af[m * K + k] * bf[n * K + k];
    double err = fabs(s - d[m * N + n]); maxerr = err > maxerr ? err : maxerr; bad += err > 1e-3;
  }
  printf("%s: %d of %d wrong, max err %g (d[0]=%g)\n", cudaGetErrorString(e), bad, M * N, maxerr, d[0]);
  return 0;
}
