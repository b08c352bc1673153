// tc_selftest.cu -- parity probe of the tcgen05 building blocks (tc.cuh): one
// CTA computes D[128 x N] = A[128 x K] . B[N x K]^T with fp16 operands in the
// canonical K-major packing, bulk-copied to shared memory, fp32 accumulation in
// TMEM, read back with tcgen05.ld.  Used by tests/test_gpu_tc.py.
#include <cuda_fp16.h>

#include "bagel_internal.h"
#include "tc.cuh"

namespace {

__global__ void __launch_bounds__(128) k_tc_selftest(const __half* __restrict__ A, const __half* __restrict__ B,
                                                     int N, int K, float* __restrict__ D, uint32_t ncols) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __half* sA = reinterpret_cast<__half*>(sm);
  __half* sB = sA + 128 * K;
  __shared__ __align__(8) uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  if (tid == 0) {
    tc::mbar_init(&bar_load, 1);
    tc::mbar_init(&bar_mma, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&tmem_base, ncols);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    const uint32_t bytesA = 128u * K * 2u, bytesB = (uint32_t)N * K * 2u;
    tc::mbar_arrive_expect_tx(&bar_load, bytesA + bytesB);
    tc::bulk_g2s(sA, A, bytesA, &bar_load);
    tc::bulk_g2s(sB, B, bytesB, &bar_load);
    tc::mbar_wait(&bar_load, 0);
    tc::tc_fence_after();
    const uint32_t idesc = tc::idesc_f16(128, N);
    const uint32_t sbo = (uint32_t)(K / 8) * 128u;
    for (int s = 0; s < K / 16; ++s) {
      const uint64_t ad = tc::umma_desc(tc::smem_u32(sA) + s * 256u, 128u, sbo);
      const uint64_t bd = tc::umma_desc(tc::smem_u32(sB) + s * 256u, 128u, sbo);
      tc::mma_f16(tbase, ad, bd, idesc, s > 0 ? 1u : 0u);
    }
    tc::umma_commit(&bar_mma);
  }
  tc::mbar_wait(&bar_mma, 0);
  __syncwarp();
  tc::tc_fence_after();
  const int row = 32 * warp + (tid % 32);
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tc::tmem_ld16(tbase + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0, v);
    tc::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 16; ++i) D[(size_t)row * N + c0 + i] = v[i];
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, ncols);
}

}  // namespace

int tc_selftest_launch(const void* A, const void* B, int N, int K, float* D, cudaStream_t st) {
  uint32_t ncols = 32;
  while ((int)ncols < N) ncols <<= 1;
  const size_t smem = (size_t)(128 + N) * K * 2;
  cudaFuncSetAttribute(k_tc_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_tc_selftest<<<1, 128, smem, st>>>((const __half*)A, (const __half*)B, N, K, D, ncols);
  return 1;
}
