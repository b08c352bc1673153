// tc_selftest.cu -- parity probe of the tcgen05 building blocks (tc.cuh): one
// CTA computes D[128 x N] = A[128 x K] . B[N x K]^T with fp16 operands in the
// canonical K-major packing, bulk-copied to shared memory, fp32 accumulation in
// TMEM, read back with tcgen05.ld.  Used by tests/test_gpu_tc.py.
#include <cuda_fp16.h>

#include "bagel_internal.h"
#include "tc.cuh"

namespace {

// mode 0: A and B from shared memory (canonical packing).  mode 1: A from TMEM -- A given
// row-major (128 x K fp16) is written to TMEM columns [ncols_d, ncols_d + K/2) with tcgen05.st
// by the thread owning each row, then the "TS" tcgen05.mma reads it.
__global__ void __launch_bounds__(128) k_tc_selftest(const __half* __restrict__ A, const __half* __restrict__ B,
                                                     int N, int K, float* __restrict__ D, uint32_t ncols,
                                                     int mode, uint32_t acol) {
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
  if (mode == 1) {
    // each thread writes its row of A (row = 32 * warp + lane) into TMEM, 8 columns (16 fp16) at a time
    const int row = 32 * warp + (tid % 32);
    for (int c0 = 0; c0 < K / 2; c0 += 8) {
      uint32_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const __half lo = A[(size_t)row * K + 2 * (c0 + u)], hi = A[(size_t)row * K + 2 * (c0 + u) + 1];
        v[u] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
      }
      tc::tmem_st8(tbase + ((uint32_t)(32 * warp) << 16) + acol + (uint32_t)c0, v);
    }
    tc::tmem_st_wait();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
  }
  if (tid == 0) {
    const uint32_t bytesA = mode == 0 ? 128u * K * 2u : 0u, bytesB = (uint32_t)N * K * 2u;
    tc::mbar_arrive_expect_tx(&bar_load, bytesA + bytesB);
    if (mode == 0) tc::bulk_g2s(sA, A, bytesA, &bar_load);
    tc::bulk_g2s(sB, B, bytesB, &bar_load);
    tc::mbar_wait(&bar_load, 0);
    tc::tc_fence_after();
    const uint32_t idesc = tc::idesc_f16(128, N);
    const uint32_t sbo = (uint32_t)(K / 8) * 128u;
    for (int s = 0; s < K / 16; ++s) {
      const uint64_t ad = tc::umma_desc(tc::smem_u32(sA) + s * 256u, 128u, sbo);
      const uint64_t bd = tc::umma_desc(tc::smem_u32(sB) + s * 256u, 128u, sbo);
      if (mode == 0)
        tc::mma_f16(tbase, ad, bd, idesc, s > 0 ? 1u : 0u);
      else
        tc::mma_f16_ts(tbase, tbase + acol + (uint32_t)(s * 8), bd, idesc, s > 0 ? 1u : 0u);
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

int tc_selftest_launch(const void* A, const void* B, int N, int K, float* D, int mode, cudaStream_t st) {
  uint32_t ncols = 32;
  const uint32_t need = mode == 1 ? (uint32_t)(N + K / 2) : (uint32_t)N;
  while (ncols < need) ncols <<= 1;
  const size_t smem = (size_t)(128 + N) * K * 2;
  bagel_set_smem_attr(k_tc_selftest, smem);
  k_tc_selftest<<<1, 128, smem, st>>>((const __half*)A, (const __half*)B, N, K, D, ncols, mode, (uint32_t)N);
  return 1;
}

// ---------------------------------------------------------------- CTA-pair (cta_group::2) probe
// A 2-CTA cluster computes D[256 x N] = A[256 x K] . B[N x K]^T with one M = 256 MMA chain issued
// by the leader: CTA r holds A rows 128 r .. 128 r + 127 and B rows (N/2) r .. (N/2)(r + 1) - 1 in
// shared memory (canonical packing, same offsets in both CTAs) and reads D rows 128 r .. back
// from its own TMEM.  A is given as [A rows 0-127 packed | A rows 128-255 packed], B likewise.
namespace {
__global__ void __launch_bounds__(128) k_tc_selftest2(const __half* __restrict__ A, const __half* __restrict__ B,
                                                      int N, int K, float* __restrict__ D, uint32_t ncols, int ts) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __half* sA = reinterpret_cast<__half*>(sm);
  __half* sB = sA + 128 * K;
  __shared__ __align__(8) uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  const uint32_t rank = tc::cluster_rank();
  if (tid == 0) {
    tc::mbar_init(&bar_load, 1);
    tc::mbar_init(&bar_mma, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc2(&tmem_base, ncols);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  tc::cluster_sync();
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    const uint32_t bytesA = 128u * K * 2u, bytesB = (uint32_t)(N / 2) * K * 2u;
    tc::mbar_arrive_expect_tx(&bar_load, bytesA + bytesB);
    tc::bulk_g2s(sA, A + (size_t)rank * 128 * K, bytesA, &bar_load);
    tc::bulk_g2s(sB, B + (size_t)rank * (N / 2) * K, bytesB, &bar_load);
    tc::mbar_wait(&bar_load, 0);
  }
  __syncthreads();
  if (ts) {
    // TS form: this CTA's 128 rows of A (given row-major after the two packed halves) -> TMEM
    // columns [N, N + K/2) of the row's lane, two fp16 per column
    const __half* Ar = A + (size_t)256 * K + (size_t)rank * 128 * K;
    const int row = 32 * warp + (tid % 32);
    for (int c0 = 0; c0 < K / 2; c0 += 8) {
      uint32_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const __half lo = Ar[(size_t)row * K + 2 * (c0 + u)], hi = Ar[(size_t)row * K + 2 * (c0 + u) + 1];
        v[u] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
      }
      tc::tmem_st8(tbase + ((uint32_t)(32 * warp) << 16) + (uint32_t)N + (uint32_t)c0, v);
    }
    tc::tmem_st_wait();
    tc::tc_fence_before();
    __syncthreads();
  }
  tc::cluster_sync();  // both CTAs' operands are in shared memory / TMEM
  if (rank == 0 && tid == 0) {
    tc::tc_fence_after();
    const uint32_t idesc = tc::idesc_f16(256, N);
    const uint32_t sbo = (uint32_t)(K / 8) * 128u;
    for (int s = 0; s < K / 16; ++s) {
      const uint64_t ad = tc::umma_desc(tc::smem_u32(sA) + s * 256u, 128u, sbo);
      const uint64_t bd = tc::umma_desc(tc::smem_u32(sB) + s * 256u, 128u, sbo);
      if (ts)
        tc::mma_f16_ts2(tbase, tbase + (uint32_t)N + (uint32_t)(s * 8), bd, idesc, s > 0 ? 1u : 0u);
      else
        tc::mma_f16_2(tbase, ad, bd, idesc, s > 0 ? 1u : 0u);
    }
    tc::umma_commit2_mc(&bar_mma, 3);
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
    for (int i = 0; i < 16; ++i) D[(size_t)(rank * 128 + row) * N + c0 + i] = v[i];
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();
  if (warp == 0) tc::tmem_dealloc2(tbase, ncols);
}
}  // namespace

int tc_selftest2_launch(const void* A, const void* B, int N, int K, float* D, int ts, cudaStream_t st) {
  uint32_t ncols = 32;
  while (ncols < (uint32_t)N + (ts ? (uint32_t)K / 2 : 0u)) ncols <<= 1;
  const size_t smem = (size_t)(128 + N / 2) * K * 2;
  bagel_set_smem_attr(k_tc_selftest2, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2, 1, 1);
  cfg.blockDim = dim3(128, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  (void)cudaLaunchKernelEx(&cfg, k_tc_selftest2, (const __half*)A, (const __half*)B, N, K, D, ncols, ts);
  return 1;
}

// ---------------------------------------------------------------- MMA issue-rate microbenchmark
// Every CTA issues `iters` back-to-back tcgen05.mma (M=128, N, K=16; A from smem (mode 0) or TMEM
// (mode 1)) into one accumulator and records the cycles from first issue to commit completion.
namespace {
__global__ void __launch_bounds__(128) k_tc_bench(int N, int iters, int mode, long long* cycles) {
  const int unroll = mode & 16;  // issue 8 MMAs per loop trip (fixed accumulator pattern)
  const int nacc = (mode >> 1) & 7;  // >0: round-robin over nacc independent accumulators of N columns
  mode &= 1;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  // zero operands: A 128x16, B Nx16 fp16
  for (int i = tid; i < (128 + N) * 16 / 2; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0u;
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&tmem_base, 512);
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t t = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_f16(128, N);
    const uint64_t ad = tc::umma_desc(tc::smem_u32(sm), 128, 256);
    const uint64_t bd = tc::umma_desc(tc::smem_u32(sm) + 128 * 16 * 2, 128, 256);
    const long long c0 = clock64();
    if (unroll) {
      const uint32_t d1 = nacc > 1 ? t + (uint32_t)N : t;
      for (int i = 0; i < iters; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t d = (u & 1) ? d1 : t;
          if (mode == 0)
            tc::mma_f16(d, ad, bd, idesc, (i + u) > 1 ? 1u : 0u);
          else
            tc::mma_f16_ts(d, t + 256u, bd, idesc, (i + u) > 1 ? 1u : 0u);
        }
      }
    } else
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = nacc > 0 ? t + (uint32_t)((i % nacc) * N) : t;
      const uint32_t acc = nacc > 0 ? (i >= nacc ? 1u : 0u) : (i > 0 ? 1u : 0u);
      if (mode == 0)
        tc::mma_f16(d, ad, bd, idesc, acc);
      else
        tc::mma_f16_ts(d, t + 256u, bd, idesc, acc);
    }
    tc::umma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    cycles[blockIdx.x] = clock64() - c0;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(t, 512);
}
}  // namespace

// CTA pairs: every 2-CTA cluster's leader issues `iters` back-to-back tcgen05.mma.cta_group::2
// (M = 256, N, K = 16, A and B from shared memory) into one accumulator.
namespace {
__global__ void __launch_bounds__(128) k_tc_bench2(int N, int iters, int ts, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  const uint32_t rank = tc::cluster_rank();
  for (int i = tid; i < (128 + N / 2) * 16 / 2; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0u;
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc2(&tmem_base, 512);
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  tc::cluster_sync();
  const uint32_t t = tmem_base;
  if (rank == 0 && tid == 0) {
    const uint32_t idesc = tc::idesc_f16(256, N);
    const uint64_t ad = tc::umma_desc(tc::smem_u32(sm), 128, 256);
    const uint64_t bd = tc::umma_desc(tc::smem_u32(sm) + 128 * 16 * 2, 128, 256);
    const long long c0 = clock64();
    if (ts)
      for (int i = 0; i < iters; ++i) tc::mma_f16_ts2(t, t + 256u, bd, idesc, i > 0 ? 1u : 0u);
    else
      for (int i = 0; i < iters; ++i) tc::mma_f16_2(t, ad, bd, idesc, i > 0 ? 1u : 0u);
    tc::umma_commit2_mc(&bar, 3);
    tc::mbar_wait(&bar, 0);
    cycles[blockIdx.x / 2] = clock64() - c0;
  } else if (tid == 0) {
    tc::mbar_wait(&bar, 0);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();
  if (warp == 0) tc::tmem_dealloc2(t, 512);
}
}  // namespace

int tc_bench_launch(int N, int iters, int mode, int ctas, long long* cycles, cudaStream_t st) {
  const size_t smem = 200 * 1024;  // one CTA per SM
  if (mode & 64) {  // CTA pairs: `ctas` clusters of 2 (mode 65: A from TMEM)
    bagel_set_smem_attr(k_tc_bench2, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * ctas, 1, 1);
    cfg.blockDim = dim3(128, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    (void)cudaLaunchKernelEx(&cfg, k_tc_bench2, N, iters, mode & 1, cycles);
    return 1;
  }
  bagel_set_smem_attr(k_tc_bench, smem);
  k_tc_bench<<<ctas, 128, smem, st>>>(N, iters, mode, cycles);
  return 1;
}
