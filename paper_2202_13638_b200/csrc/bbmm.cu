// bbmm.cu -- NEXT-1 at large N: the BBMM estimate of the log marginal likelihood and its gradient
// (Eq.5-6; the paper learns the GP with GPyTorch, whose default engine is BBMM
// [gardner2018]; reading R39), in float64 on the GPU:
//   probes z_1 .. z_t Rademacher from Philox4x32-10 (key = seed, ctr = (i, n >> 2, 0x4242424D, 4),
//   sign bit of word n & 3); ONE batched conjugate-gradient run of exactly J iterations (no
//   preconditioner) solves Khat [u_0 .. u_t] = [y z_1 .. z_t]; each probe's CG coefficients give its
//   Lanczos tridiagonal T_i (T_jj = 1/a_j + b_{j-1}/a_{j-1}, T_{j,j+1} = sqrt(b_j)/a_j), and
//     log|Khat|       ~ (1/t) sum_i ||z_i||^2 e_1^T log(T_i) e_1        (stochastic Lanczos quadrature)
//     y^T Khat^-1 y   ~ y^T u_0
//     tr(Khat^-1 dK)  ~ (1/t) sum_i u_i^T dK z_i                         (Hutchinson)
//     mll = -1/2 y^T u_0 - 1/2 log|Khat| - N/2 log 2 pi,  d mll/d phi_j = 1/2 u_0^T dK_j u_0 - 1/2 tr(..).
// Work per CG iteration: one pass over the stored fp64 Khat (N^2 x 8 bytes) multiplying all t + 1
// vectors at once (HBM-bound: a persistent kernel, one CTA per SM, whose warp 0 also streams Khat
// tiles and the matching slices of the t + 1 search directions into a shared-memory ring with 1-D
// bulk copies (TMA engine) while 8 warps run the float64 FMAs); the gradient is one pass over all
// (a, b) pairs with the kernel regenerated.  Every reduction runs in a fixed order (deterministic); the small
// tridiagonal eigenproblems (J x J) are solved on the host (implicit QL).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>

#include <atomic>
#include <utility>
#include <vector>

#include "bagel_internal.h"
#include "philox.cuh"
#include "tc.cuh"

namespace bbmm {

constexpr int MAXC = 17;      // t + 1 <= 17 columns (probes <= 16)
constexpr int LDV = 256;      // vector / Khat row stride granularity (pads are zero)
constexpr int RED = 256;      // threads of the reduction kernels
constexpr int GC = 9;         // columns per CTA of the gradient pass (t = 8: one pass)
constexpr int GT = 64;        // gradient pair tile

struct Hyp {
  double inv_l2[BAGEL_MAX_D];
  double s, noise;
};

// Khat row-major with row stride ld (pad columns 0)
__global__ void k_khat(const float* __restrict__ X, int N, int ld, int d, Hyp h, double* __restrict__ K) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ld) return;
  for (int i = blockIdx.y; i < N; i += gridDim.y) {  // grid.y is capped at 65535 rows per pass
    if (j >= N) {
      K[(size_t)i * ld + j] = 0.0;
      continue;
    }
    double q = 0.0;
#pragma unroll
    for (int c = 0; c < BAGEL_MAX_D; ++c)
      if (c < d) {
        const double df = (double)X[(size_t)i * d + c] - (double)X[(size_t)j * d + c];
        q += df * df * h.inv_l2[c];
      }
    double v = h.s * exp(-0.5 * q);
    if (i == j) v += h.noise;
    K[(size_t)i * ld + j] = v;
  }
}

// rhs columns [y | z_1 .. z_t] (stride ld): the Rademacher probes from Philox
__global__ void k_rhs(const float* __restrict__ Y, int ystride, int N, int ld, int t, uint64_t seed,
                      double* __restrict__ Z) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  Z[n] = (double)Y[(size_t)n * ystride];
  for (int i = 0; i < t; ++i) {
    const uint4 o = bagel_philox4x32_10(make_uint4((uint32_t)i, (uint32_t)(n >> 2), 0x4242424Du, 4u),
                                        (uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32));
    const uint32_t w = (n & 3) == 0 ? o.x : (n & 3) == 1 ? o.y : (n & 3) == 2 ? o.z : o.w;
    Z[(size_t)(i + 1) * ld + n] = (w >> 31) ? -1.0 : 1.0;
  }
}

// ---------------------------------------------------------------- block MVM  Q = Khat P
// Work units u = (row block rb of TR rows, column chunk ch of TC columns), u = rb NCH + ch; the grid
// (one CTA per SM) splits [0, NRB NCH) into equal contiguous ranges, so every SM streams the same
// number of Khat bytes.  Per unit one lane of warp 0 issues two 2-D tensor copies (TMA: the TR x TC
// Khat tile and the NC x TC direction slice) into one ring stage, NST - 1 units ahead of the compute; consumer warp w owns rows R w .. R w + R - 1 of the unit
// and lanes cover column pairs (16-byte shared loads, each direction pair reused for R rows, each
// Khat pair for NC columns).  Shared-memory wavefronts per unit (reads + TMA writes) bound the rate:
// R = 4 rows per warp; 16 warps (latency hiding) for NC <= 9, 8 warps (fewer direction re-reads) above.  A row block's sums are flushed (fixed butterfly)
// when its last chunk or the CTA's range ends, into partial slot rb + g (unique: the ranges are
// monotone); k_mvm_fixup adds a row block's slots in CTA order (deterministic for a given SM count)
// and emits the CTA partials of p.q for the CG step.
template <int NC>
struct MvmCfg {
  static constexpr int MW = NC <= 9 ? 16 : 8;      // warps (warp 0 also issues the copies)
  static constexpr int R = 4;                      // rows per warp
  static constexpr int TR = MW * R;                // rows per unit
  static constexpr int TC = NC <= 9 ? 64 : 128;    // columns per unit
  static constexpr int KD = TR * TC;               // Khat doubles per stage
  static constexpr int SD = KD + NC * TC;          // stage doubles
  static constexpr int NST = (200 * 1024) / (SD * 8) > 8 ? 8 : (200 * 1024) / (SD * 8);
  static constexpr size_t SMEM = (size_t)NST * SD * 8 + 2 * NST * sizeof(uint64_t);
};

__host__ __device__ __forceinline__ int first_cta(long long u, long long U, int G) {
  return (int)(((u + 1) * G - 1) / U);  // largest g with floor(g U / G) <= u
}

struct MvmMaps {
  CUtensorMap k;  // Khat: FLOAT64 (ld, N) row-major, box (TC, TR); rows >= N arrive zero-filled
  CUtensorMap p;  // directions: FLOAT64 (ld, NC), box (TC, NC)
};

template <int NC>
__global__ void __launch_bounds__(32 * MvmCfg<NC>::MW, 1)
    k_mvm(const __grid_constant__ MvmMaps maps, double* __restrict__ part, int NRB, int NCH) {
  using Cfg = MvmCfg<NC>;
  constexpr int R = Cfg::R, TR = Cfg::TR, TC = Cfg::TC, NST = Cfg::NST, MW = Cfg::MW;
  extern __shared__ __align__(128) uint8_t smraw[];
  double* stg = reinterpret_cast<double*>(smraw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + (size_t)NST * Cfg::SD * 8);
  uint64_t* empty = full + NST;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long U = (long long)NRB * NCH;
  const int G = gridDim.x, g = blockIdx.x;
  const long long u0 = (long long)g * U / G, u1 = (long long)(g + 1) * U / G;
  const int nu = (int)(u1 - u0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], MW);
    }
    tc::fence_mbar_init();
  }
  __syncthreads();
  // warp 0 doubles as the producer: unit i's copies are issued NST - 1 units ahead
  int prb = (int)(u0 / NCH), pch = (int)(u0 % NCH);  // next unit to load
  auto produce = [&](int i) {
    const int s = i % NST;
    tc::mbar_wait(&empty[s], ((uint32_t)(i / NST) & 1u) ^ 1u);
    const int rb = prb, ch = pch;
    if (++pch == NCH) {
      pch = 0;
      ++prb;
    }
    if (lane == 0) {
      tc::mbar_arrive_expect_tx(&full[s], (uint32_t)(Cfg::SD * 8));
      double* dst = stg + (size_t)s * Cfg::SD;
      const uint32_t bar = tc::smem_u32(&full[s]);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
          ::"r"(tc::smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(&maps.k)), "r"(ch * TC), "r"(rb * TR), "r"(bar)
          : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
          ::"r"(tc::smem_u32(dst + Cfg::KD)), "l"(reinterpret_cast<uint64_t>(&maps.p)), "r"(ch * TC), "r"(0), "r"(bar)
          : "memory");
    }
  };
  if (warp == 0)
    for (int i = 0; i < min(NST - 1, nu); ++i) produce(i);
  double acc[R][NC];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[r][c] = 0.0;
  int rb = (int)(u0 / NCH), ch = (int)(u0 % NCH);  // unit being consumed
  for (int i = 0; i < nu; ++i) {
    if (warp == 0 && i + NST - 1 < nu) produce(i + NST - 1);
    const int s = i % NST;
    tc::mbar_wait(&full[s], (uint32_t)(i / NST) & 1u);
    const double2* Ks = reinterpret_cast<const double2*>(stg + (size_t)s * Cfg::SD) + warp * R * (TC / 2);
    const double2* Ps = reinterpret_cast<const double2*>(stg + (size_t)s * Cfg::SD + Cfg::KD);
#pragma unroll
    for (int k = 0; k < TC / 64; ++k) {
      double2 kv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) kv[r] = Ks[r * (TC / 2) + lane + 32 * k];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double2 pv = Ps[c * (TC / 2) + lane + 32 * k];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r][c] = fma(kv[r].y, pv.y, fma(kv[r].x, pv.x, acc[r][c]));
      }
    }
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&empty[s]);
    if (ch == NCH - 1 || i == nu - 1) {
      double* dst = part + (size_t)(rb + g) * NC * TR;
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          double v = acc[r][c];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane == 0) dst[c * TR + warp * R + r] = v;
          acc[r][c] = 0.0;
        }
    }
    if (++ch == NCH) {
      ch = 0;
      ++rb;
    }
  }
}

// Q[c][row] = sum over the CTAs g that touched the row's block (ascending) of slot rb + g; and the
// CTA partials of p_c . q_c (one row per thread, RED rows per CTA: the k_dots partition)
__global__ void __launch_bounds__(RED) k_mvm_fixup(const double* __restrict__ part, int N, int ld, int nc, int TR,
                                                   int NCH, long long U, int G, const double* __restrict__ P,
                                                   double* __restrict__ Q, double* __restrict__ pq_part) {
  __shared__ double red[RED];
  const int row = blockIdx.x * RED + threadIdx.x;
  int g0 = 0, g1 = -1, rb = 0, r = 0;
  if (row < N) {
    rb = row / TR;
    r = row % TR;
    g0 = first_cta((long long)rb * NCH, U, G);
    g1 = first_cta((long long)rb * NCH + NCH - 1, U, G);
  }
  for (int c = 0; c < nc; ++c) {
    double v = 0.0;
    for (int g = g0; g <= g1; ++g) v += part[((size_t)(rb + g) * nc + c) * TR + r];
    if (row < N) Q[(size_t)c * ld + row] = v;
    red[threadIdx.x] = row < N ? P[(size_t)c * ld + row] * v : 0.0;
    __syncthreads();
    for (int o = RED / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) pq_part[(size_t)blockIdx.x * MAXC + c] = red[0];
    __syncthreads();
  }
}

struct MvmPlan {
  int NRB, NCH, G, TR;
};

template <int NC>
static MvmPlan mvm_plan(int N, int ld, int sms) {
  MvmPlan pl;
  pl.TR = MvmCfg<NC>::TR;
  pl.NRB = (N + pl.TR - 1) / pl.TR;
  pl.NCH = ld / MvmCfg<NC>::TC;
  pl.G = (int)std::min<long long>(sms, (long long)pl.NRB * pl.NCH);
  return pl;
}

static PFN_cuTensorMapEncodeTiled_v12000 tmap_encode() {
  static const PFN_cuTensorMapEncodeTiled_v12000 encode = [] {  // thread-safe one-time lookup
    PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&f), cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return f;
  }();
  return encode;
}

static bool tmap_f64(CUtensorMap* m, const double* base, int cols, int rows, int ld, int box_c, int box_r) {
  const auto encode = tmap_encode();
  if (!encode) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  const cuuint32_t box[2] = {(cuuint32_t)box_c, (cuuint32_t)box_r};
  const cuuint32_t es[2] = {1, 1};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// returns false when the tensor maps cannot be encoded
template <int NC>
static bool mvm_launch(const double* K, int N, int ld, const double* P, double* part, double* Q, double* pq_part,
                       int sms, cudaStream_t st) {
  static std::atomic<unsigned long long> devices{0};
  if (bagel_first_on_device(devices))
    cudaFuncSetAttribute(k_mvm<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)MvmCfg<NC>::SMEM);
  const MvmPlan pl = mvm_plan<NC>(N, ld, sms);
  MvmMaps maps;
  if (!tmap_f64(&maps.k, K, ld, N, ld, MvmCfg<NC>::TC, MvmCfg<NC>::TR) ||
      !tmap_f64(&maps.p, P, ld, NC, ld, MvmCfg<NC>::TC, NC))
    return false;
  k_mvm<NC><<<pl.G, 32 * MvmCfg<NC>::MW, MvmCfg<NC>::SMEM, st>>>(maps, part, pl.NRB, pl.NCH);
  k_mvm_fixup<<<(N + RED - 1) / RED, RED, 0, st>>>(part, N, ld, NC, pl.TR, pl.NCH, (long long)pl.NRB * pl.NCH, pl.G,
                                                   P, Q, pq_part);
  return true;
}

using MvmFn = bool (*)(const double*, int, int, const double*, double*, double*, double*, int, cudaStream_t);
template <int... I>
static MvmFn mvm_table_impl(int nc, std::integer_sequence<int, I...>) {
  static const MvmFn t[] = {mvm_launch<I + 1>...};
  return t[nc - 1];
}
static MvmFn mvm_fn(int nc) { return mvm_table_impl(nc, std::make_integer_sequence<int, MAXC>{}); }

// ---------------------------------------------------------------- CG vector steps
// per-CTA partial dot products of column pairs (a_c, b_c), c < nc (stride ld): part[blk][c]
__global__ void __launch_bounds__(RED) k_dots(const double* __restrict__ A, const double* __restrict__ Bv, int N, int ld,
                                              int nc, double* __restrict__ part) {
  __shared__ double red[RED];
  for (int c = 0; c < nc; ++c) {
    double v = 0.0;
    for (int n = blockIdx.x * RED + threadIdx.x; n < N; n += gridDim.x * RED)
      v += A[(size_t)c * ld + n] * Bv[(size_t)c * ld + n];
    red[threadIdx.x] = v;
    __syncthreads();
    for (int o = RED / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) part[(size_t)blockIdx.x * MAXC + c] = red[0];
    __syncthreads();
  }
}

// CG state: rr_hist[j][c] = r_j . r_j of column c (0 once the column stopped: an exactly vanished
// residual).  Iteration j, step 1: alpha = rr_j / (p.q) from the p.q partials (summed in CTA order by
// every CTA), u += alpha p, r -= alpha q, and the CTA partials of r.r.  CTA 0 records alpha.
__global__ void __launch_bounds__(RED) k_update_ur(int N, int ld, int nc, int nblk, const double* __restrict__ pq_part,
                                                   const double* __restrict__ rr_hist, double* __restrict__ al_hist,
                                                   int j, int J, const double* __restrict__ P,
                                                   const double* __restrict__ Qv, double* __restrict__ U,
                                                   double* __restrict__ R, double* __restrict__ rr_part) {
  // rr_part == nullptr (preconditioned CG): no r.r partials, r^T P^-1 r comes from k_apply_w
  __shared__ double alpha_s[MAXC];
  __shared__ double red[RED];
  if (threadIdx.x < nc) {
    const int c = threadIdx.x;
    const double rr = rr_hist[(size_t)j * MAXC + c];
    double pq = 0.0;
    for (int b = 0; b < nblk; ++b) pq += pq_part[(size_t)b * MAXC + c];
    const double a = rr > 0.0 ? rr / pq : 0.0;
    alpha_s[c] = a;
    if (blockIdx.x == 0 && rr > 0.0) al_hist[(size_t)c * J + j] = a;
  }
  __syncthreads();
  const int n = blockIdx.x * RED + threadIdx.x;
  for (int c = 0; c < nc; ++c) {
    double rv = 0.0;
    if (n < N) {
      const size_t o = (size_t)c * ld + n;
      rv = R[o];
      if (rr_hist[(size_t)j * MAXC + c] > 0.0) {
        const double a = alpha_s[c];
        U[o] = fma(a, P[o], U[o]);
        rv = fma(-a, Qv[o], rv);
        R[o] = rv;
      }
    }
    if (!rr_part) continue;
    red[threadIdx.x] = rv * rv;
    __syncthreads();
    for (int o = RED / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) rr_part[(size_t)blockIdx.x * MAXC + c] = red[0];
    __syncthreads();
  }
}

// step 2: beta = rr_{j+1} / rr_j, p = r + beta p (preconditioned: rr = r^T P^-1 r, R = the
// preconditioned residual P^-1 r); CTA 0 records beta, the iteration count and rr_{j+1} (0 when the
// column stopped, so it stays stopped)
__global__ void __launch_bounds__(RED) k_update_p(int N, int ld, int nc, int nblk, const double* __restrict__ rr_part,
                                                  double* __restrict__ rr_hist, double* __restrict__ be_hist,
                                                  int* __restrict__ its, int j, int J, const double* __restrict__ R,
                                                  double* __restrict__ P) {
  __shared__ double beta_s[MAXC];
  if (threadIdx.x < nc) {
    const int c = threadIdx.x;
    const double rr = rr_hist[(size_t)j * MAXC + c];
    double be = 0.0, rr2 = 0.0;
    if (rr > 0.0) {
      for (int b = 0; b < nblk; ++b) rr2 += rr_part[(size_t)b * MAXC + c];
      be = rr2 / rr;
    }
    beta_s[c] = be;
    if (blockIdx.x == 0) {
      rr_hist[(size_t)(j + 1) * MAXC + c] = rr > 0.0 && rr2 > 0.0 ? rr2 : 0.0;
      if (rr > 0.0) {
        be_hist[(size_t)c * J + j] = be;
        its[c] = j + 1;
      }
    }
  }
  __syncthreads();
  const int n = blockIdx.x * RED + threadIdx.x;
  if (n >= N) return;
  for (int c = 0; c < nc; ++c) {
    const size_t o = (size_t)c * ld + n;
    P[o] = fma(beta_s[c], P[o], R[o]);
  }
}

// ---------------------------------------------------------------- preconditioner (reading R40)
constexpr int KMAX = 64;  // preconditioner rank bound

// greedy pivoted Cholesky of K_f = Khat - sn2 I, step m: the pivot = argmax of the residual diagonal
// over the unpivoted rows (lowest index on ties), one CTA; stop[0] = 1 (rank m) once it is <= 0
__global__ void __launch_bounds__(1024) k_pchol_argmax(int N, const double* __restrict__ dg, int* __restrict__ used,
                                                       int m, int* __restrict__ piv, double* __restrict__ dmax,
                                                       int* __restrict__ stop) {
  __shared__ double bv[1024];
  __shared__ int bi[1024];
  if (stop[0]) return;
  double v = 0.0;
  int idx = -1;
  for (int n = threadIdx.x; n < N; n += 1024)
    if (!used[n] && (idx < 0 || dg[n] > v)) {
      v = dg[n];
      idx = n;
    }
  bv[threadIdx.x] = v;
  bi[threadIdx.x] = idx;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double v2 = bv[threadIdx.x + o];
      const int i2 = bi[threadIdx.x + o];
      const int i1 = bi[threadIdx.x];
      if (i2 >= 0 && (i1 < 0 || v2 > bv[threadIdx.x] || (v2 == bv[threadIdx.x] && i2 < i1))) {
        bv[threadIdx.x] = v2;
        bi[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (bi[0] < 0 || !(bv[0] > 0.0)) {
      stop[0] = 1;
      stop[1] = m;
    } else {
      piv[m] = bi[0];
      dmax[0] = bv[0];
      used[bi[0]] = 1;
      stop[1] = m + 1;
    }
  }
}

// column m: L[m][n] = (K_f[p][n] - sum_{j<m} L[j][n] L[j][p]) / sqrt(d_p); d_n -= L[m][n]^2
__global__ void k_pchol_col(int N, int ld, const double* __restrict__ K, double sn2, double* __restrict__ L,
                            double* __restrict__ dg, int m, const int* __restrict__ piv,
                            const double* __restrict__ dmax, const int* __restrict__ stop) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N || stop[0]) return;
  const int p = piv[m];
  double v = K[(size_t)p * ld + n];
  if (n == p) v -= sn2;
  for (int j = 0; j < m; ++j) v -= L[(size_t)j * ld + n] * L[(size_t)j * ld + p];
  const double l = v / sqrt(dmax[0]);
  L[(size_t)m * ld + n] = l;
  dg[n] -= l * l;
}

__global__ void k_pchol_init(int N, int ld, const double* __restrict__ K, double sn2, double* __restrict__ dg,
                             int* __restrict__ used) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  dg[n] = K[(size_t)n * ld + n] - sn2;
  used[n] = 0;
}

// G[i][j] = sum_n L[i][n] L[j][n] (one CTA per pair, fixed-order tree)
__global__ void __launch_bounds__(RED) k_gram(int N, int ld, int k, const double* __restrict__ L, double* __restrict__ G) {
  __shared__ double red[RED];
  const int i = blockIdx.x, j = blockIdx.y;
  double v = 0.0;
  for (int n = threadIdx.x; n < N; n += RED) v += L[(size_t)i * ld + n] * L[(size_t)j * ld + n];
  red[threadIdx.x] = v;
  __syncthreads();
  for (int o = RED / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) G[i * k + j] = red[0];
}

// Gaussian probes z_i = L g_i[0..k) + sn g_i[k..k+N): g_i[j] = Box-Muller word j & 3 of
// Philox(key = seed, ctr = (i, j >> 2, 0x4242424E, 5)); column 0 = y
__device__ __forceinline__ double bbmm_gauss(uint64_t seed, int i, int j) {
  const uint4 o = bagel_philox4x32_10(make_uint4((uint32_t)i, (uint32_t)(j >> 2), 0x4242424Eu, 5u),
                                      (uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32));
  return bagel_normal_d(o, j & 3);
}
__global__ void k_rhs_pc(const float* __restrict__ Y, int ystride, int N, int ld, int t, int k, uint64_t seed,
                         const double* __restrict__ L, double sn, double* __restrict__ Z) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  Z[n] = (double)Y[(size_t)n * ystride];
  for (int i = 0; i < t; ++i) {
    double v = sn * bbmm_gauss(seed, i, k + n);
    for (int m = 0; m < k; ++m) v += L[(size_t)m * ld + n] * bbmm_gauss(seed, i, m);
    Z[(size_t)(i + 1) * ld + n] = v;
  }
}

// Woodbury apply W = P^-1 V = (V - L C^-1 L^T V) / sn2 for the nc columns, in three steps.
// (a) CTA partials of L^T V: part[blk][m][c] (RED rows per CTA: the k_dots partition; per (m, c) a
//     fixed shuffle butterfly per warp, then the 8 warps in order)
__global__ void __launch_bounds__(RED) k_lt_part(int N, int ld, int nc, int k, const double* __restrict__ L,
                                                 const double* __restrict__ V, double* __restrict__ part) {
  __shared__ double red[RED / 32][MAXC];
  const int n = blockIdx.x * RED + threadIdx.x, warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  double v[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) v[c] = c < nc && n < N ? V[(size_t)c * ld + n] : 0.0;
  for (int m = 0; m < k; ++m) {
    const double l = n < N ? L[(size_t)m * ld + n] : 0.0;
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      if (c >= nc) break;
      double x = l * v[c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) red[warp][c] = x;
    }
    __syncthreads();
    if (threadIdx.x < nc) {
      double x = 0.0;
      for (int w = 0; w < RED / 32; ++w) x += red[w][threadIdx.x];
      part[((size_t)blockIdx.x * KMAX + m) * MAXC + threadIdx.x] = x;
    }
    __syncthreads();
  }
}
// (b) one CTA: T[m][c] = sum over the CTAs in order; Yk[c][i] = sum_m Cinv[i][m] T[m][c]
__global__ void __launch_bounds__(1024) k_lt_fin(int nblk, int nc, int k, const double* __restrict__ part,
                                                 const double* __restrict__ Cinv, double* __restrict__ Yk) {
  __shared__ double T[KMAX][MAXC];
  for (int idx = threadIdx.x; idx < k * nc; idx += blockDim.x) {
    const int m = idx / nc, c = idx % nc;
    double x = 0.0;
    for (int b = 0; b < nblk; ++b) x += part[((size_t)b * KMAX + m) * MAXC + c];
    T[m][c] = x;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < k * nc; idx += blockDim.x) {
    const int i = idx / nc, c = idx % nc;
    double x = 0.0;
    for (int m = 0; m < k; ++m) x += Cinv[i * k + m] * T[m][c];
    Yk[c * KMAX + i] = x;
  }
}
// (c) W = (V - L Yk) / sn2 (and copies into W2 when given), the CTA partials of V^T W per column
__global__ void __launch_bounds__(RED) k_apply_w(int N, int ld, int nc, int k, const double* __restrict__ L,
                                                 const double* __restrict__ Yk, double sn2,
                                                 const double* __restrict__ V, double* __restrict__ W,
                                                 double* __restrict__ W2, double* __restrict__ W3,
                                                 double* __restrict__ rz_part) {
  __shared__ double red[RED];
  __shared__ double ys[MAXC][KMAX];
  for (int idx = threadIdx.x; idx < nc * k; idx += RED) ys[idx / k][idx % k] = Yk[(idx / k) * KMAX + idx % k];
  __syncthreads();
  const int n = blockIdx.x * RED + threadIdx.x;
  for (int c = 0; c < nc; ++c) {
    double x = 0.0;
    if (n < N) {
      const size_t o = (size_t)c * ld + n;
      double a = V[o];
      for (int m = 0; m < k; ++m) a -= L[(size_t)m * ld + n] * ys[c][m];
      const double w = a / sn2;
      W[o] = w;
      if (W2) W2[o] = w;
      if (W3) W3[o] = w;
      x = V[o] * w;
    }
    red[threadIdx.x] = x;
    __syncthreads();
    for (int o = RED / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) rz_part[(size_t)blockIdx.x * MAXC + c] = red[0];
    __syncthreads();
  }
}

// ---------------------------------------------------------------- gradient pass
// For every pair (a, b): w_c[a] v_c[b] (K_ab r2_ab,l .., K_ab) for the GC columns c = GC blockIdx.y + ..,
// with (w_0, v_0) = (u_0, u_0), (w_c, v_c) = (u_c, z_c), r2_l = (x_al - x_bl)^2 / l_l^2 and K_ab =
// s exp(-sum_l r2_l / 2) regenerated (cheaper than re-reading Khat).  A CTA owns GT b's (one per thread
// of each quarter: x_b and v_c[b] in registers) and walks every a in tiles of GT (x_a, w_c[a] staged
// in shared memory, broadcast reads); the thread sums are reduced by a fixed shuffle butterfly, then
// across the 8 warps in warp order.  Per-CTA partials [b tile][c][MAX_D + 1] (l = MAX_D holds the
// signal-variance term sum w K v).
__global__ void __launch_bounds__(256) k_grad_pairs(const float* __restrict__ X, int N, int ld, int d, Hyp h, int nc,
                                                    const double* __restrict__ U, const double* __restrict__ Z,
                                                    double* __restrict__ part) {
  __shared__ double xa_s[GT][BAGEL_MAX_D];
  __shared__ double wa_s[GC][GT];
  __shared__ double wred[8][GC][BAGEL_MAX_D + 1];
  const int tj = blockIdx.x, c0 = blockIdx.y * GC;
  const int ncl = min(GC, nc - c0);
  const int bl = threadIdx.x % GT, ag = threadIdx.x / GT;
  const int b = tj * GT + bl;
  double xb[BAGEL_MAX_D], vb[GC];
#pragma unroll
  for (int l = 0; l < BAGEL_MAX_D; ++l) xb[l] = b < N && l < d ? (double)X[(size_t)b * d + l] : 0.0;
#pragma unroll
  for (int c = 0; c < GC; ++c) {
    const int cc = c0 + c;
    vb[c] = c < ncl && b < N ? (cc == 0 ? U[b] : Z[(size_t)cc * ld + b]) : 0.0;
  }
  double acc[GC][BAGEL_MAX_D + 1];
#pragma unroll
  for (int c = 0; c < GC; ++c)
#pragma unroll
    for (int l = 0; l <= BAGEL_MAX_D; ++l) acc[c][l] = 0.0;
  for (int a0 = 0; a0 < N; a0 += GT) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < GT * BAGEL_MAX_D; idx += 256) {
      const int a = a0 + idx / BAGEL_MAX_D, l = idx % BAGEL_MAX_D;
      xa_s[idx / BAGEL_MAX_D][l] = a < N && l < d ? (double)X[(size_t)a * d + l] : 0.0;
    }
    for (int idx = threadIdx.x; idx < GC * GT; idx += 256) {
      const int c = idx / GT, a = a0 + idx % GT;
      wa_s[c][idx % GT] = c < ncl && a < N ? U[(size_t)(c0 + c) * ld + a] : 0.0;
    }
    __syncthreads();
    const int alim = min(GT, N - a0);
    if (b < N)
      for (int al = ag; al < alim; al += 256 / GT) {
        double r2[BAGEL_MAX_D], q = 0.0;
#pragma unroll
        for (int l = 0; l < BAGEL_MAX_D; ++l) {
          r2[l] = 0.0;
          if (l < d) {
            const double df = xa_s[al][l] - xb[l];
            r2[l] = df * df * h.inv_l2[l];
            q += r2[l];
          }
        }
        const double k = h.s * exp(-0.5 * q);
#pragma unroll
        for (int c = 0; c < GC; ++c) {
          const double wv = wa_s[c][al] * vb[c] * k;
#pragma unroll
          for (int l = 0; l < BAGEL_MAX_D; ++l) acc[c][l] = fma(wv, r2[l], acc[c][l]);
          acc[c][BAGEL_MAX_D] += wv;
        }
      }
  }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
#pragma unroll
  for (int c = 0; c < GC; ++c)
#pragma unroll
    for (int l = 0; l <= BAGEL_MAX_D; ++l) {
      double v = acc[c][l];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) wred[warp][c][l] = v;
    }
  __syncthreads();
  if (threadIdx.x < GC * (BAGEL_MAX_D + 1)) {
    const int c = threadIdx.x / (BAGEL_MAX_D + 1), l = threadIdx.x % (BAGEL_MAX_D + 1);
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += wred[w][c][l];
    if (c < ncl) part[((size_t)tj * MAXC + c0 + c) * (BAGEL_MAX_D + 1) + l] = v;
  }
}

// fixed-order sum of the pair partials: out[c][l]; one CTA per (c, l), strided partial sums then a tree
__global__ void __launch_bounds__(RED) k_grad_sum(const double* __restrict__ part, size_t nblk, int d,
                                                  double* __restrict__ out) {
  __shared__ double red[RED];
  const int c = blockIdx.x, l = blockIdx.y;
  if (l >= d && l < BAGEL_MAX_D) return;
  double v = 0.0;
  for (size_t b = threadIdx.x; b < nblk; b += RED) v += part[(b * MAXC + c) * (BAGEL_MAX_D + 1) + l];
  red[threadIdx.x] = v;
  __syncthreads();
  for (int o = RED / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[c * (BAGEL_MAX_D + 1) + l] = red[0];
}

}  // namespace bbmm

// e_1^T log(T) e_1 of a symmetric tridiagonal matrix (diagonal a[0..n), off-diagonal b[0..n-1)) by
// the implicit QL algorithm with Wilkinson shifts, tracking the first row of the eigenvector matrix.
static double tridiag_e1_log_e1(std::vector<double> a, std::vector<double> b) {
  const int n = (int)a.size();
  std::vector<double> e(n, 0.0), z(n, 0.0);
  for (int i = 0; i + 1 < n; ++i) e[i] = b[i];
  z[0] = 1.0;  // first components of the eigenvectors
  for (int l = 0; l < n; ++l) {
    for (int iter = 0; iter < 60; ++iter) {
      int m = l;
      for (; m < n - 1; ++m) {
        const double dd = fabs(a[m]) + fabs(a[m + 1]);
        if (fabs(e[m]) <= 1e-16 * dd) break;
      }
      if (m == l) break;
      double g = (a[l + 1] - a[l]) / (2.0 * e[l]);
      double r = hypot(g, 1.0);
      g = a[m] - a[l] + e[l] / (g + (g >= 0 ? r : -r));
      double s = 1.0, c = 1.0, p = 0.0;
      int i = m - 1;
      for (; i >= l; --i) {
        double f = s * e[i], bb = c * e[i];
        r = hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) {
          a[i + 1] -= p;
          e[m] = 0.0;
          break;
        }
        s = f / r;
        c = g / r;
        g = a[i + 1] - p;
        r = (a[i] - g) * s + 2.0 * c * bb;
        p = s * r;
        a[i + 1] = g + p;
        g = c * r - bb;
        const double zf = z[i + 1];
        z[i + 1] = s * z[i] + c * zf;
        z[i] = c * z[i] - s * zf;
      }
      if (r == 0.0 && i >= l) continue;
      a[l] -= p;
      e[l] = g;
      e[m] = 0.0;
    }
  }
  double v = 0.0;
  for (int k = 0; k < n; ++k) v += z[k] * z[k] * log(a[k]);
  return v;
}

using namespace bbmm;

static size_t bbmm_ld(int N) { return (size_t)(N + LDV - 1) / LDV * LDV; }
constexpr int MAX_G = 1024;  // bound on the MVM grid (SM count) for the partial slots

size_t bbmm_workspace_doubles(int N, int nc, int J) {
  const size_t ld = bbmm_ld(N);
  const size_t nblk = (N + RED - 1) / RED, ntile = (N + GT - 1) / GT, nrb = (N + 31) / 32;
  return (size_t)N * ld + 7 * (size_t)nc * ld + 2 * (size_t)nc * J + 2 * std::max<size_t>(nblk, 1) * MAXC +
         (size_t)(J + 1) * MAXC + ntile * MAXC * (BAGEL_MAX_D + 1) + MAXC * (BAGEL_MAX_D + 1) +
         (nrb + MAX_G) * MAXC * 32 +
         /* preconditioner: L, residual diagonal, pivot flags, L^T V partials, Yk, C^-1, pivots */
         (size_t)KMAX * ld + 2 * ld + std::max<size_t>(nblk, 1) * KMAX * MAXC + MAXC * KMAX + KMAX * KMAX +
         2 * KMAX + 8;
}

// Cholesky (lower, in place) and inverse of the k x k matrix C = sn2 I + L^T L (host, k <= 64);
// returns log|C| or NaN if C is not positive definite.
static double small_spd_inverse(std::vector<double>& C, int k, std::vector<double>& Cinv) {
  double ld = 0.0;
  for (int j = 0; j < k; ++j) {
    double a = C[(size_t)j * k + j];
    for (int m = 0; m < j; ++m) a -= C[(size_t)j * k + m] * C[(size_t)j * k + m];
    if (!(a > 0.0)) return NAN;
    const double r = sqrt(a);
    C[(size_t)j * k + j] = r;
    ld += 2.0 * log(r);
    for (int i = j + 1; i < k; ++i) {
      double v = C[(size_t)i * k + j];
      for (int m = 0; m < j; ++m) v -= C[(size_t)i * k + m] * C[(size_t)j * k + m];
      C[(size_t)i * k + j] = v / r;
    }
  }
  Cinv.assign((size_t)k * k, 0.0);
  std::vector<double> e(k);
  for (int col = 0; col < k; ++col) {  // C^-1 e_col by forward / back substitution
    for (int i = 0; i < k; ++i) {
      double v = i == col ? 1.0 : 0.0;
      for (int m = 0; m < i; ++m) v -= C[(size_t)i * k + m] * e[m];
      e[i] = v / C[(size_t)i * k + i];
    }
    for (int i = k - 1; i >= 0; --i) {
      double v = e[i];
      for (int m = i + 1; m < k; ++m) v -= C[(size_t)m * k + i] * e[m];
      e[i] = v / C[(size_t)i * k + i];
    }
    for (int i = 0; i < k; ++i) Cinv[(size_t)i * k + col] = e[i];
  }
  return ld;
}

// Runs the BBMM estimate on the stream and returns it on the host: logdet, quad (y^T u_0) and, when
// grad is non-NULL, d mll / d phi (d + 2).  kp > 0: GPyTorch's rank-kp pivoted-Cholesky preconditioner
// (reading R40); *rank_out = the rank reached.  ws: bbmm_workspace_doubles(N, t + 1, J) doubles;
// its: nc ints.
int bbmm_launch(const float* X, const float* Y, int ystride, int N, int d, const double* log_hyp, int t, int J,
                int kp, uint64_t seed, double* ws, int* its_dev, double* logdet, double* quad, double* grad,
                int* rank_out, cudaStream_t st) {
  const int nc = t + 1;
  Hyp h{};
  for (int c = 0; c < d; ++c) h.inv_l2[c] = exp(-2.0 * log_hyp[c]);
  h.s = exp(log_hyp[d]);
  h.noise = exp(log_hyp[d + 1]);
  const int nblk = (N + RED - 1) / RED;
  const int ld = (int)bbmm_ld(N);
  const int ntile = (N + GT - 1) / GT;
  double* K = ws;
  double* Z = K + (size_t)N * ld;
  double* U = Z + (size_t)nc * ld;
  double* R = U + (size_t)nc * ld;
  double* P = R + (size_t)nc * ld;
  double* Qv = P + (size_t)nc * ld;
  double* W = Qv + (size_t)nc * ld;   // preconditioned residual P^-1 r
  double* W0 = W + (size_t)nc * ld;   // P^-1 rhs (the gradient's second vectors)
  double* al = W0 + (size_t)nc * ld;
  double* be = al + (size_t)nc * J;
  double* part = be + (size_t)nc * J;                       // p.q partials / general dot partials
  double* rr_part = part + (size_t)std::max(nblk, 1) * MAXC;  // r.r (r^T P^-1 r) partials
  double* rr_hist = rr_part + (size_t)std::max(nblk, 1) * MAXC;
  double* gpart = rr_hist + (size_t)(J + 1) * MAXC;
  double* gsum = gpart + (size_t)ntile * MAXC * (BAGEL_MAX_D + 1);
  double* mpart = gsum + MAXC * (BAGEL_MAX_D + 1);
  double* Lp = mpart + ((size_t)(N + 31) / 32 + MAX_G) * MAXC * 32;
  double* dg = Lp + (size_t)KMAX * ld;
  int* used = reinterpret_cast<int*>(dg + ld);
  double* ltp = dg + 2 * (size_t)ld;
  double* Yk = ltp + (size_t)std::max(nblk, 1) * KMAX * MAXC;
  double* Cinv_d = Yk + MAXC * KMAX;
  double* dmax = Cinv_d + KMAX * KMAX;
  int* piv = reinterpret_cast<int*>(dmax + 1);   // KMAX ints
  int* stop = piv + KMAX;                        // [stop, rank]
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  sms = std::min(sms, MAX_G);

  k_khat<<<dim3(ld / 256, std::min(N, 65535)), 256, 0, st>>>(X, N, ld, d, h, K);
  const MvmFn mvm = mvm_fn(nc);
  cudaMemsetAsync(Z, 0, sizeof(double) * 7 * (size_t)nc * ld, st);  // Z U R P Q W W0, pads stay 0
  cudaMemsetAsync(its_dev, 0, sizeof(int) * nc, st);
  int k = 0;
  double logdetP = 0.0;
  std::vector<double> rr0(MAXC, 0.0);
  std::vector<double> part_h((size_t)nblk * MAXC);
  if (kp > 0) {
    // rank-kp pivoted Cholesky of K_f (2 launches per pivot), then C = sn2 I + L^T L on the host
    cudaMemsetAsync(stop, 0, 2 * sizeof(int), st);
    k_pchol_init<<<(N + 255) / 256, 256, 0, st>>>(N, ld, K, h.noise, dg, used);
    for (int m = 0; m < kp; ++m) {
      k_pchol_argmax<<<1, 1024, 0, st>>>(N, dg, used, m, piv, dmax, stop);
      k_pchol_col<<<(N + 255) / 256, 256, 0, st>>>(N, ld, K, h.noise, Lp, dg, m, piv, dmax, stop);
    }
    int stop_h[2] = {0, 0};
    cudaMemcpyAsync(stop_h, stop, sizeof(stop_h), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
    k = stop_h[1];
    if (k > 0) {
      k_gram<<<dim3(k, k), RED, 0, st>>>(N, ld, k, Lp, Cinv_d);  // L^T L, staged in the C^-1 slot
      std::vector<double> C((size_t)k * k), Ci;
      cudaMemcpyAsync(C.data(), Cinv_d, sizeof(double) * (size_t)k * k, cudaMemcpyDeviceToHost, st);
      if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
      for (int i = 0; i < k; ++i) C[(size_t)i * k + i] += h.noise;
      const double ldC = small_spd_inverse(C, k, Ci);
      if (!(ldC == ldC)) return -3;
      logdetP = ldC;
      cudaMemcpyAsync(Cinv_d, Ci.data(), sizeof(double) * (size_t)k * k, cudaMemcpyHostToDevice, st);
    }
    logdetP += (double)(N - k) * log(h.noise);
    // Gaussian probes z ~ N(0, P); W0 = P^-1 [y z_1 ..], P = R = rhs, rz_0 = rhs^T W0
    k_rhs_pc<<<(N + 255) / 256, 256, 0, st>>>(Y, ystride, N, ld, t, k, seed, Lp, sqrt(h.noise), Z);
    cudaMemcpyAsync(R, Z, sizeof(double) * (size_t)nc * ld, cudaMemcpyDeviceToDevice, st);
    k_lt_part<<<nblk, RED, 0, st>>>(N, ld, nc, k, Lp, Z, ltp);
    k_lt_fin<<<1, 1024, 0, st>>>(nblk, nc, k, ltp, Cinv_d, Yk);
    k_apply_w<<<nblk, RED, 0, st>>>(N, ld, nc, k, Lp, Yk, h.noise, Z, W0, P, W, part);
  } else {
    k_rhs<<<(N + 255) / 256, 256, 0, st>>>(Y, ystride, N, ld, t, seed, Z);
    cudaMemcpyAsync(R, Z, sizeof(double) * (size_t)nc * ld, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(P, Z, sizeof(double) * (size_t)nc * ld, cudaMemcpyDeviceToDevice, st);
    k_dots<<<nblk, RED, 0, st>>>(R, R, N, ld, nc, part);
  }
  // rr_0 (r.r, or r^T P^-1 r): CTA partials summed in CTA order on the host
  cudaMemcpyAsync(part_h.data(), part, sizeof(double) * (size_t)nblk * MAXC, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
  for (int c = 0; c < nc; ++c)
    for (int b = 0; b < nblk; ++b) rr0[c] += part_h[(size_t)b * MAXC + c];
  cudaMemcpyAsync(rr_hist, rr0.data(), sizeof(double) * MAXC, cudaMemcpyHostToDevice, st);
  for (int j = 0; j < J; ++j) {
    if (!mvm(K, N, ld, P, mpart, Qv, part, sms, st)) return -2;
    if (kp > 0) {
      k_update_ur<<<nblk, RED, 0, st>>>(N, ld, nc, nblk, part, rr_hist, al, j, J, P, Qv, U, R, nullptr);
      k_lt_part<<<nblk, RED, 0, st>>>(N, ld, nc, k, Lp, R, ltp);
      k_lt_fin<<<1, 1024, 0, st>>>(nblk, nc, k, ltp, Cinv_d, Yk);
      k_apply_w<<<nblk, RED, 0, st>>>(N, ld, nc, k, Lp, Yk, h.noise, R, W, nullptr, nullptr, rr_part);
      k_update_p<<<nblk, RED, 0, st>>>(N, ld, nc, nblk, rr_part, rr_hist, be, its_dev, j, J, W, P);
    } else {
      k_update_ur<<<nblk, RED, 0, st>>>(N, ld, nc, nblk, part, rr_hist, al, j, J, P, Qv, U, R, rr_part);
      k_update_p<<<nblk, RED, 0, st>>>(N, ld, nc, nblk, rr_part, rr_hist, be, its_dev, j, J, R, P);
    }
  }
  const double* Vg = kp > 0 ? W0 : Z;  // the gradient's second vectors: P^-1 z_i (or z_i)
  // y^T u_0 (column 0 of the rhs is y)
  k_dots<<<nblk, RED, 0, st>>>(Z, U, N, ld, 1, part);
  std::vector<double> al_h((size_t)nc * J), be_h((size_t)nc * J);
  std::vector<int> its_h(nc);
  cudaMemcpyAsync(part_h.data(), part, sizeof(double) * (size_t)nblk * MAXC, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(al_h.data(), al, sizeof(double) * (size_t)nc * J, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(be_h.data(), be, sizeof(double) * (size_t)nc * J, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(its_h.data(), its_dev, sizeof(int) * nc, cudaMemcpyDeviceToHost, st);
  std::vector<double> gs_h((size_t)MAXC * (BAGEL_MAX_D + 1), 0.0);
  if (grad) {
    k_grad_pairs<<<dim3(ntile, (nc + GC - 1) / GC), 256, 0, st>>>(X, N, ld, d, h, nc, U, Vg, gpart);
    k_grad_sum<<<dim3(nc, BAGEL_MAX_D + 1), RED, 0, st>>>(gpart, (size_t)ntile, d, gsum);
    cudaMemcpyAsync(gs_h.data(), gsum, sizeof(double) * (size_t)MAXC * (BAGEL_MAX_D + 1), cudaMemcpyDeviceToHost, st);
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
  double q = 0.0;
  for (int b = 0; b < nblk; ++b) q += part_h[(size_t)b * MAXC];
  *quad = q;
  double lds = 0.0;
  for (int i = 1; i <= t; ++i) {
    const int n = its_h[i];
    std::vector<double> ta(n), tb(n > 0 ? n - 1 : 0);
    const double* a_ = al_h.data() + (size_t)i * J;
    const double* b_ = be_h.data() + (size_t)i * J;
    for (int j = 0; j < n; ++j) {
      ta[j] = 1.0 / a_[j] + (j > 0 ? b_[j - 1] / a_[j - 1] : 0.0);
      if (j + 1 < n) tb[j] = sqrt(b_[j]) / a_[j];
    }
    lds += rr0[i] * tridiag_e1_log_e1(ta, tb);  // z^T P^-1 z (= ||z||^2 = N for Rademacher, kp = 0)
  }
  *logdet = logdetP + lds / (double)t;
  if (rank_out) *rank_out = k;
  if (grad) {
    // noise derivative: dKhat / dlog sn2 = sn2 I -> w^T v sums (u_0.u_0 and u_c.v_c)
    std::vector<double> dots(nc, 0.0);
    k_dots<<<nblk, RED, 0, st>>>(U, U, N, ld, 1, part);
    cudaMemcpyAsync(part_h.data(), part, sizeof(double) * (size_t)nblk * MAXC, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
    for (int b = 0; b < nblk; ++b) dots[0] += part_h[(size_t)b * MAXC];
    k_dots<<<nblk, RED, 0, st>>>(U + ld, Vg + ld, N, ld, t, part);
    cudaMemcpyAsync(part_h.data(), part, sizeof(double) * (size_t)nblk * MAXC, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
    for (int c = 1; c < nc; ++c)
      for (int b = 0; b < nblk; ++b) dots[c] += part_h[(size_t)b * MAXC + c - 1];
    for (int l = 0; l < d + 2; ++l) {
      double q0, tr = 0.0;
      if (l < d + 1) {
        const int src = l < d ? l : BAGEL_MAX_D;
        q0 = gs_h[src];
        for (int c = 1; c < nc; ++c) tr += gs_h[(size_t)c * (BAGEL_MAX_D + 1) + src];
      } else {
        q0 = h.noise * dots[0];
        for (int c = 1; c < nc; ++c) tr += h.noise * dots[c];
      }
      grad[l] = 0.5 * q0 - 0.5 * tr / (double)t;
    }
  }
  return 0;
}
