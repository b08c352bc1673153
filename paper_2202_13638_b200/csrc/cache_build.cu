// cache_build.cu -- the one-time LOVE cache ("the one-time
// caching operation required for BAGEL's fast predictions takes ~0.6s"),
// built in float64 on the GPU (plain CUDA, north star item (4)):
//   Khat = K(X, X) + sigma_n^2 I                         (Eq.4)
//   Lanczos(Khat, q1 = y/||y||, k steps), classical Gram-Schmidt twice,
//   deterministic Philox restart on breakdown           (reading R20)
//   R = L_T^-1 Q^T with T = L_T L_T^T (bidiagonal L_T)   (LOVE root, K^-1 ~ R^T R)
//   alpha = Khat^-1 y by blocked right-looking Cholesky (reading R21)
//   V = s [alpha | alpha o X | R^T] packed for the hot path (fp32).
// Every reduction runs in a fixed order (run-to-run bitwise determinism).
// Roofline: Khat MVMs are HBM-bound (8 N^2 bytes each); the Cholesky trailing
// update is FP64-FMA bound (N^3/3 flops).  Both are one-time costs.
#include "bagel_internal.h"
#include "philox.cuh"

namespace {

struct EllD {
  double inv_l2[BAGEL_MAX_D];
};

__global__ void k_khat(const float* __restrict__ X, int N, int d, EllD e, double s, double noise,
                       double* __restrict__ K) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  for (int i = blockIdx.y; i < N; i += gridDim.y) {  // grid.y is capped at 65535 rows per pass
    double q = 0.0;
    for (int c = 0; c < d; ++c) {
      const double df = (double)X[(size_t)i * d + c] - (double)X[(size_t)j * d + c];
      q += df * df * e.inv_l2[c];
    }
    double v = s * exp(-0.5 * q);
    if (i == j) v += noise;
    K[(size_t)i * N + j] = v;
  }
}

constexpr int NB = 64;  // Cholesky block

// Factor the NB x NB diagonal block in shared memory (lower, right-looking).
__global__ void __launch_bounds__(256) k_potrf_diag(double* __restrict__ A, int N, int kb,
                                                    int* __restrict__ pivot_flag) {
  __shared__ double L[NB][NB + 1];
  const int nb = min(NB, N - kb);
  const int tid = threadIdx.x;
  if (*pivot_flag) return;  // an earlier block already failed
  for (int idx = tid; idx < nb * nb; idx += blockDim.x) {
    const int i = idx / nb, j = idx % nb;
    L[i][j] = (j <= i) ? A[(size_t)(kb + i) * N + kb + j] : 0.0;
  }
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    const double djj = L[j][j];
    if (!(djj > 0.0)) {
      if (tid == 0) *pivot_flag = kb + j + 1;
      return;  // uniform: every thread reads the same djj
    }
    const double ljj = sqrt(djj);
    __syncthreads();
    if (tid == 0) L[j][j] = ljj;
    for (int i = j + 1 + tid; i < nb; i += blockDim.x) L[i][j] /= ljj;
    __syncthreads();
    const int rem = nb - j - 1;
    for (int idx = tid; idx < rem * rem; idx += blockDim.x) {
      const int i = j + 1 + idx / rem, c = j + 1 + idx % rem;
      if (c <= i) L[i][c] -= L[i][j] * L[c][j];
    }
    __syncthreads();
  }
  for (int idx = tid; idx < nb * nb; idx += blockDim.x) {
    const int i = idx / nb, j = idx % nb;
    A[(size_t)(kb + i) * N + kb + j] = (j <= i) ? L[i][j] : 0.0;
  }
}

// Panel solve: rows i >= kb + nb: L[i, kb:kb+nb] = A[i, kb:kb+nb] L11^-T (one thread per row).
constexpr int TR = 32;  // rows per panel-solve CTA
__global__ void __launch_bounds__(TR) k_trsm_panel(double* __restrict__ A, int N, int kb,
                                                   const int* __restrict__ pivot_flag) {
  __shared__ double L11[NB * (NB + 1) / 2];  // packed lower triangle, row j at j (j + 1) / 2
  __shared__ double Xr[TR][NB + 1];
  if (*pivot_flag) return;
  const int nb = min(NB, N - kb);
  const int r0 = kb + nb + blockIdx.x * TR;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < nb * nb; idx += TR) {
    const int i = idx / nb, j = idx % nb;
    if (j <= i) L11[i * (i + 1) / 2 + j] = A[(size_t)(kb + i) * N + kb + j];
  }
  for (int idx = tid; idx < TR * nb; idx += TR) {
    const int r = idx / nb, j = idx % nb;
    Xr[r][j] = (r0 + r < N) ? A[(size_t)(r0 + r) * N + kb + j] : 0.0;
  }
  __syncthreads();
  if (r0 + tid < N) {
    for (int j = 0; j < nb; ++j) {
      const double* Lj = L11 + j * (j + 1) / 2;
      double acc = Xr[tid][j];
      for (int l = 0; l < j; ++l) acc -= Xr[tid][l] * Lj[l];
      Xr[tid][j] = acc / Lj[j];
    }
  }
  __syncthreads();
  for (int idx = tid; idx < TR * nb; idx += TR) {
    const int r = idx / nb, j = idx % nb;
    if (r0 + r < N) A[(size_t)(r0 + r) * N + kb + j] = Xr[r][j];
  }
}

// Deferred trailing update A[i][j] -= sum_{l < nbk} A[i][kb + l] A[j][kb + l] for base <= j <= i < N,
// j < col_end (lower triangle), on 128 x 128 tiles: 16 x 16 threads, 8 x 8 accumulators each; the two
// 128 x 8 slices of the L columns per K step are double-buffered in shared memory (the next slice's
// global loads are in flight while the current one is multiplied).
constexpr int ST = 128, SK = 8;
__global__ void __launch_bounds__(256) k_syrk(double* __restrict__ A, int N, int kb, int nbk, int base, int col_end,
                                              const int* __restrict__ pivot_flag) {
  if (*pivot_flag) return;
  const int i0 = base + blockIdx.y * ST, j0 = base + blockIdx.x * ST;
  if (j0 >= col_end || j0 > i0 + ST - 1) return;  // past the columns, or entirely above the diagonal
  __shared__ double As[2][SK][ST];
  __shared__ double Bs[2][SK][ST];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  // staging: thread -> (row r = threadIdx.x / 2, K elements 4 (threadIdx.x % 2) .. + 3) of both slices
  const int sr = threadIdx.x / 2, sl = 4 * (threadIdx.x % 2);
  const bool ai = i0 + sr < N, bj = j0 + sr < N;
  const double* arow = A + (size_t)(i0 + sr) * N + kb;
  const double* brow = A + (size_t)(j0 + sr) * N + kb;
  double ra[4], rb[4];
  auto fetch = [&](int l0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int l = l0 + sl + q;
      ra[q] = ai && l < nbk ? arow[l] : 0.0;
      rb[q] = bj && l < nbk ? brow[l] : 0.0;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      As[buf][sl + q][sr] = ra[q];
      Bs[buf][sl + q][sr] = rb[q];
    }
  };
  double acc[8][8];
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[u][v] = 0.0;
  fetch(0);
  stash(0);
  __syncthreads();
  const int nch = (nbk + SK - 1) / SK;
  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
    if (c + 1 < nch) fetch((c + 1) * SK);
#pragma unroll
    for (int l = 0; l < SK; ++l) {
      double a[8], b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a[u] = As[buf][l][ty + 16 * u];
        b[u] = Bs[buf][l][tx + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    if (c + 1 < nch) stash(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int i = i0 + ty + 16 * u, j = j0 + tx + 16 * v;
      if (i < N && j < col_end && j <= i) A[(size_t)i * N + j] -= acc[u][v];
    }
}

// ---- triangular solves (blocked; diagonal block sequential in shared memory)
__global__ void k_widen_col(const float* __restrict__ y, int stride, int N, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) out[i] = (double)y[(size_t)i * stride];
}

__global__ void __launch_bounds__(64) k_trsv_diag_fwd(const double* __restrict__ L, int N, int kb,
                                                      double* __restrict__ z) {
  __shared__ double zs[NB];
  const int nb = min(NB, N - kb), tid = threadIdx.x;
  if (tid < nb) zs[tid] = z[kb + tid];
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    if (tid == j) zs[j] /= L[(size_t)(kb + j) * N + kb + j];
    __syncthreads();
    if (tid > j && tid < nb) zs[tid] -= L[(size_t)(kb + tid) * N + kb + j] * zs[j];
    __syncthreads();
  }
  if (tid < nb) z[kb + tid] = zs[tid];
}

// z[i] -= sum_l L[i][kb+l] z[kb+l], i >= kb+nb; one warp per row.
__global__ void k_gemv_fwd(const double* __restrict__ L, int N, int kb, double* __restrict__ z) {
  const int nb = min(NB, N - kb);
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  const int i = kb + nb + warp;
  if (i >= N) return;
  double acc = 0.0;
  for (int l = lane; l < nb; l += 32) acc += L[(size_t)i * N + kb + l] * z[kb + l];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) z[i] -= acc;
}

__global__ void __launch_bounds__(64) k_trsv_diag_bwd(const double* __restrict__ L, int N, int kb,
                                                      double* __restrict__ a) {
  __shared__ double as[NB];
  const int nb = min(NB, N - kb), tid = threadIdx.x;
  if (tid < nb) as[tid] = a[kb + tid];
  __syncthreads();
  for (int j = nb - 1; j >= 0; --j) {
    if (tid == j) as[j] /= L[(size_t)(kb + j) * N + kb + j];
    __syncthreads();
    if (tid < j) as[tid] -= L[(size_t)(kb + j) * N + kb + tid] * as[j];
    __syncthreads();
  }
  if (tid < nb) a[kb + tid] = as[tid];
}

// a[i] -= sum_l L[kb+l][i] a[kb+l], i < kb; one thread per column (coalesced).
__global__ void k_gemv_bwd(const double* __restrict__ L, int N, int kb, double* __restrict__ a) {
  const int nb = min(NB, N - kb);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= kb) return;
  double acc = 0.0;
  for (int l = 0; l < nb; ++l) acc += L[(size_t)(kb + l) * N + i] * a[kb + l];
  a[i] -= acc;
}

// ---- Lanczos building blocks
// v = K q, one warp per row (K symmetric, full storage).
__global__ void k_symv(const double* __restrict__ K, int N, const double* __restrict__ q,
                       double* __restrict__ v) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (warp >= N) return;
  const double* row = K + (size_t)warp * N;
  double acc = 0.0;
  for (int n = lane; n < N; n += 32) acc += row[n] * q[n];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) v[warp] = acc;
}

template <int THREADS>
__device__ double block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
#pragma unroll
  for (int s = THREADS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  return sh[0];
}

// out[blockIdx.x] = <Q[blockIdx.x], v>; with nq = 1 and Q = a this is a dot product.
__global__ void __launch_bounds__(512) k_rowdot(const double* __restrict__ Q, int N,
                                                const double* __restrict__ v, double* __restrict__ out) {
  __shared__ double sh[512];
  const double* q = Q + (size_t)blockIdx.x * N;
  double acc = 0.0;
  for (int n = threadIdx.x; n < N; n += 512) acc += q[n] * v[n];
  const double s = block_sum<512>(acc, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// v[n] -= sum_i Q[i][n] c[i]
__global__ void k_gemv_sub(const double* __restrict__ Q, int nq, int N, const double* __restrict__ c,
                           double* __restrict__ v) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  double acc = 0.0;
  for (int i = 0; i < nq; ++i) acc += Q[(size_t)i * N + n] * c[i];
  v[n] -= acc;
}

__global__ void k_scale_copy(const double* __restrict__ v, double inv, double* __restrict__ q, int N) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n < N) q[n] = v[n] * inv;
}

__global__ void k_restart_vec(uint32_t idx, int m, int N, double* __restrict__ v) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const uint4 o = bagel_philox4x32_10(make_uint4(idx, (uint32_t)(n >> 2), (uint32_t)m, 1u),
                                      0x4C4F5645u, 0u);
  v[n] = bagel_normal_d(o, n & 3);
}

// R_j = (q_j - le_j R_{j-1}) / ld_j, one thread per column n (coalesced over n).
__global__ void k_love_R(const double* __restrict__ Q, const double* __restrict__ ld,
                         const double* __restrict__ le, int k, int N, double* __restrict__ R) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  double prev = 0.0;
  for (int j = 0; j < k; ++j) {
    double v = Q[(size_t)j * N + n];
    if (j > 0) v -= le[j] * prev;
    v /= ld[j];
    R[(size_t)j * N + n] = v;
    prev = v;
  }
}

struct QScale {
  float q[BAGEL_MAX_D];
};

// V[n] = s [alpha_n | alpha_n X_n | R_{:,n}] (fp32), Xs[n][c] = X_nc KAPPA / l_c.
__global__ void k_pack(const float* __restrict__ X, const double* __restrict__ alpha,
                       const double* __restrict__ R, int N, int d, int k, double s, QScale qs,
                       int Cld, float* __restrict__ V, float* __restrict__ Xs) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  float* row = V + (size_t)n * Cld;
  const double a = alpha[n];
  row[0] = (float)(s * a);
  for (int c = 0; c < d; ++c) {
    const float x = X[(size_t)n * d + c];
    row[1 + c] = (float)(s * a * (double)x);
    Xs[(size_t)n * d + c] = x * qs.q[c];
  }
  for (int j = 0; j < k; ++j) row[1 + d + j] = (float)(s * R[(size_t)j * N + n]);
  for (int c = 1 + d + k; c < Cld; ++c) row[c] = 0.0f;
}

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace

int cb_build_khat(const float* X, int N, int d, const float* ell_host, double s, double noise,
                  double* K, cudaStream_t st) {
  EllD e{};
  for (int c = 0; c < d; ++c) e.inv_l2[c] = 1.0 / ((double)ell_host[c] * (double)ell_host[c]);
  dim3 grid(cdiv(N, 256), N < 65535 ? N : 65535);
  k_khat<<<grid, 256, 0, st>>>(X, N, d, e, s, noise, K);
  return 1;
}

// Blocked right-looking Cholesky with deferred trailing updates: super-panels of NB2 = 256 columns are
// factored block by block (NB = 64: diagonal block, panel solve over all rows below, update of the
// super-panel's remaining columns only); the trailing matrix right of the super-panel is updated
// once per super-panel with K = 256, so it is streamed N / 256 instead of N / 64 times.
constexpr int NB2 = 256;
int cb_cholesky(double* K, int N, int* pivot_flag, cudaStream_t st) {
  int launches = 0;
  for (int KB = 0; KB < N; KB += NB2) {
    const int pe = (N - KB < NB2) ? N : KB + NB2;
    for (int kb = KB; kb < pe; kb += NB) {
      const int nb = (N - kb < NB) ? N - kb : NB;
      k_potrf_diag<<<1, 256, 0, st>>>(K, N, kb, pivot_flag);
      ++launches;
      const int rem = N - kb - nb;
      if (rem > 0) {
        k_trsm_panel<<<cdiv(rem, TR), TR, 0, st>>>(K, N, kb, pivot_flag);
        ++launches;
        const int base = kb + nb;
        if (base < pe) {  // the super-panel's remaining columns, all rows below
          k_syrk<<<dim3(cdiv(pe - base, ST), cdiv(N - base, ST)), 256, 0, st>>>(K, N, kb, nb, base, pe, pivot_flag);
          ++launches;
        }
      }
    }
    if (pe < N) {  // everything right of the super-panel, K = its width
      k_syrk<<<dim3(cdiv(N - pe, ST), cdiv(N - pe, ST)), 256, 0, st>>>(K, N, KB, pe - KB, pe, N, pivot_flag);
      ++launches;
    }
  }
  return launches;
}

int cb_cholesky_solve(const double* L, int N, const float* y, int ystride, double* alpha,
                      double* tmp, cudaStream_t st) {
  int launches = 1;
  k_widen_col<<<cdiv(N, 256), 256, 0, st>>>(y, ystride, N, alpha);
  for (int kb = 0; kb < N; kb += NB) {
    k_trsv_diag_fwd<<<1, 64, 0, st>>>(L, N, kb, alpha);
    const int nb = (N - kb < NB) ? N - kb : NB;
    const int rem = N - kb - nb;
    launches++;
    if (rem > 0) {
      k_gemv_fwd<<<cdiv((long long)rem * 32, 256), 256, 0, st>>>(L, N, kb, alpha);
      launches++;
    }
  }
  const int last = ((N - 1) / NB) * NB;
  for (int kb = last; kb >= 0; kb -= NB) {
    k_trsv_diag_bwd<<<1, 64, 0, st>>>(L, N, kb, alpha);
    launches++;
    if (kb > 0) {
      k_gemv_bwd<<<cdiv(kb, 256), 256, 0, st>>>(L, N, kb, alpha);
      launches++;
    }
  }
  (void)tmp;
  return launches;
}

int cb_symv(const double* K, int N, const double* q, double* v, cudaStream_t st) {
  k_symv<<<cdiv((long long)N * 32, 256), 256, 0, st>>>(K, N, q, v);
  return 1;
}

int cb_dot(const double* a, const double* b, int N, double* out, cudaStream_t st) {
  k_rowdot<<<1, 512, 0, st>>>(a, N, b, out);
  return 1;
}

int cb_gemv_t(const double* Q, int nq, int N, const double* v, double* c, cudaStream_t st) {
  k_rowdot<<<nq, 512, 0, st>>>(Q, N, v, c);
  return 1;
}

int cb_gemv_sub(const double* Q, int nq, int N, const double* c, double* v, cudaStream_t st) {
  k_gemv_sub<<<cdiv(N, 256), 256, 0, st>>>(Q, nq, N, c, v);
  return 1;
}

int cb_scale_copy(const double* v, double scale_inv, double* q, int N, cudaStream_t st) {
  k_scale_copy<<<cdiv(N, 256), 256, 0, st>>>(v, scale_inv, q, N);
  return 1;
}

int cb_probe_from_y(const float* Y, int ystride, int N, double* v, cudaStream_t st) {
  k_widen_col<<<cdiv(N, 256), 256, 0, st>>>(Y, ystride, N, v);
  return 1;
}

int cb_restart_vector(uint32_t restart_idx, int m, int N, double* v, cudaStream_t st) {
  k_restart_vec<<<cdiv(N, 256), 256, 0, st>>>(restart_idx, m, N, v);
  return 1;
}

int cb_love_R(const double* Q, const double* ld, const double* le, int k, int N, double* R,
              cudaStream_t st) {
  k_love_R<<<cdiv(N, 256), 256, 0, st>>>(Q, ld, le, k, N, R);
  return 1;
}

int cb_pack(const float* X, const double* alpha, const double* R, int N, int d, int k, float s,
            const float* qscale_host, int Cld, float* V, float* Xs, cudaStream_t st) {
  QScale qs{};
  for (int c = 0; c < d; ++c) qs.q[c] = qscale_host[c];
  k_pack<<<cdiv(N, 128), 128, 0, st>>>(X, alpha, R, N, d, k, (double)s, qs, Cld, V, Xs);
  return 1;
}
