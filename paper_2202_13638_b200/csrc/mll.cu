// mll.cu -- "Learn GP transition dynamics using D" (Alg.1): the exact log marginal
// likelihood of one output GP and its gradient in the log-hyperparameters (Eq.5-6, P:77-80;
// SURVEY.md §8(f) NEXT-1), in float64 on the GPU:
//   Khat = K(X, X) + sigma_n^2 I,  L = chol(Khat),  alpha = Khat^-1 y
//   log p(y | X, phi) = -1/2 y^T alpha - sum_i log L_ii - N/2 log(2 pi)          (Eq.5, reading R33)
//   d/d phi_j        = 1/2 tr((alpha alpha^T - Khat^-1) dKhat/dphi_j)            (Eq.6, reading R33)
// with phi = [log l_1 .. log l_d, log s, log sigma_n^2] (log-parameters):
//   dK_ij / dlog l_c = K_ij (x_ic - x_jc)^2 / l_c^2,  dK_ij / dlog s = K_ij,  dKhat / dlog sn2 = sn2 I.
// Khat^-1 = L^-T L^-1 is never stored: the gradient kernel forms each 64 x 64 tile of it from the
// triangular inverse Linv = L^-1 (blocked, below) and reduces it against alpha alpha^T and the
// regenerated kernel tile in its epilogue.  All reductions run in a fixed order (deterministic).
// Roofline: fp64 FMA bound -- Cholesky N^3/3, triangular inverse N^3/3, Khat^-1 tiles N^3/3 flops.
#include <math.h>

#include <algorithm>

#include "bagel_internal.h"

namespace {

constexpr int TB = 64;  // tile / block size (matches the Cholesky block of cache_build.cu)

struct Hyp64 {
  double inv_l2[BAGEL_MAX_D];
  double s, noise;
};

__global__ void k_khat64(const float* __restrict__ X, int N, int d, Hyp64 h, double* __restrict__ K) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  for (int i = blockIdx.y; i < N; i += gridDim.y) {  // grid.y is capped at 65535 rows per pass
    double q = 0.0;
    for (int c = 0; c < d; ++c) {
      const double df = (double)X[(size_t)i * d + c] - (double)X[(size_t)j * d + c];
      q += df * df * h.inv_l2[c];
    }
    double v = h.s * exp(-0.5 * q);
    if (i == j) v += h.noise;
    K[(size_t)i * N + j] = v;
  }
}

// out[0] = sum_i log L_ii, out[1] = y^T alpha (one CTA, fixed order)
__global__ void __launch_bounds__(256) k_mll_scalars(const double* __restrict__ L, int N, const float* __restrict__ y,
                                                     int ystride, const double* __restrict__ alpha,
                                                     double* __restrict__ out) {
  __shared__ double r0[256], r1[256];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < N; i += 256) {
    a += log(L[(size_t)i * N + i]);
    b += (double)y[(size_t)i * ystride] * alpha[i];
  }
  r0[threadIdx.x] = a;
  r1[threadIdx.x] = b;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      r0[threadIdx.x] += r0[threadIdx.x + o];
      r1[threadIdx.x] += r1[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = r0[0];
    out[1] = r1[0];
  }
}

// Diagonal blocks of Linv: Linv_II = L_II^-1 (thread c solves L_II x = e_c by forward substitution;
// its column lives in Li itself: every element is written and re-read by the same thread).
__global__ void __launch_bounds__(TB) k_trtri_diag(const double* __restrict__ L, int N, double* __restrict__ Li) {
  __shared__ double Ls[TB][TB + 1];
  const int i0 = blockIdx.x * TB, nb = min(TB, N - i0), c = threadIdx.x;
  for (int r = 0; r < nb; ++r)
    if (c < nb) Ls[r][c] = L[(size_t)(i0 + r) * N + i0 + c];
  __syncthreads();
  if (c < nb) {
    double* col = Li + (size_t)i0 * N + i0 + c;
    for (int r = 0; r < nb; ++r) {
      double acc = (r == c) ? 1.0 : 0.0;
      for (int k = c; k < r; ++k) acc -= Ls[r][k] * col[(size_t)k * N];
      col[(size_t)r * N] = r < c ? 0.0 : acc / Ls[r][r];
    }
  }
}

// acc[u][v] += sum_l A(l, ty + 16u) B(l, tx + 16v) over one 16-deep chunk staged in shared memory
__device__ __forceinline__ void mma16(const double (&As)[16][TB], const double (&Bs)[16][TB], int tx, int ty,
                                      double (&acc)[4][4]) {
#pragma unroll
  for (int l = 0; l < 16; ++l) {
    double a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = As[l][ty + 16 * u];
      b[u] = Bs[l][tx + 16 * u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
  }
}

// Off-diagonal blocks of block row I (all J < I in parallel, one CTA each):
//   Linv_IJ = -Linv_II sum_{K=J}^{I-1} L_IK Linv_KJ   (block rows < I are final)
__global__ void __launch_bounds__(256) k_trtri_row(const double* __restrict__ L, int N, int I,
                                                   double* __restrict__ Li) {
  const int J = blockIdx.x;
  const int i0 = I * TB, j0 = J * TB;
  const int ni = min(TB, N - i0);
  __shared__ double As[16][TB];
  __shared__ double Bs[16][TB];
  __shared__ double Ts[TB][TB];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[4][4] = {};
  for (int K = J; K < I; ++K) {
    const int k0 = K * TB;
    for (int l0 = 0; l0 < TB; l0 += 16) {
      for (int idx = threadIdx.x; idx < 16 * TB; idx += 256) {
        const int r = idx / 16, l = idx % 16;  // A(l, r) = L[i0 + r][k0 + l0 + l]
        As[l][r] = (r < ni) ? L[(size_t)(i0 + r) * N + k0 + l0 + l] : 0.0;
        const int lb = idx / TB, cb = idx % TB;  // B(l, c) = Linv[k0 + l0 + l][j0 + c]
        Bs[lb][cb] = Li[(size_t)(k0 + l0 + lb) * N + j0 + cb];
      }
      __syncthreads();
      mma16(As, Bs, tx, ty, acc);
      __syncthreads();
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) Ts[ty + 16 * u][tx + 16 * v] = acc[u][v];
  __syncthreads();
  double out[4][4] = {};
  for (int l0 = 0; l0 < ni; l0 += 16) {
    for (int idx = threadIdx.x; idx < 16 * TB; idx += 256) {
      const int r = idx / 16, l = idx % 16;  // A(l, r) = Linv_II[r][l0 + l]
      As[l][r] = (r < ni && l0 + l < ni) ? Li[(size_t)(i0 + r) * N + i0 + l0 + l] : 0.0;
      const int lb = idx / TB, cb = idx % TB;  // B(l, c) = T[l0 + l][c]
      Bs[lb][cb] = (l0 + lb < ni) ? Ts[l0 + lb][cb] : 0.0;
    }
    __syncthreads();
    mma16(As, Bs, tx, ty, out);
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int r = ty + 16 * u;
      if (r < ni) Li[(size_t)(i0 + r) * N + j0 + tx + 16 * v] = -out[u][v];
    }
}

// Gradient tiles: CTA (I >= J) forms Kinv_IJ = sum_{K >= I} Linv_KI^T Linv_KJ, then reduces
// W = alpha alpha^T - Kinv against the regenerated K tile:
//   part[0..d-1] += w K r_c^2 / l_c^2,  part[d] += w K,  part[d+1] += W_ii (diagonal tiles),
// w = W_ij, counted twice for I > J (symmetry).  Per-CTA partials, fixed order.
constexpr int NPART = BAGEL_MAX_D + 2;
__global__ void __launch_bounds__(256) k_grad_tiles(const double* __restrict__ Li, int N, int d,
                                                    const float* __restrict__ X, const double* __restrict__ alpha,
                                                    Hyp64 h, double* __restrict__ part) {
  // triangular tile index -> (I, J), I >= J
  const int t = blockIdx.x;
  int I = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((I + 1) * (I + 2) / 2 <= t) ++I;
  while (I * (I + 1) / 2 > t) --I;
  const int J = t - I * (I + 1) / 2;
  const int nbk = (N + TB - 1) / TB;
  const int i0 = I * TB, j0 = J * TB;
  __shared__ double As[16][TB];
  __shared__ double Bs[16][TB];
  __shared__ double red[256];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[4][4] = {};
  for (int K = I; K < nbk; ++K) {
    const int k0 = K * TB;
    for (int l0 = 0; l0 < TB; l0 += 16) {
      for (int idx = threadIdx.x; idx < 16 * TB; idx += 256) {
        const int l = idx / TB, c = idx % TB;
        const int k = k0 + l0 + l;
        As[l][c] = (k < N && i0 + c < N) ? Li[(size_t)k * N + i0 + c] : 0.0;
        Bs[l][c] = (k < N && j0 + c < N) ? Li[(size_t)k * N + j0 + c] : 0.0;
      }
      __syncthreads();
      mma16(As, Bs, tx, ty, acc);
      __syncthreads();
    }
  }
  const double wsym = (I == J) ? 1.0 : 2.0;
  double p[NPART];
#pragma unroll
  for (int c = 0; c < NPART; ++c) p[c] = 0.0;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int i = i0 + ty + 16 * u, j = j0 + tx + 16 * v;
      if (i < N && j < N) {
        const double W = alpha[i] * alpha[j] - acc[u][v];
        double q = 0.0, r2[BAGEL_MAX_D];
#pragma unroll
        for (int c = 0; c < BAGEL_MAX_D; ++c) {
          r2[c] = 0.0;
          if (c < d) {
            const double df = (double)X[(size_t)i * d + c] - (double)X[(size_t)j * d + c];
            r2[c] = df * df * h.inv_l2[c];
            q += r2[c];
          }
        }
        const double wk = wsym * W * h.s * exp(-0.5 * q);
#pragma unroll
        for (int c = 0; c < BAGEL_MAX_D; ++c) p[c] += wk * r2[c];
        p[BAGEL_MAX_D] += wk;
        if (i == j) p[BAGEL_MAX_D + 1] += W;
      }
    }
  for (int c = 0; c < NPART; ++c) {
    if (c >= d && c < BAGEL_MAX_D) continue;
    red[threadIdx.x] = p[c];
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) part[(size_t)t * NPART + c] = red[0];
    __syncthreads();
  }
}

// grad[c] = 1/2 sum_t part[t][c] (c < d: log l_c; d: log s), grad[d+1] = 1/2 sn2 sum_t part[t][diag]
__global__ void __launch_bounds__(256) k_grad_final(const double* __restrict__ part, int ntiles, int d, double noise,
                                                    double* __restrict__ grad) {
  __shared__ double red[256];
  for (int c = 0; c < d + 2; ++c) {
    const int src = c < d ? c : (c == d ? BAGEL_MAX_D : BAGEL_MAX_D + 1);
    double a = 0.0;
    for (int t = threadIdx.x; t < ntiles; t += 256) a += part[(size_t)t * NPART + src];
    red[threadIdx.x] = a;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) grad[c] = 0.5 * red[0] * (c == d + 1 ? noise : 1.0);
    __syncthreads();
  }
}

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace

// Exact-GP variance cache ("AutoDiff on exact GPs"): L = chol(Khat),
// alpha = Khat^-1 y, Li = L^-1, so that var = s - ||L^-1 k||^2 (Eq.3 exactly) is the LOVE query with
// R = L^-1 at rank N.  Hyperparameters as gp_load holds them (float, widened).
int exact_launch(const float* X, const float* Y, int ystride, int N, int d, const float* ell, float s, float noise,
                 double* K, double* Li, double* alpha, int* pivot_flag, cudaStream_t st) {
  Hyp64 h{};
  for (int c = 0; c < d; ++c) h.inv_l2[c] = 1.0 / ((double)ell[c] * (double)ell[c]);
  h.s = (double)s;
  h.noise = (double)noise;
  int launches = 0;
  k_khat64<<<dim3(cdiv(N, 256), std::min(N, 65535)), 256, 0, st>>>(X, N, d, h, K);
  ++launches;
  launches += cb_cholesky(K, N, pivot_flag, st);
  launches += cb_cholesky_solve(K, N, Y, ystride, alpha, nullptr, st);
  const int nb = cdiv(N, TB);
  cudaMemsetAsync(Li, 0, (size_t)N * N * sizeof(double), st);
  k_trtri_diag<<<nb, TB, 0, st>>>(K, N, Li);
  ++launches;
  for (int I = 1; I < nb; ++I) {
    k_trtri_row<<<I, 256, 0, st>>>(K, N, I, Li);
    ++launches;
  }
  return launches;
}

int mll_part_count(int N) {
  const int nb = cdiv(N, TB);
  return nb * (nb + 1) / 2 * NPART;
}

// K (N x N) receives L; Li (N x N) receives L^-1; alpha (N), sc (2), part (mll_part_count), grad (d + 2).
// log_hyp: d + 2 values [log l_c | log s | log sn2].  Returns launches; *pivot_flag > 0 on failure.
int mll_launch(const float* X, const float* Y, int ystride, int N, int d, const double* log_hyp, double* K,
               double* Li, double* alpha, double* sc, double* part, double* grad, int* pivot_flag, bool want_grad,
               cudaStream_t st) {
  Hyp64 h{};
  for (int c = 0; c < d; ++c) h.inv_l2[c] = exp(-2.0 * log_hyp[c]);
  h.s = exp(log_hyp[d]);
  h.noise = exp(log_hyp[d + 1]);
  int launches = 0;
  k_khat64<<<dim3(cdiv(N, 256), std::min(N, 65535)), 256, 0, st>>>(X, N, d, h, K);
  ++launches;
  launches += cb_cholesky(K, N, pivot_flag, st);
  launches += cb_cholesky_solve(K, N, Y, ystride, alpha, nullptr, st);
  k_mll_scalars<<<1, 256, 0, st>>>(K, N, Y, ystride, alpha, sc);
  ++launches;
  if (!want_grad) return launches;
  const int nb = cdiv(N, TB);
  cudaMemsetAsync(Li, 0, (size_t)N * N * sizeof(double), st);
  k_trtri_diag<<<nb, TB, 0, st>>>(K, N, Li);
  ++launches;
  for (int I = 1; I < nb; ++I) {
    k_trtri_row<<<I, 256, 0, st>>>(K, N, I, Li);
    ++launches;
  }
  const int ntiles = nb * (nb + 1) / 2;
  k_grad_tiles<<<ntiles, 256, 0, st>>>(Li, N, d, X, alpha, h, part);
  k_grad_final<<<1, 256, 0, st>>>(part, ntiles, d, h.noise, grad);
  return launches + 2;
}
