// gp_step.cu -- one batched GP query of the rollout (north star item (2)),
// v0 CUDA-core (FFMA) implementation; the correctness anchor for the tcgen05
// version.  For a batch of query points x* (B x d) and every output m:
//
//   pass 1   [mu | sum_n k a X_c | z] = ktilde(x*, X) . V_m        (Eq.2; LOVE z = R k)
//            V_m = s_m [alpha | alpha o X | R^T]  (N x (1+d+k)), ktilde in (0,1]
//            generated on the fly from exp2(-||x_hat - X_hat||^2), never stored.
//   reduce 1 v = s - ||z||^2 (LOVE Eq.3), sigma, J^mu_c = (sum k a X_c - x*_c mu) / l_c^2
//   pass 2   w = R^T z on the fly, sum_n w_n k_n [1 | X_n]            (autodiff of Eq.3)
//            -> J^v_c = (2 / l_c^2) sum_n w k (x*_c - X_nc)  (difference form; finished by the caller)
//
// The contraction over N is split S ways for parallelism; partial sums are
// reduced in a fixed order (deterministic).  Dominant work: 2 p N (1+d+k) +
// 2 p N k flops per query; these kernels are FP32-FFMA bound.
#include "bagel_internal.h"

namespace {

constexpr int P1_BM = 128, P1_BC = 64, P1_BN = 32, P1_THREADS = 128;
constexpr int P2_BM = 64, P2_BN = 64, P2_JC = 32, P2_THREADS = 128;
constexpr int P2_LD = 1 + BAGEL_MAX_D;  // partial per (split, m, row): [sum wk, sum wk X_0..X_{d-1}]

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

template <int D>
__global__ void __launch_bounds__(P1_THREADS) k_pass1(GpDesc g, const float* __restrict__ xstar, int B,
                                                      const float* __restrict__ Xs,
                                                      const float* __restrict__ V, int n_per_split,
                                                      float* __restrict__ P1) {
  __shared__ float xq[D][P1_BM];
  __shared__ __align__(16) float Ks[P1_BN][P1_BM];
  __shared__ __align__(16) float Vs[P1_BN][P1_BC];
  __shared__ float Xt[P1_BN][D];

  const int tid = threadIdx.x;
  const int row0 = blockIdx.x * P1_BM, col0 = blockIdx.y * P1_BC;
  const int m = blockIdx.z % g.p, split = blockIdx.z / g.p;
  const int n_begin = split * n_per_split;
  const int n_end = min(g.N, n_begin + n_per_split);

  for (int r = tid; r < P1_BM; r += P1_THREADS) {
    const int row = row0 + r;
#pragma unroll
    for (int c = 0; c < D; ++c) xq[c][r] = row < B ? xstar[(size_t)row * D + c] : 0.0f;
  }
  const int ty = tid / 8, tx = tid % 8;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;

  const float* Vm = V + (size_t)m * g.N * g.Cld;
  const float* Xm = Xs;  // raw X (N x D): differences first, then the per-dimension scale
  for (int n0 = n_begin; n0 < n_end; n0 += P1_BN) {
    __syncthreads();
    for (int i = tid; i < P1_BN * P1_BC / 4; i += P1_THREADS) {
      const int nn = i / (P1_BC / 4), cc = (i % (P1_BC / 4)) * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (n0 + nn < n_end) v = *reinterpret_cast<const float4*>(Vm + (size_t)(n0 + nn) * g.Cld + col0 + cc);
      *reinterpret_cast<float4*>(&Vs[nn][cc]) = v;
    }
    for (int i = tid; i < P1_BN * D; i += P1_THREADS) {
      const int nn = i / D, c = i % D;
      Xt[nn][c] = (n0 + nn < n_end) ? Xm[(size_t)(n0 + nn) * D + c] : 1e18f;
    }
    __syncthreads();
    for (int i = tid; i < P1_BN * P1_BM; i += P1_THREADS) {
      const int nn = i / P1_BM, r = i % P1_BM;
      float q = 0.0f;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const float df = (xq[c][r] - Xt[nn][c]) * g.qscale[m][c];
        q = fmaf(df, df, q);
      }
      Ks[nn][r] = exp2f(-q);
    }
    __syncthreads();
#pragma unroll 4
    for (int nn = 0; nn < P1_BN; ++nn) {
      const float4 a0 = *reinterpret_cast<const float4*>(&Ks[nn][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&Ks[nn][ty * 8 + 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Vs[nn][tx * 8]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Vs[nn][tx * 8 + 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
  }
  float* out = P1 + (size_t)(split * g.p + m) * B * g.Cld;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = row0 + ty * 8 + i;
    if (row < B) {
      float* o = out + (size_t)row * g.Cld + col0 + tx * 8;
      *reinterpret_cast<float4*>(o) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
      *reinterpret_cast<float4*>(o + 4) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    }
  }
}

// Sum pass-1 partials; LOVE variance in float64 accumulation of z^2; J^mu.
template <int D>
__global__ void __launch_bounds__(128) k_reduce1(GpDesc g, const float* __restrict__ xstar, int B, int S1,
                                                 const float* __restrict__ P1, float* __restrict__ Z,
                                                 float* __restrict__ mu_out, float* __restrict__ var_out,
                                                 float* __restrict__ jmu_out, float* __restrict__ sig_out) {
  const int b = blockIdx.x, m = blockIdx.y, tid = threadIdx.x;
  __shared__ float head[1 + BAGEL_MAX_D];
  __shared__ double red[128];
  double zz = 0.0;
  for (int c = tid; c < g.C; c += 128) {
    float v = 0.0f;
    for (int s = 0; s < S1; ++s) v += P1[((size_t)(s * g.p + m) * B + b) * g.Cld + c];
    if (c <= D) {
      head[c] = v;
    } else {
      Z[((size_t)m * B + b) * g.k + (c - 1 - D)] = v;
      zz += (double)v * (double)v;
    }
  }
  red[tid] = zz;
  __syncthreads();
  for (int s = 64; s > 0; s >>= 1) {
    if (tid < s) red[tid] += red[tid + s];
    __syncthreads();
  }
  if (tid == 0) {
    const float v = (float)((double)g.s[m] - red[0]);
    const float vh = fmaxf(v, BAGEL_VAR_FLOOR);
    const float sg = sqrtf(vh);
    mu_out[(size_t)m * B + b] = head[0];
    var_out[(size_t)m * B + b] = v;
    if (sig_out) sig_out[(size_t)b * g.p + m] = v > BAGEL_VAR_FLOOR ? sg : -sg;
  }
  if (tid < D && jmu_out) {
    const float xs = xstar[(size_t)b * D + tid];
    jmu_out[((size_t)b * g.p + m) * D + tid] = (head[1 + tid] - xs * head[0]) * g.ell2inv[m][tid];
  }
}

template <int D>
__global__ void __launch_bounds__(P2_THREADS) k_pass2(GpDesc g, const float* __restrict__ xstar, int B,
                                                      const float* __restrict__ X,
                                                      const float* __restrict__ Xs,
                                                      const float* __restrict__ V,
                                                      const float* __restrict__ Z, int n_per_split,
                                                      float* __restrict__ P2) {
  extern __shared__ __align__(16) float smem[];
  float* Zt = smem;                          // k x P2_BM  (z transposed: Zt[j][r])
  float* Rt = Zt + (size_t)g.k * P2_BM;      // P2_JC x (P2_BN + 1)
  float* xq = Rt + P2_JC * (P2_BN + 1);      // D x P2_BM
  float* Xt = xq + D * P2_BM;                // P2_BN x D (scaled)
  float* Xr = Xt + P2_BN * D;                // P2_BN x D (raw)
  constexpr int RLD = P2_BN + 1;

  const int tid = threadIdx.x;
  const int row0 = blockIdx.x * P2_BM, m = blockIdx.y, split = blockIdx.z;
  const int n_begin = split * n_per_split;
  const int n_end = min(g.N, n_begin + n_per_split);
  const int k = g.k;

  for (int i = tid; i < k * P2_BM; i += P2_THREADS) {
    const int r = i / k, j = i % k;  // coalesced over j
    const int row = row0 + r;
    Zt[(size_t)j * P2_BM + r] = row < B ? Z[((size_t)m * B + row) * k + j] : 0.0f;
  }
  for (int r = tid; r < P2_BM; r += P2_THREADS) {
    const int row = row0 + r;
#pragma unroll
    for (int c = 0; c < D; ++c) xq[c * P2_BM + r] = row < B ? xstar[(size_t)row * D + c] : 0.0f;
  }
  const int ty = tid / 16, tx = tid % 16;  // rows ty*8..+8, n = tx*4..+4
  float acc[8][1 + D];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int c = 0; c <= D; ++c) acc[i][c] = 0.0f;

  const float* Vm = V + (size_t)m * g.N * g.Cld + 1 + D;  // R^T columns
  const float* Xm = Xs + (size_t)m * g.N * D;
  for (int n0 = n_begin; n0 < n_end; n0 += P2_BN) {
    __syncthreads();
    for (int i = tid; i < P2_BN * D; i += P2_THREADS) {
      const int nn = i / D, c = i % D;
      const bool ok = n0 + nn < n_end;
      Xt[nn * D + c] = ok ? Xm[(size_t)(n0 + nn) * D + c] : 0.0f;
      Xr[nn * D + c] = ok ? X[(size_t)(n0 + nn) * D + c] : 0.0f;
    }
    float w[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) w[i][e] = 0.0f;
    for (int j0 = 0; j0 < k; j0 += P2_JC) {
      __syncthreads();
      for (int i = tid; i < P2_BN * P2_JC; i += P2_THREADS) {
        const int nn = i / P2_JC, jj = i % P2_JC;
        float v = 0.0f;
        if (n0 + nn < n_end && j0 + jj < k) v = Vm[(size_t)(n0 + nn) * g.Cld + j0 + jj];
        Rt[jj * RLD + nn] = v;
      }
      __syncthreads();
      const int jn = min(P2_JC, k - j0);
      for (int jj = 0; jj < jn; ++jj) {
        const float4 a0 = *reinterpret_cast<const float4*>(&Zt[(size_t)(j0 + jj) * P2_BM + ty * 8]);
        const float4 a1 = *reinterpret_cast<const float4*>(&Zt[(size_t)(j0 + jj) * P2_BM + ty * 8 + 4]);
        const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        float bb[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) bb[e] = Rt[jj * RLD + tx * 4 + e];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int e = 0; e < 4; ++e) w[i][e] = fmaf(a[i], bb[e], w[i][e]);
      }
    }
    // (s w_n) * ktilde_n accumulated against [1 | X_n]
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int nn = tx * 4 + e;
      if (n0 + nn >= n_end) continue;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = ty * 8 + i;
        float q = 0.0f, dx[D];
#pragma unroll
        for (int c = 0; c < D; ++c) {
          dx[c] = xq[c * P2_BM + r] - Xr[nn * D + c];
          const float df = dx[c] * g.qscale[m][c];
          q = fmaf(df, df, q);
        }
        const float t = w[i][e] * exp2f(-q);
        acc[i][0] += t;
        // difference form: sum_n (s w_n k_n) (x*_c - X_nc)
#pragma unroll
        for (int c = 0; c < D; ++c) acc[i][1 + c] = fmaf(t, dx[c], acc[i][1 + c]);
      }
    }
  }
  // reduce over the 16 tx lanes sharing a row (half-warp), fixed xor-tree order
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int c = 0; c <= D; ++c) {
      float v = acc[i][c];
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      acc[i][c] = v;
    }
  if (tx == 0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = row0 + ty * 8 + i;
      if (row < B) {
        float* o = P2 + ((size_t)(split * g.p + m) * B + row) * P2_LD;
#pragma unroll
        for (int c = 0; c <= D; ++c) o[c] = acc[i][c];
      }
    }
  }
}

template <int D>
__global__ void k_finish_predict(GpDesc g, const float* __restrict__ xstar, int B, int S2,
                                 const float* __restrict__ P2, const float* __restrict__ mu,
                                 const float* __restrict__ var, float* __restrict__ mean_out,
                                 float* __restrict__ var_out, float* __restrict__ dvar) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * g.p) return;
  const int b = idx / g.p, m = idx % g.p;
  float sums[1 + D];
#pragma unroll
  for (int c = 0; c <= D; ++c) sums[c] = 0.0f;
  for (int s = 0; s < S2; ++s) {
    const float* src = P2 + ((size_t)(s * g.p + m) * B + b) * P2_LD;
#pragma unroll
    for (int c = 0; c <= D; ++c) sums[c] += src[c];
  }
  if (mean_out) mean_out[idx] = mu[(size_t)m * B + b];
  if (var_out) var_out[idx] = var[(size_t)m * B + b];
  if (dvar) {
#pragma unroll
    for (int c = 0; c < D; ++c)
      dvar[(size_t)idx * D + c] =
          2.0f * g.ell2inv[m][c] * sums[1 + c];  // sums[1 + c] = sum_n w_n k_n (x*_c - X_nc)
  }
}

}  // namespace

void gs_choose_splits(const bagel_ctx* c, int B, int* S1, int* S2) {
  const int target = 3 * c->num_sms;  // >= ~3 waves of CTAs
  const int tiles1 = cdiv(B, P1_BM) * cdiv(c->gp.C, P1_BC) * c->gp.p;
  const int max1 = cdiv(c->gp.N, 4 * P1_BN);  // keep >= 4 n-tiles per split
  int s1 = cdiv(target, tiles1);
  *S1 = s1 < 1 ? 1 : (s1 > max1 ? max1 : s1);
  const int tiles2 = cdiv(B, P2_BM) * c->gp.p;
  const int max2 = cdiv(c->gp.N, 2 * P2_BN);
  int s2 = cdiv(target, tiles2);
  *S2 = s2 < 1 ? 1 : (s2 > max2 ? max2 : s2);
}

#define DISPATCH_D(dv, ...)                            \
  switch (dv) {                                        \
    case 2: { constexpr int D = 2; __VA_ARGS__; break; } \
    case 3: { constexpr int D = 3; __VA_ARGS__; break; } \
    case 4: { constexpr int D = 4; __VA_ARGS__; break; } \
    case 5: { constexpr int D = 5; __VA_ARGS__; break; } \
    case 6: { constexpr int D = 6; __VA_ARGS__; break; } \
    case 7: { constexpr int D = 7; __VA_ARGS__; break; } \
    case 8: { constexpr int D = 8; __VA_ARGS__; break; } \
    default: break;                                    \
  }

int gs_pass1(const bagel_ctx* c, const float* xstar, int B, cudaStream_t st) {
  const int S1 = c->ws.S1;
  const int nps = cdiv(cdiv(c->gp.N, S1), P1_BN) * P1_BN;
  dim3 grid(cdiv(B, P1_BM), cdiv(c->gp.C, P1_BC), c->gp.p * S1);
  DISPATCH_D(c->gp.d, (k_pass1<D><<<grid, P1_THREADS, 0, st>>>(c->gp, xstar, B, c->X, c->V, nps, c->ws.P1)));
  return 1;
}

int gs_reduce1(const bagel_ctx* c, const float* xstar, int B, float* jmu_out, float* sig_out,
               cudaStream_t st) {
  dim3 grid(B, c->gp.p);
  DISPATCH_D(c->gp.d, (k_reduce1<D><<<grid, 128, 0, st>>>(c->gp, xstar, B, c->ws.S1, c->ws.P1, c->ws.Z,
                                                          c->ws.mu, c->ws.var, jmu_out, sig_out)));
  return 1;
}

size_t gs_pass2_smem(int k, int d) {
  return sizeof(float) * ((size_t)k * P2_BM + P2_JC * (P2_BN + 1) + d * P2_BM + 2 * P2_BN * d);
}

int gs_pass2(const bagel_ctx* c, const float* xstar, int B, cudaStream_t st) {
  const int S2 = c->ws.S2;
  const int nps = cdiv(cdiv(c->gp.N, S2), P2_BN) * P2_BN;
  dim3 grid(cdiv(B, P2_BM), c->gp.p, S2);
  const size_t smem = gs_pass2_smem(c->gp.k, c->gp.d);
  DISPATCH_D(c->gp.d, ({
    static std::atomic<unsigned long long> devices{0};  // the opt-in is per device
    if (bagel_first_on_device(devices)) bagel_set_smem_attr(k_pass2<D>, 200 * 1024);
    k_pass2<D><<<grid, P2_THREADS, smem, st>>>(c->gp, xstar, B, c->X, c->Xs, c->V, c->ws.Z, nps, c->ws.P2);
  }));
  return 1;
}

int gs_finish_predict(const bagel_ctx* c, const float* xstar, int B, float* mean, float* var,
                      float* dmean, float* dvar, cudaStream_t st) {
  (void)dmean;  // written by gs_reduce1
  DISPATCH_D(c->gp.d, (k_finish_predict<D><<<cdiv(B * c->gp.p, 128), 128, 0, st>>>(
                          c->gp, xstar, B, c->ws.S2eff, c->ws.P2, c->ws.mu, c->ws.var, mean, var, dvar)));
  return 1;
}
