// rollout.cu -- everything of the rollout except the GP contraction:
//   init       G = r(x0, g) (Alg.1), tape x_0, policy u_0 = pi(x_0, g)
//   epilogue   per step: finish J^v, eps (Philox), x' = x + mu + sigma eps (Eq.9-10),
//              G += r(x', g), tape row (a8), next action u' = pi(x', g)
//   reverse    hand-written reverse mode over the tape, t = T-1..0 (SURVEY
//              Appendix B): MLP recomputed, theta-bar accumulated per CTA in smem
//   reduce     fixed-order sum of the per-CTA theta-bar partials and of the returns
//              (L = -(1/B_global) sum_b G_b)
// The policy is the tanh MLP of P:149 (hidden and output tanh, reading R13);
// phi = [x, g] or [x, g, g - x] (R14).  These kernels are latency / L2 bound
// (|theta| and the tape are small); no tensor-core work here in v0.
#include "bagel_internal.h"
#include "philox.cuh"

namespace {

constexpr int EPI_ROWS = 32, EPI_THREADS = 256;
constexpr int REV_ROWS = 8, REV_THREADS = 256;
constexpr int P2_LD = 1 + BAGEL_MAX_D;

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

__device__ __forceinline__ float reward_fn(const RewardDesc& rw, const float* x, const float* g, int p) {
  float q = 0.0f;
  for (int c = 0; c < p; ++c) {
    const float df = x[c] - g[c];
    q = fmaf(rw.Q[c] * df, df, q);
  }
  return expf(-q * rw.inv_two_sr2);
}

// act: rows x act_total (smem).  Layer l activations start at aoff(l) = sum_{i<l} sizes[i].
__device__ __forceinline__ int act_off(const PolicyDesc& P, int l) {
  int o = 0;
  for (int i = 0; i < l; ++i) o += P.sizes[i];
  return o;
}

// h0 = phi(x, g) for `nrows` rows whose x and g are given (row-major B x p slices).
__device__ void phi_rows(const PolicyDesc& P, int p, const float* x, const float* g, int nrows,
                         int valid, float* act) {
  for (int idx = threadIdx.x; idx < nrows * P.sizes[0]; idx += blockDim.x) {
    const int r = idx / P.sizes[0], i = idx % P.sizes[0];
    float v = 0.0f;
    if (r < valid) {
      if (i < p) v = x[(size_t)r * p + i];
      else if (i < 2 * p) v = g[(size_t)r * p + i - p];
      else v = g[(size_t)r * p + i - 2 * p] - x[(size_t)r * p + i - 2 * p];
    }
    act[r * P.act_total + i] = v;
  }
}

// h_{l+1} = tanh(W_l h_l + b_l) for every layer (block-cooperative; act in smem).
__device__ void mlp_forward_rows(const PolicyDesc& P, const float* __restrict__ theta, int nrows, float* act) {
  int off_in = 0;
  for (int l = 0; l < P.n_layers; ++l) {
    const int in = P.sizes[l], out = P.sizes[l + 1];
    const int off_out = off_in + in;
    const float* W = theta + P.w_off[l];
    const float* bb = theta + P.b_off[l];
    __syncthreads();
    for (int idx = threadIdx.x; idx < nrows * out; idx += blockDim.x) {
      const int r = idx / out, o = idx % out;
      const float* h = act + r * P.act_total + off_in;
      const float* w = W + (size_t)o * in;
      float a = __ldg(bb + o);
      for (int i = 0; i < in; ++i) a = fmaf(__ldg(w + i), h[i], a);
      act[r * P.act_total + off_out + o] = tanhf(a);
    }
    off_in = off_out;
  }
  __syncthreads();
}

template <int D>
__device__ void write_xstar(const PolicyDesc& P, int p, const float* act, int nrows, int row0, int B,
                            float* __restrict__ xstar, const float* xrows) {
  const int uoff = act_off(P, P.n_layers);
  for (int idx = threadIdx.x; idx < nrows * D; idx += blockDim.x) {
    const int r = idx / D, c = idx % D;
    if (row0 + r >= B) continue;
    xstar[(size_t)(row0 + r) * D + c] = c < p ? xrows[(size_t)r * p + c] : act[r * P.act_total + uoff + c - p];
  }
}

template <int D>
__global__ void __launch_bounds__(EPI_THREADS) k_init(PolicyDesc P, RewardDesc rw, int p,
                                                      const float* __restrict__ theta,
                                                      const float* __restrict__ x0,
                                                      const float* __restrict__ goals, int B,
                                                      float* __restrict__ tape_x0, double* __restrict__ G,
                                                      float* __restrict__ xstar) {
  extern __shared__ float act[];
  const int row0 = blockIdx.x * EPI_ROWS;
  const int valid = min(EPI_ROWS, B - row0);
  for (int r = threadIdx.x; r < valid; r += blockDim.x) {
    const int b = row0 + r;
    G[b] = (double)reward_fn(rw, x0 + (size_t)b * p, goals + (size_t)b * p, p);
    for (int c = 0; c < p; ++c) tape_x0[(size_t)b * p + c] = x0[(size_t)b * p + c];
  }
  phi_rows(P, p, x0 + (size_t)row0 * p, goals + (size_t)row0 * p, EPI_ROWS, valid, act);
  mlp_forward_rows(P, theta, EPI_ROWS, act);
  write_xstar<D>(P, p, act, EPI_ROWS, row0, B, xstar, x0 + (size_t)row0 * p);
}

template <int D>
__global__ void __launch_bounds__(EPI_THREADS) k_epilogue(
    PolicyDesc P, RewardDesc rw, GpDesc g, const float* __restrict__ theta, const float* __restrict__ goals,
    int B, int t, int S2, const float* __restrict__ P2, const float* __restrict__ mu,
    const float* __restrict__ var, const float* __restrict__ tape_x_t, const float* __restrict__ sig_t,
    float* __restrict__ jv_t, float* __restrict__ tape_x_next, double* __restrict__ G,
    float* __restrict__ xstar, uint64_t seed, long long traj_offset, int policy_next,
    int* __restrict__ err_flag, float* __restrict__ trace_mu, float* __restrict__ trace_var) {
  extern __shared__ float act[];
  __shared__ float xn_s[EPI_ROWS * BAGEL_MAX_P];
  const int p = g.p;
  const int row0 = blockIdx.x * EPI_ROWS;
  const int valid = min(EPI_ROWS, B - row0);
  for (int r = threadIdx.x; r < valid; r += blockDim.x) {
    const int b = row0 + r;
    const float4 e4 = bagel_rollout_eps4(seed, (uint32_t)(traj_offset + b), (uint32_t)t);
    float xn[BAGEL_MAX_P];
    bool finite = true;
    for (int m = 0; m < p; ++m) {
      float sums[1 + D];
#pragma unroll
      for (int c = 0; c <= D; ++c) sums[c] = 0.0f;
      for (int s = 0; s < S2; ++s) {
        const float* src = P2 + ((size_t)(s * p + m) * B + b) * P2_LD;
#pragma unroll
        for (int c = 0; c <= D; ++c) sums[c] += src[c];
      }
      const float* xs = xstar + (size_t)b * D;
#pragma unroll
      for (int c = 0; c < D; ++c)
        jv_t[((size_t)b * p + m) * D + c] = 2.0f * g.ell2inv[m][c] * (xs[c] * sums[0] - sums[1 + c]);
      const float sg = fabsf(sig_t[(size_t)b * p + m]);
      const float mum = mu[(size_t)m * B + b];
      xn[m] = tape_x_t[(size_t)b * p + m] + mum + sg * bagel_f4get(e4, m & 3);
      finite = finite && isfinite(xn[m]);
      if (trace_mu) trace_mu[(size_t)b * p + m] = mum;
      if (trace_var) trace_var[(size_t)b * p + m] = var[(size_t)m * B + b];
    }
    if (!finite) atomicMin(err_flag, t * B + b);
    for (int m = 0; m < p; ++m) {
      tape_x_next[(size_t)b * p + m] = xn[m];
      xn_s[r * p + m] = xn[m];
    }
    G[b] += (double)reward_fn(rw, xn, goals + (size_t)b * p, p);
  }
  if (!policy_next) return;  // uniform
  __syncthreads();
  phi_rows(P, p, xn_s, goals + (size_t)row0 * p, EPI_ROWS, valid, act);
  mlp_forward_rows(P, theta, EPI_ROWS, act);
  write_xstar<D>(P, p, act, EPI_ROWS, row0, B, xstar, xn_s);
}

// ------------------------------------------------------------------ reverse
// smem: gacc[n_params] | act[REV_ROWS x act_total] | dl[2][REV_ROWS x max_width] | xbar | xsbar
template <int D>
__global__ void __launch_bounds__(REV_THREADS) k_reverse(
    PolicyDesc P, RewardDesc rw, int p, const float* __restrict__ theta, const float* __restrict__ goals,
    int B, int T, const float* __restrict__ tape_x, const float* __restrict__ tape_sig,
    const float* __restrict__ tape_jmu, const float* __restrict__ tape_jv, uint64_t seed,
    long long traj_offset, float invB, float* __restrict__ theta_part) {
  extern __shared__ float sm[];
  float* gacc = sm;
  float* act = gacc + ((P.n_params + 3) & ~3);
  float* dl0 = act + REV_ROWS * P.act_total;
  float* dl1 = dl0 + REV_ROWS * P.max_width;
  float* xbar = dl1 + REV_ROWS * P.max_width;  // REV_ROWS x p
  float* xsbar = xbar + REV_ROWS * BAGEL_MAX_P;  // REV_ROWS x D
  __shared__ float gs[REV_ROWS * BAGEL_MAX_P];

  const int tid = threadIdx.x;
  const int row0 = blockIdx.x * REV_ROWS;
  const int valid = min(REV_ROWS, B - row0);
  const float inv_sr2 = 2.0f * rw.inv_two_sr2;
  for (int i = tid; i < P.n_params; i += blockDim.x) gacc[i] = 0.0f;
  for (int i = tid; i < REV_ROWS * p; i += blockDim.x) {
    const int r = i / p, c = i % p;
    gs[i] = r < valid ? goals[(size_t)(row0 + r) * p + c] : 0.0f;
  }
  __syncthreads();
  // xbar_T = (1/B) r_T Q (x_T - g) / sigma_r^2
  if (tid < REV_ROWS) {
    const int r = tid;
    for (int c = 0; c < p; ++c) xbar[r * p + c] = 0.0f;
    if (r < valid) {
      const float* xT = tape_x + ((size_t)T * B + row0 + r) * p;
      const float rr = reward_fn(rw, xT, gs + r * p, p);
      for (int c = 0; c < p; ++c) xbar[r * p + c] = invB * rr * rw.Q[c] * (xT[c] - gs[r * p + c]) * inv_sr2;
    }
  }
  const int L = P.n_layers;
  const int uoff = act_off(P, L);
  for (int t = T - 1; t >= 0; --t) {
    __syncthreads();
    const float* xt = tape_x + ((size_t)t * B + row0) * p;
    // xs_bar = sum_m xbar_m (Jmu_m + [v > floor] eps_m / (2 sigma_m) Jv_m)
    if (tid < REV_ROWS) {
      const int r = tid;
      for (int c = 0; c < D; ++c) xsbar[r * D + c] = 0.0f;
      if (r < valid) {
        const int b = row0 + r;
        const float4 e4 = bagel_rollout_eps4(seed, (uint32_t)(traj_offset + b), (uint32_t)t);
        for (int m = 0; m < p; ++m) {
          const float sg = tape_sig[((size_t)t * B + b) * p + m];
          const float f = sg > 0.0f ? bagel_f4get(e4, m & 3) / (2.0f * sg) : 0.0f;
          const float* jm = tape_jmu + (((size_t)t * B + b) * p + m) * D;
          const float* jv = tape_jv + (((size_t)t * B + b) * p + m) * D;
          const float xb = xbar[r * p + m];
#pragma unroll
          for (int c = 0; c < D; ++c) xsbar[r * D + c] = fmaf(xb, jm[c] + f * jv[c], xsbar[r * D + c]);
        }
      }
    }
    phi_rows(P, p, xt, gs, REV_ROWS, valid, act);
    mlp_forward_rows(P, theta, REV_ROWS, act);  // ends with __syncthreads
    // delta_L = ubar (1 - u^2)
    {
      const int q = P.sizes[L];
      for (int idx = tid; idx < REV_ROWS * q; idx += blockDim.x) {
        const int r = idx / q, o = idx % q;
        const float u = act[r * P.act_total + uoff + o];
        dl0[r * P.max_width + o] = r < valid ? xsbar[r * D + p + o] * (1.0f - u * u) : 0.0f;
      }
    }
    float* dcur = dl0;
    float* dprev = dl1;
    int off_in = uoff;
    for (int l = L - 1; l >= 0; --l) {
      __syncthreads();
      const int in = P.sizes[l], out = P.sizes[l + 1];
      off_in -= in;
      const float* W = theta + P.w_off[l];
      // theta-bar: W_l[o][i] += sum_r delta[r][o] h_l[r][i];  b_l[o] += sum_r delta[r][o]
      for (int idx = tid; idx < out * in + out; idx += blockDim.x) {
        float a = 0.0f;
        if (idx < out * in) {
          const int o = idx / in, i = idx % in;
#pragma unroll
          for (int r = 0; r < REV_ROWS; ++r) a = fmaf(dcur[r * P.max_width + o], act[r * P.act_total + off_in + i], a);
          gacc[P.w_off[l] + idx] += a;
        } else {
          const int o = idx - out * in;
#pragma unroll
          for (int r = 0; r < REV_ROWS; ++r) a += dcur[r * P.max_width + o];
          gacc[P.b_off[l] + o] += a;
        }
      }
      // h-bar_l = W_l^T delta; delta_{l-1} = h-bar (1 - h^2) for hidden layers
      for (int idx = tid; idx < REV_ROWS * in; idx += blockDim.x) {
        const int r = idx / in, i = idx % in;
        float a = 0.0f;
        for (int o = 0; o < out; ++o) a = fmaf(__ldg(W + (size_t)o * in + i), dcur[r * P.max_width + o], a);
        if (l > 0) {
          const float h = act[r * P.act_total + off_in + i];
          a *= (1.0f - h * h);
        }
        dprev[r * P.max_width + i] = a;
      }
      float* tmp = dcur;
      dcur = dprev;
      dprev = tmp;
    }
    __syncthreads();
    // xbar_t = xbar_{t+1} + xs_bar[:p] + d phi/dx^T h0-bar + d(r_t / B)/dx_t
    if (tid < REV_ROWS && tid < valid) {
      const int r = tid;
      const float* x = xt + (size_t)r * p;
      const float rr = reward_fn(rw, x, gs + r * p, p);
      for (int c = 0; c < p; ++c) {
        float hb = dcur[r * P.max_width + c];
        if (P.phi_mode == 1) hb -= dcur[r * P.max_width + 2 * p + c];
        xbar[r * p + c] += xsbar[r * D + c] + hb + invB * rr * rw.Q[c] * (x[c] - gs[r * p + c]) * inv_sr2;
      }
    }
  }
  __syncthreads();
  float* out = theta_part + (size_t)blockIdx.x * P.n_params;
  for (int i = tid; i < P.n_params; i += blockDim.x) out[i] = gacc[i];
}

__global__ void k_reduce_grad(const float* __restrict__ part, int nblk, int n_params,
                              float* __restrict__ grad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_params) return;
  float a = 0.0f;
  for (int b = 0; b < nblk; ++b) a += part[(size_t)b * n_params + i];
  grad[i] = a;
}

__global__ void __launch_bounds__(1024) k_reduce_cost(const double* __restrict__ G, int B, double invB,
                                                      double* __restrict__ cost) {
  __shared__ double sh[1024];
  double a = 0.0;
  for (int b = threadIdx.x; b < B; b += 1024) a += G[b];
  sh[threadIdx.x] = a;
  __syncthreads();
  for (int s = 512; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *cost = -invB * sh[0];
}

__global__ void k_copy_returns(const double* __restrict__ G, int B, float* __restrict__ ret) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) ret[b] = (float)G[b];
}

__global__ void k_philox_raw(const uint32_t* __restrict__ ctr, uint32_t k0, uint32_t k1, int n,
                             uint32_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint4 o = bagel_philox4x32_10(make_uint4(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]), k0, k1);
  out[4 * i] = o.x;
  out[4 * i + 1] = o.y;
  out[4 * i + 2] = o.z;
  out[4 * i + 3] = o.w;
}

__global__ void k_philox_normals(uint64_t seed, long long traj_offset, int B, int T, int p,
                                 float* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)B * T) return;
  const int t = (int)(i / B), b = (int)(i % B);
  const float4 e = bagel_rollout_eps4(seed, (uint32_t)(traj_offset + b), (uint32_t)t);
  for (int m = 0; m < p; ++m) out[((size_t)t * B + b) * p + m] = bagel_f4get(e, m & 3);
}

#define DISPATCH_D(dv, ...)                              \
  switch (dv) {                                          \
    case 2: { constexpr int D = 2; __VA_ARGS__; break; } \
    case 3: { constexpr int D = 3; __VA_ARGS__; break; } \
    case 4: { constexpr int D = 4; __VA_ARGS__; break; } \
    case 5: { constexpr int D = 5; __VA_ARGS__; break; } \
    case 6: { constexpr int D = 6; __VA_ARGS__; break; } \
    case 7: { constexpr int D = 7; __VA_ARGS__; break; } \
    case 8: { constexpr int D = 8; __VA_ARGS__; break; } \
    default: break;                                      \
  }

size_t epi_smem(const PolicyDesc& P) { return sizeof(float) * EPI_ROWS * P.act_total; }

}  // namespace

size_t ro_reverse_smem(const PolicyDesc& P) {
  return sizeof(float) * (((P.n_params + 3) & ~3) + REV_ROWS * P.act_total + 2 * REV_ROWS * P.max_width +
                          REV_ROWS * BAGEL_MAX_P + REV_ROWS * BAGEL_MAX_D);
}
size_t ro_epilogue_smem(const PolicyDesc& P) { return epi_smem(P); }
int ro_reverse_block_rows() { return REV_ROWS; }

void ro_set_attributes() {
  static bool done = false;
  if (done) return;
  done = true;
  for (int dv = 2; dv <= 8; ++dv) {
    DISPATCH_D(dv, ({
      cudaFuncSetAttribute(k_reverse<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_epilogue<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      cudaFuncSetAttribute(k_init<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    }));
  }
}

int ro_init(const bagel_ctx* c, const float* theta, const float* x0, const float* goals, int B,
            cudaStream_t st) {
  ro_set_attributes();
  DISPATCH_D(c->gp.d, (k_init<D><<<cdiv(B, EPI_ROWS), EPI_THREADS, epi_smem(c->pol), st>>>(
                          c->pol, c->rw, c->gp.p, theta, x0, goals, B, c->ws.tape_x, c->ws.G, c->ws.xstar)));
  return 1;
}

int ro_step_epilogue(const bagel_ctx* c, const float* theta, const float* goals, int B, int t, int T,
                     uint64_t seed, long long traj_offset, bool policy_next, float* trace_mu,
                     float* trace_var, cudaStream_t st) {
  (void)T;
  const int p = c->gp.p, d = c->gp.d;
  const Workspace& w = c->ws;
  DISPATCH_D(d, (k_epilogue<D><<<cdiv(B, EPI_ROWS), EPI_THREADS, epi_smem(c->pol), st>>>(
                    c->pol, c->rw, c->gp, theta, goals, B, t, w.S2eff, w.P2, w.mu, w.var,
                    w.tape_x + (size_t)t * B * p, w.tape_sig + (size_t)t * B * p,
                    w.tape_jv + (size_t)t * B * p * d, w.tape_x + (size_t)(t + 1) * B * p, w.G, w.xstar,
                    seed, traj_offset, policy_next ? 1 : 0, w.err_flag, trace_mu, trace_var)));
  return 1;
}

int ro_reverse(const bagel_ctx* c, const float* theta, const float* goals, int B, int T, uint64_t seed,
               long long traj_offset, long long B_global, int* nblk_out, cudaStream_t st) {
  ro_set_attributes();
  const int nblk = cdiv(B, REV_ROWS);
  *nblk_out = nblk;
  const Workspace& w = c->ws;
  DISPATCH_D(c->gp.d, (k_reverse<D><<<nblk, REV_THREADS, ro_reverse_smem(c->pol), st>>>(
                          c->pol, c->rw, c->gp.p, theta, goals, B, T, w.tape_x, w.tape_sig, w.tape_jmu,
                          w.tape_jv, seed, traj_offset, (float)(1.0 / (double)B_global), w.theta_part)));
  return 1;
}

int ro_reduce(const bagel_ctx* c, int nblk, int B, long long B_global, float* grad, cudaStream_t st) {
  k_reduce_grad<<<cdiv(c->pol.n_params, 256), 256, 0, st>>>(c->ws.theta_part, nblk, c->pol.n_params, grad);
  k_reduce_cost<<<1, 1024, 0, st>>>(c->ws.G, B, 1.0 / (double)B_global, c->ws.cost_dev);
  return 2;
}

int ro_copy_returns(const bagel_ctx* c, int B, float* ret, cudaStream_t st) {
  k_copy_returns<<<cdiv(B, 256), 256, 0, st>>>(c->ws.G, B, ret);
  return 1;
}

int ro_philox_raw(const uint32_t* ctr, uint32_t k0, uint32_t k1, int n, uint32_t* out, cudaStream_t st) {
  k_philox_raw<<<cdiv(n, 256), 256, 0, st>>>(ctr, k0, k1, n, out);
  return 1;
}

int ro_philox_normals(uint64_t seed, long long traj_offset, int B, int T, int p, float* out,
                      cudaStream_t st) {
  k_philox_normals<<<cdiv((long long)B * T, 256), 256, 0, st>>>(seed, traj_offset, B, T, p, out);
  return 1;
}
