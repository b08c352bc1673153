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

constexpr int EPI_ROWS = 8;
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
// thetaT holds every W_l transposed (Wt[i][o], same offsets as theta) so that the
// threads of a warp (consecutive o) read consecutive weights: coalesced, L1-resident.
__device__ void mlp_forward_rows(const PolicyDesc& P, const float* __restrict__ thetaT, int nrows, float* act) {
  int off_in = 0;
  for (int l = 0; l < P.n_layers; ++l) {
    const int in = P.sizes[l], out = P.sizes[l + 1];
    const int off_out = off_in + in;
    const float* Wt = thetaT + P.w_off[l];
    const float* bb = thetaT + P.b_off[l];
    __syncthreads();
    for (int idx = threadIdx.x; idx < nrows * out; idx += blockDim.x) {
      const int r = idx / out, o = idx % out;
      const float* h = act + r * P.act_total + off_in;
      float a0 = bb[o], a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;  // 4 independent chains (ILP)
      int i = 0;
      for (; i + 4 <= in; i += 4) {
        a0 = fmaf(Wt[(size_t)i * out + o], h[i], a0);
        a1 = fmaf(Wt[(size_t)(i + 1) * out + o], h[i + 1], a1);
        a2 = fmaf(Wt[(size_t)(i + 2) * out + o], h[i + 2], a2);
        a3 = fmaf(Wt[(size_t)(i + 3) * out + o], h[i + 3], a3);
      }
      for (; i < in; ++i) a0 = fmaf(Wt[(size_t)i * out + o], h[i], a0);
      act[r * P.act_total + off_out + o] = tanhf((a0 + a1) + (a2 + a3));
    }
    off_in = off_out;
  }
  __syncthreads();
}

// thetaT: per layer W_l^T (in x out), biases copied.
__global__ void k_transpose_theta(PolicyDesc P, const float* __restrict__ theta, float* __restrict__ thetaT) {
  for (int l = 0; l < P.n_layers; ++l) {
    const int in = P.sizes[l], out = P.sizes[l + 1];
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < in * out + out; idx += gridDim.x * blockDim.x) {
      if (idx < in * out) {
        const int i = idx / out, o = idx % out;
        thetaT[P.w_off[l] + idx] = theta[P.w_off[l] + o * in + i];
      } else {
        thetaT[P.b_off[l] + idx - in * out] = theta[P.b_off[l] + idx - in * out];
      }
    }
  }
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

// ---------------------------------------------------------------- warp-per-rows policy forward
// The block stages thetaT (every W_l transposed, Wt[i][o], plus biases) in shared memory once;
// each warp then evaluates u = pi(x, g) for RPW rows at a time: lanes own output units
// o = lane + 32 k, activations live in a per-warp shared buffer.  No block-wide barrier after
// the staging.
constexpr int WARP_ROWS_BLOCK = 4;  // warps per block
constexpr int RPW = 2;              // rows per warp
constexpr int ROWS_BLOCK = WARP_ROWS_BLOCK * RPW;

__device__ void stage_theta(const PolicyDesc& P, const float* __restrict__ thetaT, float* th_s) {
  const int n4 = P.n_params / 4;
  for (int i = threadIdx.x; i < n4; i += blockDim.x)
    reinterpret_cast<float4*>(th_s)[i] = __ldg(reinterpret_cast<const float4*>(thetaT) + i);
  for (int i = 4 * n4 + threadIdx.x; i < P.n_params; i += blockDim.x) th_s[i] = __ldg(thetaT + i);
  __syncthreads();
}

// rows r < nr of this warp: x[r], g[r] (p each); u_out[r] (q each).  buf: RPW x 2 x BAGEL_MAX_WIDTH
__device__ void warp_policy(const PolicyDesc& P, int p, const float* th_s, const float* x, const float* g, int nr,
                            float* buf, float* u_out) {
  const int lane = threadIdx.x % 32;
  constexpr int W2 = 2 * BAGEL_MAX_WIDTH;
  for (int r = 0; r < RPW; ++r)
    for (int i = lane; i < P.sizes[0]; i += 32) {
      float v = 0.0f;
      if (r < nr) {
        const float* xr = x + r * p;
        const float* gr = g + r * p;
        if (i < p) v = xr[i];
        else if (i < 2 * p) v = gr[i - p];
        else v = gr[i - 2 * p] - xr[i - 2 * p];
      }
      buf[r * W2 + i] = v;
    }
  __syncwarp();
  int cur = 0;
  for (int l = 0; l < P.n_layers; ++l) {
    const int in = P.sizes[l], out = P.sizes[l + 1];
    const float* Wt = th_s + P.w_off[l];
    const float* bb = th_s + P.b_off[l];
    const int nxt = BAGEL_MAX_WIDTH - cur;
    if (out >= 16) {
      // lanes over output units; 2 interleaved chains per row
      for (int o = lane; o < out; o += 32) {
        float acc[RPW][2];
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
          acc[r][0] = bb[o];
          acc[r][1] = 0.0f;
        }
        int i = 0;
        for (; i + 2 <= in; i += 2) {
          const float w0 = Wt[i * out + o], w1 = Wt[(i + 1) * out + o];
#pragma unroll
          for (int r = 0; r < RPW; ++r) {
            acc[r][0] = fmaf(w0, buf[r * W2 + cur + i], acc[r][0]);
            acc[r][1] = fmaf(w1, buf[r * W2 + cur + i + 1], acc[r][1]);
          }
        }
        if (i < in) {
          const float w0 = Wt[i * out + o];
#pragma unroll
          for (int r = 0; r < RPW; ++r) acc[r][0] = fmaf(w0, buf[r * W2 + cur + i], acc[r][0]);
        }
#pragma unroll
        for (int r = 0; r < RPW; ++r) buf[r * W2 + nxt + o] = tanhf(acc[r][0] + acc[r][1]);
      }
    } else {
      // narrow layer (e.g. the action head): lanes over inputs, butterfly reduction
      for (int o = 0; o < out; ++o) {
        float acc[RPW];
#pragma unroll
        for (int r = 0; r < RPW; ++r) acc[r] = 0.0f;
        for (int i = lane; i < in; i += 32) {
          const float wv = Wt[i * out + o];
#pragma unroll
          for (int r = 0; r < RPW; ++r) acc[r] = fmaf(wv, buf[r * W2 + cur + i], acc[r]);
        }
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
#pragma unroll
          for (int sh = 16; sh > 0; sh >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], sh);
          if (lane == 0) buf[r * W2 + nxt + o] = tanhf(acc[r] + bb[o]);
        }
      }
    }
    __syncwarp();
    cur = nxt;
  }
  const int q = P.sizes[P.n_layers];
  for (int r = 0; r < nr; ++r)
    for (int o = lane; o < q; o += 32) u_out[r * BAGEL_MAX_D + o] = buf[r * W2 + cur + o];
  __syncwarp();
}

size_t policy_smem(const PolicyDesc& P) {
  return sizeof(float) * (((P.n_params + 3) & ~3) + (size_t)WARP_ROWS_BLOCK * RPW * 2 * BAGEL_MAX_WIDTH);
}

template <int D>
__global__ void __launch_bounds__(32 * WARP_ROWS_BLOCK) k_init(PolicyDesc P, RewardDesc rw, int p,
                                                              const float* __restrict__ thetaT,
                                                              const float* __restrict__ x0,
                                                              const float* __restrict__ goals, int B,
                                                              float* __restrict__ tape_x0, double* __restrict__ G,
                                                              float* __restrict__ xstar) {
  extern __shared__ __align__(16) float sm[];
  float* th_s = sm;
  float* bufs = sm + ((P.n_params + 3) & ~3);
  __shared__ float us[WARP_ROWS_BLOCK][RPW][BAGEL_MAX_D];
  stage_theta(P, thetaT, th_s);
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int b0 = blockIdx.x * ROWS_BLOCK + w * RPW;
  if (b0 >= B) return;  // warp-uniform
  const int nr = min(RPW, B - b0);
  const float* x = x0 + (size_t)b0 * p;
  const float* g = goals + (size_t)b0 * p;
  if (lane < nr) G[b0 + lane] = (double)reward_fn(rw, x + lane * p, g + lane * p, p);
  for (int i = lane; i < nr * p; i += 32) tape_x0[(size_t)b0 * p + i] = x[i];
  warp_policy(P, p, th_s, x, g, nr, bufs + (size_t)w * RPW * 2 * BAGEL_MAX_WIDTH, &us[w][0][0]);
  for (int i = lane; i < nr * D; i += 32) {
    const int r = i / D, c = i % D;
    xstar[(size_t)(b0 + r) * D + c] = c < p ? x[r * p + c] : us[w][r][c - p];
  }
}

template <int D>
__global__ void __launch_bounds__(32 * WARP_ROWS_BLOCK) k_epilogue(
    PolicyDesc P, RewardDesc rw, GpDesc g, const float* __restrict__ thetaT, const float* __restrict__ goals,
    int B, int t, int S2, const float* __restrict__ P2, const float* __restrict__ mu,
    const float* __restrict__ var, const float* __restrict__ tape_x_t, const float* __restrict__ sig_t,
    float* __restrict__ jv_t, float* __restrict__ tape_x_next, double* __restrict__ G,
    float* __restrict__ xstar, uint64_t seed, long long traj_offset, int policy_next,
    int* __restrict__ err_flag, float* __restrict__ trace_mu, float* __restrict__ trace_var) {
  extern __shared__ __align__(16) float sm[];
  float* th_s = sm;
  float* bufs = sm + ((P.n_params + 3) & ~3);
  __shared__ float us[WARP_ROWS_BLOCK][RPW][BAGEL_MAX_D];
  __shared__ float xn_s[WARP_ROWS_BLOCK][RPW * BAGEL_MAX_P];
  if (policy_next) stage_theta(P, thetaT, th_s);
  const int p = g.p;
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int b0 = blockIdx.x * ROWS_BLOCK + w * RPW;
  if (b0 >= B) return;  // warp-uniform
  const int nr = min(RPW, B - b0);
  // lane = r * p * (D + 1) + m * (D + 1) + c: pass-2 partial of (row r, output m, column c)
  const int per_row = p * (D + 1);
  const int nl = nr * per_row;  // <= 2 * 4 * 9 = 72 > 32 possible: loop
  for (int base = 0; base < RPW * per_row; base += 32) {
    const int li = base + lane;
    const bool act = li < nl;
    const int r = act ? li / per_row : 0, m = act ? (li % per_row) / (D + 1) : 0, c = act ? li % (D + 1) : 0;
    const int b = b0 + r;
    float part = 0.0f;
    if (act)
      for (int s = 0; s < S2; ++s) part += P2[((size_t)(s * p + m) * B + b) * P2_LD + c];
    // the c = 0 partial (sum w k) of the same (r, m) sits at lane li - c (same 32-lane window
    // only when aligned; fetch it from global instead to keep lanes independent)
    float s0 = part;
    if (act && c > 0) {
      s0 = 0.0f;
      for (int s = 0; s < S2; ++s) s0 += P2[((size_t)(s * p + m) * B + b) * P2_LD];
      jv_t[((size_t)b * p + m) * D + c - 1] = 2.0f * g.ell2inv[m][c - 1] * (xstar[(size_t)b * D + c - 1] * s0 - part);
    }
  }
  if (lane < nr * p) {
    const int r = lane / p, m = lane % p, b = b0 + r;
    const float4 e4 = bagel_rollout_eps4(seed, (uint32_t)(traj_offset + b), (uint32_t)t);
    const float sg = fabsf(sig_t[(size_t)b * p + m]);
    const float mum = mu[(size_t)m * B + b];
    const float xn = tape_x_t[(size_t)b * p + m] + mum + sg * bagel_f4get(e4, m & 3);
    if (!isfinite(xn)) atomicMin(err_flag, t * B + b);
    tape_x_next[(size_t)b * p + m] = xn;
    xn_s[w][r * p + m] = xn;
    if (trace_mu) trace_mu[(size_t)b * p + m] = mum;
    if (trace_var) trace_var[(size_t)b * p + m] = var[(size_t)m * B + b];
  }
  __syncwarp();
  const float* gb = goals + (size_t)b0 * p;
  if (lane < nr) G[b0 + lane] += (double)reward_fn(rw, &xn_s[w][lane * p], gb + lane * p, p);
  if (!policy_next) return;
  warp_policy(P, p, th_s, xn_s[w], gb, nr, bufs + (size_t)w * RPW * 2 * BAGEL_MAX_WIDTH, &us[w][0][0]);
  for (int i = lane; i < nr * D; i += 32) {
    const int r = i / D, c = i % D;
    xstar[(size_t)(b0 + r) * D + c] = c < p ? xn_s[w][r * p + c] : us[w][r][c - p];
  }
}

// ------------------------------------------------------------------ reverse
// smem: gacc[n_params] | act[REV_ROWS x act_total] | dl[2][REV_ROWS x max_width] | xbar | xsbar
template <int D>
__global__ void __launch_bounds__(REV_THREADS) k_reverse(
    PolicyDesc P, RewardDesc rw, int p, const float* __restrict__ theta, const float* __restrict__ thetaT,
    const float* __restrict__ goals, int B, int T, const float* __restrict__ tape_x, const float* __restrict__ tape_sig,
    const float* __restrict__ tape_jmu, const float* __restrict__ tape_jv, uint64_t seed,
    long long traj_offset, float invB, float* __restrict__ theta_part) {
  extern __shared__ __align__(16) float sm[];
  const int np4 = (P.n_params + 3) & ~3;
  float* th_s = sm;                 // theta (W_l row-major) for h-bar = W^T delta
  float* thT_s = th_s + np4;        // theta^T for the forward recompute
  float* gacc = thT_s + np4;
  float* act = gacc + np4;
  float* dl0 = act + REV_ROWS * P.act_total;
  float* dl1 = dl0 + REV_ROWS * P.max_width;
  float* xbar = dl1 + REV_ROWS * P.max_width;  // REV_ROWS x p
  float* xsbar = xbar + REV_ROWS * BAGEL_MAX_P;  // REV_ROWS x D
  __shared__ float gs[REV_ROWS * BAGEL_MAX_P];

  const int tid = threadIdx.x;
  const int row0 = blockIdx.x * REV_ROWS;
  const int valid = min(REV_ROWS, B - row0);
  const float inv_sr2 = 2.0f * rw.inv_two_sr2;
  for (int i = tid; i < P.n_params; i += blockDim.x) {
    gacc[i] = 0.0f;
    th_s[i] = __ldg(theta + i);
    thT_s[i] = __ldg(thetaT + i);
  }
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
    mlp_forward_rows(P, thT_s, REV_ROWS, act);  // ends with __syncthreads
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
      const float* W = th_s + P.w_off[l];
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
        float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
        int o = 0;
        for (; o + 4 <= out; o += 4) {
          a0 = fmaf(W[(size_t)o * in + i], dcur[r * P.max_width + o], a0);
          a1 = fmaf(W[(size_t)(o + 1) * in + i], dcur[r * P.max_width + o + 1], a1);
          a2 = fmaf(W[(size_t)(o + 2) * in + i], dcur[r * P.max_width + o + 2], a2);
          a3 = fmaf(W[(size_t)(o + 3) * in + i], dcur[r * P.max_width + o + 3], a3);
        }
        for (; o < out; ++o) a0 = fmaf(W[(size_t)o * in + i], dcur[r * P.max_width + o], a0);
        float a = (a0 + a1) + (a2 + a3);
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
  return sizeof(float) * (3 * ((P.n_params + 3) & ~3) + REV_ROWS * P.act_total + 2 * REV_ROWS * P.max_width +
                          REV_ROWS * BAGEL_MAX_P + REV_ROWS * BAGEL_MAX_D);
}
size_t ro_policy_smem(const PolicyDesc& P) { return policy_smem(P); }
size_t ro_epilogue_smem(const PolicyDesc& P) { return epi_smem(P); }
int ro_reverse_block_rows() { return REV_ROWS; }

void ro_set_attributes() {
  static bool done = false;
  if (done) return;
  done = true;
  for (int dv = 2; dv <= 8; ++dv) {
    DISPATCH_D(dv, ({
      bagel_set_smem_attr(k_reverse<D>, 200 * 1024);
      bagel_set_smem_attr(k_epilogue<D>, 200 * 1024);
      bagel_set_smem_attr(k_init<D>, 200 * 1024);

    }));
  }
}

int ro_init(const bagel_ctx* c, const float* theta, const float* x0, const float* goals, int B,
            cudaStream_t st) {
  ro_set_attributes();
  k_transpose_theta<<<cdiv(c->pol.n_params, 256), 256, 0, st>>>(c->pol, theta, c->ws.thetaT);
  DISPATCH_D(c->gp.d, (k_init<D><<<cdiv(B, ROWS_BLOCK), 32 * WARP_ROWS_BLOCK, policy_smem(c->pol), st>>>(
                          c->pol, c->rw, c->gp.p, c->ws.thetaT, x0, goals, B, c->ws.tape_x, c->ws.G, c->ws.xstar)));
  return 2;
}

int ro_step_epilogue(const bagel_ctx* c, const float* theta, const float* goals, int B, int t, int T,
                     uint64_t seed, long long traj_offset, bool policy_next, float* trace_mu,
                     float* trace_var, cudaStream_t st) {
  (void)T;
  const int p = c->gp.p, d = c->gp.d;
  const Workspace& w = c->ws;
  DISPATCH_D(d, (k_epilogue<D><<<cdiv(B, ROWS_BLOCK), 32 * WARP_ROWS_BLOCK, policy_smem(c->pol), st>>>(
                    c->pol, c->rw, c->gp, w.thetaT, goals, B, t, w.S2eff, w.P2, w.mu, w.var,
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
                          c->pol, c->rw, c->gp.p, theta, w.thetaT, goals, B, T, w.tape_x, w.tape_sig, w.tape_jmu,
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
