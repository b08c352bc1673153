// rollout.cu -- everything of the rollout except the GP contraction:
//   init       G = r(x0, g) (Alg.1), tape x_0, policy u_0 = pi(x_0, g)
//   epilogue   per step: finish J^v, eps (Philox), x' = x + mu + sigma eps (Eq.9-10),
//              G += r(x', g), tape row (a8), next action u' = pi(x', g)
//   reverse    hand-written reverse mode over the tape, t = T-1..0 (SURVEY
//              Appendix B): one warp per trajectory; theta-bar as one contraction over
//              the (t, b) adjoint tape afterwards
//   reduce     fixed-order sum of the per-CTA theta-bar partials and of the returns
//              (L = -(1/B_global) sum_b G_b)
// The policy is the tanh MLP of P:149 (hidden and output tanh, reading R13);
// phi = [x, g] or [x, g, g - x] (R14).  These kernels are latency / L2 bound
// (|theta| and the tape are small); no tensor-core work here.
#include <algorithm>

#include "bagel_internal.h"
#include "philox.cuh"
#include "policy_rows.cuh"
#include "tc.cuh"

namespace {

constexpr int EPI_ROWS = 8;

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

__device__ __forceinline__ unsigned long long gtimer_ro() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
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

// Shared-memory budget of the policy kernels.  Policies whose weights do not fit (C3: 133k
// parameters) read theta^T from global memory (L1/L2-resident, lanes read consecutive weights).
constexpr size_t kPolicySmemBudget = 200 * 1024;
__host__ __device__ inline size_t policy_buf_floats() { return (size_t)WARP_ROWS_BLOCK * RPW * 2 * BAGEL_MAX_WIDTH; }
__host__ __device__ inline bool policy_theta_staged(const PolicyDesc& P) {
  return sizeof(float) * (((size_t)P.n_params + 3) / 4 * 4 + policy_buf_floats()) <= kPolicySmemBudget;
}
size_t policy_smem(const PolicyDesc& P) {
  return sizeof(float) * ((policy_theta_staged(P) ? ((size_t)P.n_params + 3) / 4 * 4 : 0) + policy_buf_floats());
}

template <int D>
__global__ void __launch_bounds__(32 * WARP_ROWS_BLOCK) k_init(PolicyDesc P, RewardDesc rw, int p,
                                                              const float* __restrict__ thetaT,
                                                              const float* __restrict__ x0,
                                                              const float* __restrict__ goals, int B,
                                                              float* __restrict__ tape_x0, double* __restrict__ G,
                                                              float* __restrict__ xstar, float* __restrict__ act0) {
  extern __shared__ __align__(16) float sm[];
  const bool staged = policy_theta_staged(P);
  const float* th_s = staged ? sm : thetaT;
  float* bufs = sm + (staged ? ((P.n_params + 3) & ~3) : 0);
  __shared__ float us[WARP_ROWS_BLOCK][RPW][BAGEL_MAX_D];
  if (staged) stage_theta(P, thetaT, sm);
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int b0 = blockIdx.x * ROWS_BLOCK + w * RPW;
  if (b0 >= B) return;  // warp-uniform
  const int nr = min(RPW, B - b0);
  const float* x = x0 + (size_t)b0 * p;
  const float* g = goals + (size_t)b0 * p;
  if (lane < nr) G[b0 + lane] = (double)rows::reward_fn(rw, x + lane * p, g + lane * p, p);
  for (int i = lane; i < nr * p; i += 32) tape_x0[(size_t)b0 * p + i] = x[i];
  rows::warp_policy<RPW>(P, p, th_s, x, g, nr, bufs + (size_t)w * RPW * 2 * BAGEL_MAX_WIDTH, &us[w][0][0],
              act0 + (size_t)b0 * P.act_ld);
  for (int i = lane; i < nr * D; i += 32) {
    const int r = i / D, c = i % D;
    xstar[(size_t)(b0 + r) * D + c] = c < p ? x[r * p + c] : us[w][r][c - p];
  }
}

template <int D>
__global__ void __launch_bounds__(32 * WARP_ROWS_BLOCK) k_epilogue(EpiArgs e, unsigned long long* __restrict__ dbg) {
  extern __shared__ __align__(16) float sm[];
  const bool staged = policy_theta_staged(e.P);
  const float* th_s = staged ? sm : e.thetaT;
  float* bufs = sm + (staged ? ((e.P.n_params + 3) & ~3) : 0);
  __shared__ float scratch[WARP_ROWS_BLOCK][rows::epi_scratch_floats<D, RPW>()];
  if (dbg && threadIdx.x == 0) dbg[blockIdx.x * 16 + 0] = gtimer_ro();
  if (staged && e.t + 1 < e.T) stage_theta(e.P, e.thetaT, sm);
  if (dbg && threadIdx.x == 0) dbg[blockIdx.x * 16 + 1] = gtimer_ro();
  const int w = threadIdx.x / 32;
  const int b0 = blockIdx.x * ROWS_BLOCK + w * RPW;
  if (b0 >= e.B) return;  // warp-uniform
  rows::epi_warp_rows<D, RPW>(e, e.t, b0, min(RPW, e.B - b0), th_s, bufs + (size_t)w * RPW * 2 * BAGEL_MAX_WIDTH,
                              scratch[w]);
  if (dbg && threadIdx.x == 0) dbg[blockIdx.x * 16 + 4] = gtimer_ro();
}

// ------------------------------------------------------------------ reverse
// The adjoint recursion couples the steps of ONE trajectory only, so it
// runs as one warp per row over t = T-1..0 with everything it needs on the tape: the combined
// state Jacobian A_t = J^mu + (eps / 2 sigma) J^v (epilogue) and every policy activation
// (forward).  The recursion emits delta_l (the pre-activation adjoints) to a tape; the parameter
// gradient sum_{t,b} delta_l h_l^T is a separate contraction over all (t, b) (k_theta_grad).
//   xs-bar_c = sum_m xbar_m A_t[m][c]                                       (c < d)
//   delta_L  = xs-bar[p:] (1 - u^2);  delta_{l-1} = (W_l^T delta_l) (1 - h_l^2)
//   xbar_t   = xbar_{t+1} + xs-bar[:p] + dphi/dx^T (W_0^T delta_0) + d(r_t / B)/dx_t
// W (row-major, as theta) is staged in shared memory once per block; each step's tape row
// (activations, A, x) is prefetched three steps ahead with cp.async into a per-warp ring, so the
// recursion itself only touches shared memory (one step of the chain is shorter than the tape's
// HBM latency).
constexpr int REV2_WARPS = 8;
constexpr int REV2_RING = 4;  // tape-row buffers per warp: steps t .. t-3 in flight (prefetch distance 3)

__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// per-warp shared region of k_reverse2: 2 adjoint buffers + 2 tape rows [act | A | x]
__host__ __device__ inline int rev2_row_floats(const PolicyDesc& P, int p, int d) {
  return (P.act_ld + p * d + p + 3) & ~3;
}
__host__ __device__ inline int rev2_warp_floats(const PolicyDesc& P, int p, int d) {
  return 2 * ((P.max_width + 3) & ~3) + REV2_RING * rev2_row_floats(P, p, d);
}
// Staged weights: every W_l transposed, Wt[i][o], rows padded to round4(out) + 4 floats (float4
// reads of a row by consecutive lanes are bank-conflict free).
__host__ __device__ inline int rev2_wt_ld(int out) { return ((out + 3) & ~3) + 4; }
__host__ __device__ inline int rev2_wt_floats(const PolicyDesc& P) {
  int n = 0;
  for (int l = 0; l < P.n_layers; ++l) n += P.sizes[l] * rev2_wt_ld(P.sizes[l + 1]);
  return n;
}
__host__ __device__ inline bool rev2_theta_staged(const PolicyDesc& P, int p, int d) {
  return sizeof(float) * ((size_t)rev2_wt_floats(P) + (size_t)REV2_WARPS * rev2_warp_floats(P, p, d)) <= 200 * 1024;
}

template <int D, bool STAGED>
__global__ void __launch_bounds__(32 * REV2_WARPS) k_reverse2(
    PolicyDesc P, RewardDesc rw, int p, const float* __restrict__ theta, const float* __restrict__ goals, int B,
    int T, const float* __restrict__ tape_x, const float* __restrict__ tape_A, const float* __restrict__ tape_act,
    float* __restrict__ tape_delta, float invB, float carry, unsigned long long* __restrict__ dbg) {
  extern __shared__ __align__(16) float sm[];
  constexpr bool staged = STAGED;  // (a compile-time choice: shared-memory W reads stay LDS)
  const int np4 = staged ? rev2_wt_floats(P) : 0;
  const int RF = rev2_row_floats(P, p, D);
  const int mw4 = (P.max_width + 3) & ~3;
  const float* th_s = staged ? sm : theta;  // W row-major, as theta (global when too large)
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  float* d0 = sm + np4 + (size_t)w * rev2_warp_floats(P, p, D);  // this warp's region
  float* d1 = d0 + mw4;
  float* rows = d1 + mw4;  // 2 x RF: [act | A | x] of one step
  if (staged) {
    int wo = 0;
    for (int l = 0; l < P.n_layers; ++l) {
      const int in = P.sizes[l], out = P.sizes[l + 1], ld = rev2_wt_ld(out);
      for (int idx = threadIdx.x; idx < in * out; idx += blockDim.x) {
        const int o = idx / in, i = idx % in;
        sm[wo + i * ld + o] = __ldg(theta + P.w_off[l] + idx);
      }
      wo += in * ld;
    }
  }
  __syncthreads();
  const int b = blockIdx.x * REV2_WARPS + w;
  if (b >= B || T <= 0) return;  // warp-uniform
  const int L = P.n_layers;
  const int q = P.sizes[L];
  const int AL = P.act_ld, pd = p * D;
  const float inv_sr2 = 2.0f * rw.inv_two_sr2;
  auto prefetch = [&](int t, float* dst) {
    const float* act = tape_act + ((size_t)t * B + b) * AL;
    const float* A = tape_A + ((size_t)t * B + b) * pd;
    const float* x = tape_x + ((size_t)t * B + b) * p;
    for (int i = lane * 4; i < AL; i += 128) cp_async16(dst + i, act + i);
    if (lane < pd) cp_async4(dst + AL + lane, A + lane);
    if (lane < p) cp_async4(dst + AL + pd + lane, x + lane);
    cp_async_commit();
  };
  for (int k = 0; k < REV2_RING - 1; ++k) {  // steps T-1, T-2, T-3 (empty groups past t = 0)
    if (T - 1 - k >= 0) prefetch(T - 1 - k, rows + k * RF);
    else cp_async_commit();
  }
  const float gl = lane < p ? goals[(size_t)b * p + lane] : 0.0f;
  float xb = 0.0f;
  {
    // xbar_T = (1/B) r(x_T) Q (x_T - g) / sigma_r^2
    const float xT = lane < p ? tape_x[((size_t)T * B + b) * p + lane] : 0.0f;
    float qd = lane < p ? rw.Q[lane] * (xT - gl) * (xT - gl) : 0.0f;
    for (int o = 16; o > 0; o >>= 1) qd += __shfl_xor_sync(0xffffffffu, qd, o);
    const float rr = expf(-qd * rw.inv_two_sr2);
    if (lane < p) xb = invB * rr * rw.Q[lane] * (xT - gl) * inv_sr2;
  }
  for (int t = T - 1; t >= 0; --t) {
    const bool stampit = dbg && blockIdx.x == 0 && threadIdx.x == 0 && t == T / 2;
    if (stampit) dbg[0] = gtimer_ro();
    float* cur = rows + ((T - 1 - t) % REV2_RING) * RF;
    if (t - (REV2_RING - 1) >= 0) prefetch(t - (REV2_RING - 1), rows + ((T - 1 - t + REV2_RING - 1) % REV2_RING) * RF);
    else cp_async_commit();
    cp_async_wait<REV2_RING - 1>();  // step t's group (issued REV2_RING - 1 groups ago) has landed
    __syncwarp();
    if (stampit) dbg[1] = gtimer_ro();
    const float* act = cur;
    const float* At = cur + AL;
    const float xt = lane < p ? cur[AL + pd + lane] : 0.0f;
    float* dl = tape_delta + ((size_t)t * B + b) * P.d_ld;
    // xs-bar_c (lane c < D)
    float xs = 0.0f;
    for (int m = 0; m < p; ++m) {
      const float xbm = __shfl_sync(0xffffffffu, xb, m);
      if (lane < D) xs = fmaf(xbm, At[m * D + lane], xs);
    }
    // delta_L = ubar (1 - u^2), ubar = xs-bar[p + o]
    for (int o = 0; o < q; o += 32) {
      const float ub = __shfl_sync(0xffffffffu, xs, min(p + o + lane, 31));
      if (o + lane < q) {
        const float u = act[P.aoff[L] + o + lane];
        d0[o + lane] = ub * (1.0f - u * u);
      }
    }
    __syncwarp();
    if (stampit) dbg[2] = gtimer_ro();
    float* dc = d0;
    float* dn = d1;
    int wt_end = np4;  // staged layers are consumed last to first
    for (int l = L - 1; l >= 0; --l) {
      const int in = P.sizes[l], out = P.sizes[l + 1];
      const float* W = th_s + P.w_off[l];
      for (int o = lane; o < out; o += 32) dl[P.doff[l] + o] = dc[o];
      const float* hin = act + P.aoff[l];  // layer l's input activations
      const int ld = rev2_wt_ld(out);
      wt_end -= in * ld;
      if (STAGED && in >= 32) {
        // lanes over inputs, two inputs per pass; W^T rows and delta read as float4
        const float* Wt = sm + wt_end;
        const float4* dv = reinterpret_cast<const float4*>(dc);
        for (int i = lane; i < in; i += 64) {
          const bool two = i + 32 < in;
          const int i2 = two ? i + 32 : i;
          const float4* w1 = reinterpret_cast<const float4*>(Wt + (size_t)i * ld);
          const float4* w2 = reinterpret_cast<const float4*>(Wt + (size_t)i2 * ld);
          float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f, c0 = 0.0f, c1 = 0.0f, c2 = 0.0f, c3 = 0.0f;
          const int n4 = out / 4;
#pragma unroll 4
          for (int o4 = 0; o4 < n4; ++o4) {
            const float4 e = dv[o4], x = w1[o4], y = w2[o4];
            a0 = fmaf(x.x, e.x, a0);
            a1 = fmaf(x.y, e.y, a1);
            a2 = fmaf(x.z, e.z, a2);
            a3 = fmaf(x.w, e.w, a3);
            c0 = fmaf(y.x, e.x, c0);
            c1 = fmaf(y.y, e.y, c1);
            c2 = fmaf(y.z, e.z, c2);
            c3 = fmaf(y.w, e.w, c3);
          }
          for (int o = 4 * n4; o < out; ++o) {
            a0 = fmaf(Wt[(size_t)i * ld + o], dc[o], a0);
            c0 = fmaf(Wt[(size_t)i2 * ld + o], dc[o], c0);
          }
          const float hb = (a0 + a1) + (a2 + a3), hb2 = (c0 + c1) + (c2 + c3);
          if (l > 0) {
            const float h = hin[i];
            dn[i] = hb * (1.0f - h * h);
            if (two) {
              const float h2 = hin[i2];
              dn[i2] = hb2 * (1.0f - h2 * h2);
            }
          } else {
            dn[i] = hb;
            if (two) dn[i2] = hb2;
          }
        }
      } else if (STAGED) {
        // narrow input from the staged W^T: lane = (o group, i), xor-reduced (fixed tree)
        const float* Wt = sm + wt_end;
        int ip = 1;
        while (ip < in) ip <<= 1;
        const int ng = 32 / ip, i = lane % ip, grp = lane / ip;
        float a = 0.0f;
        if (i < in)
          for (int o = grp; o < out; o += ng) a = fmaf(Wt[i * ld + o], dc[o], a);
        for (int sh = 16; sh >= ip; sh >>= 1) a += __shfl_xor_sync(0xffffffffu, a, sh);
        if (lane < in) {
          const float h = l > 0 ? hin[lane] : 0.0f;
          dn[lane] = l > 0 ? a * (1.0f - h * h) : a;
        }
      } else if (in >= 32) {
        // lanes over inputs, two inputs per pass, 4 o's per iteration (8 independent chains)
        for (int i = lane; i < in; i += 64) {
          const bool two = i + 32 < in;
          const int i2 = two ? i + 32 : i;
          float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f, c0 = 0.0f, c1 = 0.0f, c2 = 0.0f, c3 = 0.0f;
          int o = 0;
#pragma unroll 2
          for (; o + 4 <= out; o += 4) {
            const float e0 = dc[o], e1 = dc[o + 1], e2 = dc[o + 2], e3 = dc[o + 3];
            a0 = fmaf(W[(o + 0) * in + i], e0, a0);
            a1 = fmaf(W[(o + 1) * in + i], e1, a1);
            a2 = fmaf(W[(o + 2) * in + i], e2, a2);
            a3 = fmaf(W[(o + 3) * in + i], e3, a3);
            c0 = fmaf(W[(o + 0) * in + i2], e0, c0);
            c1 = fmaf(W[(o + 1) * in + i2], e1, c1);
            c2 = fmaf(W[(o + 2) * in + i2], e2, c2);
            c3 = fmaf(W[(o + 3) * in + i2], e3, c3);
          }
          for (; o < out; ++o) {
            a0 = fmaf(W[o * in + i], dc[o], a0);
            c0 = fmaf(W[o * in + i2], dc[o], c0);
          }
          const float hb = (a0 + a1) + (a2 + a3), hb2 = (c0 + c1) + (c2 + c3);
          if (l > 0) {
            const float h = hin[i];
            dn[i] = hb * (1.0f - h * h);
            if (two) {
              const float h2 = hin[i2];
              dn[i2] = hb2 * (1.0f - h2 * h2);
            }
          } else {
            dn[i] = hb;
            if (two) dn[i2] = hb2;
          }
        }
      } else {
        // narrow input: lane = (o group, i); groups of the o range, xor-reduced (fixed tree)
        int ip = 1;
        while (ip < in) ip <<= 1;
        const int ng = 32 / ip, i = lane % ip, grp = lane / ip;
        float a = 0.0f;
        if (i < in)
          for (int o = grp; o < out; o += ng) a = fmaf(W[o * in + i], dc[o], a);
        for (int sh = 16; sh >= ip; sh >>= 1) a += __shfl_xor_sync(0xffffffffu, a, sh);
        if (lane < in) {
          const float h = l > 0 ? hin[lane] : 0.0f;
          dn[lane] = l > 0 ? a * (1.0f - h * h) : a;
        }
      }
      __syncwarp();
      if (stampit) dbg[3 + (L - 1 - l)] = gtimer_ro();
      float* tmp = dc;
      dc = dn;
      dn = tmp;
    }
    // xbar_t = xbar_{t+1} + xs-bar[:p] + dphi/dx^T h0-bar + d(r_t / B)/dx_t; phi = [x, g] or [x, g, g - x]
    float hb_phi = 0.0f;
    if (lane < p) {
      hb_phi = dc[lane];
      if (P.phi_mode == 1) hb_phi -= dc[2 * p + lane];
    }
    float qd = lane < p ? rw.Q[lane] * (xt - gl) * (xt - gl) : 0.0f;
    for (int o = 16; o > 0; o >>= 1) qd += __shfl_xor_sync(0xffffffffu, qd, o);
    const float rr = expf(-qd * rw.inv_two_sr2);
    // carry = 1 for Delta targets (dx'/dx = I + ...), 0 for absolute targets (NEXT-4)
    if (lane < p) xb = carry * xb + xs + hb_phi + invB * rr * rw.Q[lane] * (xt - gl) * inv_sr2;
    __syncwarp();
    if (stampit) dbg[8] = gtimer_ro();
  }
}

// theta-bar = sum over (t, b) of delta_l h_l^T (weights) and delta_l (biases): a K = T B
// contraction split over the CTAs (contiguous K ranges, one partial per CTA, summed in CTA order
// by k_reduce_grad).  The tape rows of a range are contiguous, so TG_KC-row chunks of both tapes
// arrive by 1-D bulk copies (TMA engine) into a TG_ST-stage ring; each thread owns up to TG_JOBS
// TO x TI (o, i) weight tiles (or TO-bias groups) with register accumulators and reads its float4
// slices of every staged row.
constexpr int TG_THREADS = 256, TG_KC = 32, TG_ST = 3;
// Tiles of TO x TI (o, i) per job, TG_JOBS jobs per thread: every job batch streams the CTA's whole
// K range again, and each staged row costs (TO + TI) / 4 shared-memory float4 loads per TO TI FMAs,
// so wide policies (C3) use 2 jobs of 8 x 8 (5 passes over the tape instead of 17 with 4 x 4; half
// the shared-memory traffic per FMA) and small ones 2 of 4 x 4 (one pass either way).

template <int TG_JOBS, int TO, int TI>
__global__ void __launch_bounds__(TG_THREADS) k_theta_grad(PolicyDesc P, long long K, int KC,
                                                          const float* __restrict__ tape_act,
                                                          const float* __restrict__ tape_delta,
                                                          float* __restrict__ theta_part) {
  extern __shared__ __align__(16) float sm[];
  __shared__ __align__(8) uint64_t full[TG_ST];
  const int AL = P.act_ld, DL = P.d_ld;
  const int stage_f = KC * (AL + DL);
  const long long per = (K + gridDim.x - 1) / gridDim.x;
  const long long k0 = blockIdx.x * per, k1 = min(K, k0 + per);
  const int nchunks = k1 > k0 ? (int)((k1 - k0 + KC - 1) / KC) : 0;
  float* out = theta_part + (size_t)blockIdx.x * P.n_params;
  if (threadIdx.x == 0) {
    for (int s = 0; s < TG_ST; ++s) tc::mbar_init(&full[s], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  int njobs = 0;
  for (int l = 0; l < P.n_layers; ++l) njobs += ((P.sizes[l + 1] + TO - 1) / TO) * ((P.sizes[l] + TI - 1) / TI + 1);
  const int nbatch = (njobs + TG_THREADS * TG_JOBS - 1) / (TG_THREADS * TG_JOBS);
  const int total = nbatch * nchunks;  // the K range is streamed once per job batch
  // chunk g of the whole sequence: batch g / nchunks, rows of chunk g % nchunks; stage g % TG_ST
  auto issue = [&](int g) {
    const int s = g % TG_ST, c = g % nchunks;
    const long long r0 = k0 + (long long)c * KC;
    const int rows = (int)min((long long)KC, k1 - r0);
    const uint32_t ba = (uint32_t)rows * AL * 4, bd = (uint32_t)rows * DL * 4;
    tc::mbar_arrive_expect_tx(&full[s], ba + bd);
    float* dst = sm + (size_t)s * stage_f;
    tc::bulk_g2s(dst, tape_act + r0 * AL, ba, &full[s]);
    tc::bulk_g2s(dst + KC * AL, tape_delta + r0 * DL, bd, &full[s]);
  };
  if (threadIdx.x == 0)
    for (int g = 0; g < TG_ST && g < total; ++g) issue(g);
  for (int batch = 0; batch < nbatch; ++batch) {
    const int jbase = batch * TG_THREADS * TG_JOBS;
    // job u of this thread: delta slice offset, activation slice offset (-1: bias group)
    int jd[TG_JOBS], ja[TG_JOBS];
#pragma unroll
    for (int u = 0; u < TG_JOBS; ++u) {
      int j = jbase + u * TG_THREADS + threadIdx.x;
      jd[u] = -1;
      ja[u] = -1;
      for (int l = 0; l < P.n_layers && j >= 0; ++l) {
        const int no = (P.sizes[l + 1] + TO - 1) / TO, ni = (P.sizes[l] + TI - 1) / TI + 1;
        if (j < no * ni) {
          jd[u] = P.doff[l] + (j / ni) * TO;
          ja[u] = (j % ni) == ni - 1 ? -1 : P.aoff[l] + (j % ni) * TI;
        }
        j -= no * ni;
      }
    }
    float acc[TG_JOBS][TO * TI];
#pragma unroll
    for (int u = 0; u < TG_JOBS; ++u)
#pragma unroll
      for (int e = 0; e < TO * TI; ++e) acc[u][e] = 0.0f;
    for (int c = 0; c < nchunks; ++c) {
      const int g = batch * nchunks + c, s = g % TG_ST;
      const int rows = (int)min((long long)KC, k1 - (k0 + (long long)c * KC));
      tc::mbar_wait(&full[s], (uint32_t)(g / TG_ST) & 1u);
      const float* hs = sm + (size_t)s * stage_f;
      const float* ds = hs + KC * AL;
#pragma unroll
      for (int u = 0; u < TG_JOBS; ++u) {
        if (jd[u] < 0) continue;
        // (a tile may read past its segment -- into the next segment, row or the stage padding;
        // those accumulators belong to parameters that are never written)
        if (ja[u] >= 0) {
          for (int r = 0; r < rows; ++r) {
            float dv[TO], hv[TI];
#pragma unroll
            for (int q = 0; q < TO / 4; ++q) {
              const float4 d4 = *reinterpret_cast<const float4*>(ds + r * DL + jd[u] + 4 * q);
              dv[4 * q] = d4.x; dv[4 * q + 1] = d4.y; dv[4 * q + 2] = d4.z; dv[4 * q + 3] = d4.w;
            }
#pragma unroll
            for (int q = 0; q < TI / 4; ++q) {
              const float4 h4 = *reinterpret_cast<const float4*>(hs + r * AL + ja[u] + 4 * q);
              hv[4 * q] = h4.x; hv[4 * q + 1] = h4.y; hv[4 * q + 2] = h4.z; hv[4 * q + 3] = h4.w;
            }
#pragma unroll
            for (int eo = 0; eo < TO; ++eo)
#pragma unroll
              for (int ei = 0; ei < TI; ++ei) acc[u][eo * TI + ei] = fmaf(dv[eo], hv[ei], acc[u][eo * TI + ei]);
          }
        } else {
          for (int r = 0; r < rows; ++r) {
#pragma unroll
            for (int q = 0; q < TO / 4; ++q) {
              const float4 d4 = *reinterpret_cast<const float4*>(ds + r * DL + jd[u] + 4 * q);
              acc[u][4 * q] += d4.x;
              acc[u][4 * q + 1] += d4.y;
              acc[u][4 * q + 2] += d4.z;
              acc[u][4 * q + 3] += d4.w;
            }
          }
        }
      }
      __syncthreads();  // every thread is done with stage s
      if (threadIdx.x == 0 && g + TG_ST < total) issue(g + TG_ST);
    }
    // write this CTA's partial (every parameter exactly once over the batches)
#pragma unroll
    for (int u = 0; u < TG_JOBS; ++u) {
      int j = jbase + u * TG_THREADS + threadIdx.x;
      for (int l = 0; l < P.n_layers && j >= 0; ++l) {
        const int in = P.sizes[l], outw = P.sizes[l + 1];
        const int no = (outw + TO - 1) / TO, ni = (in + TI - 1) / TI + 1;
        if (j < no * ni) {
          const int o0 = (j / ni) * TO, it = j % ni;
#pragma unroll
          for (int eo = 0; eo < TO; ++eo) {
            if (o0 + eo >= outw) continue;
            if (it == ni - 1) {
              out[P.b_off[l] + o0 + eo] = nchunks ? acc[u][eo] : 0.0f;
            } else {
#pragma unroll
              for (int ei = 0; ei < TI; ++ei)
                if (it * TI + ei < in) out[P.w_off[l] + (o0 + eo) * in + it * TI + ei] = acc[u][eo * TI + ei];
            }
          }
        }
        j -= no * ni;
      }
    }
  }
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

size_t ro_reverse_smem(const PolicyDesc& P, int p, int d) {
  return sizeof(float) * ((rev2_theta_staged(P, p, d) ? (size_t)rev2_wt_floats(P) : 0) +
                          (size_t)REV2_WARPS * rev2_warp_floats(P, p, d));
}
// rows per staged chunk of the theta-gradient contraction: TG_KC, fewer for wide policies so the
// TG_ST-stage ring stays within 200 KB
int tg_chunk_rows(const PolicyDesc& P) {
  const size_t row_bytes = sizeof(float) * (size_t)(P.act_ld + P.d_ld);
  const int kc = (int)std::min<size_t>(TG_KC, (200 * 1024 - 16 * sizeof(float)) / (TG_ST * row_bytes));
  return std::max(kc, 1);
}
size_t ro_theta_grad_smem(const PolicyDesc& P) {
  // + padding: an 8-wide tile of the stage's last row may read up to 8 floats past it
  return sizeof(float) * ((size_t)TG_ST * tg_chunk_rows(P) * (P.act_ld + P.d_ld) + 16);
}
int ro_theta_blocks(const bagel_ctx* c, int B, int T) {
  const long long K = (long long)B * std::max(T, 1);
  if (theta_tc_enabled(c->pol)) return theta_tc_blocks(K);  // tensor-core path: 4,096-row K blocks
  return (int)std::max(1LL, std::min((long long)c->num_sms, K / 64));
}
size_t ro_policy_smem(const PolicyDesc& P) { return policy_smem(P); }
size_t ro_epilogue_smem(const PolicyDesc& P) { return epi_smem(P); }

void ro_set_attributes() {
  static std::atomic<unsigned long long> devices{0};
  if (!bagel_first_on_device(devices)) return;
  bagel_set_smem_attr(k_theta_grad<2, 4, 4>, 200 * 1024);
  bagel_set_smem_attr(k_theta_grad<2, 8, 8>, 200 * 1024);
  for (int dv = 2; dv <= 8; ++dv) {
    DISPATCH_D(dv, ({
      bagel_set_smem_attr(k_reverse2<D, true>, 200 * 1024);
      bagel_set_smem_attr(k_reverse2<D, false>, 200 * 1024);
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
                          c->pol, c->rw, c->gp.p, c->ws.thetaT, x0, goals, B, c->ws.tape_x, c->ws.G, c->ws.xstar,
                          c->ws.tape_act)));
  return 2;
}

EpiArgs ro_epi_args(const bagel_ctx* c, const float* goals, int B, int t, int T, uint64_t seed, long long traj_offset,
                    float* trace_mu, float* trace_var) {
  const Workspace& w = c->ws;
  EpiArgs e{};
  e.P = c->pol;
  e.rw = c->rw;
  e.g = c->gp;
  e.thetaT = w.thetaT;
  e.goals = goals;
  e.B = B;
  e.t = t;
  e.T = T;
  e.S2 = w.S2eff;
  e.P2 = w.P2;
  e.mu = w.mu;
  e.var = w.var;
  e.tape_x = w.tape_x;
  e.tape_sig = w.tape_sig;
  e.tape_jv = w.tape_jv;
  e.tape_jmu = w.tape_jmu;
  e.tape_A = w.tape_A;
  e.tape_act = w.tape_act;
  e.G = w.G;
  e.xstar = w.xstar;
  e.seed = seed;
  e.traj_offset = traj_offset;
  e.err_flag = w.err_flag;
  e.trace_mu = trace_mu;
  e.trace_var = trace_var;
  return e;
}

int ro_step_epilogue(const bagel_ctx* c, const float* theta, const float* goals, int B, int t, int T,
                     uint64_t seed, long long traj_offset, float* trace_mu, float* trace_var, cudaStream_t st) {
  EpiArgs e = ro_epi_args(c, goals, B, t, T, seed, traj_offset, trace_mu, trace_var);
  const bool wide = ro_wide_policy(c->pol);
  e.policy_external = wide ? 1 : 0;
  DISPATCH_D(c->gp.d, (k_epilogue<D><<<cdiv(B, ROWS_BLOCK), 32 * WARP_ROWS_BLOCK, policy_smem(c->pol), st>>>(
                          e, t == T - 2 ? c->tcs.dbg3 : nullptr)));
  if (wide && t + 1 < T) return 1 + mlp_forward_step(c, theta, goals, B, t + 1, st);  // tiled a1 of step t + 1
  return 1;
}

bool ro_wide_policy(const PolicyDesc& P) { return !policy_theta_staged(P); }

int ro_reverse(const bagel_ctx* c, const float* theta, const float* goals, int B, int T, uint64_t seed,
               long long traj_offset, long long B_global, int* nblk_out, cudaStream_t st) {
  (void)seed;
  (void)traj_offset;
  ro_set_attributes();
  const Workspace& w = c->ws;
  if (ro_wide_policy(c->pol)) {  // register-tiled GEMM steps (mlp_tiled.cu)
    *nblk_out = ro_theta_blocks(c, B, T);
    return T > 0 ? mlp_reverse(c, theta, goals, B, T, B_global, st) : 0;
  }
  const size_t smem = ro_reverse_smem(c->pol, c->gp.p, c->gp.d);
  const float invB = (float)(1.0 / (double)B_global);
  if (rev2_theta_staged(c->pol, c->gp.p, c->gp.d)) {
    DISPATCH_D(c->gp.d, (k_reverse2<D, true><<<cdiv(B, REV2_WARPS), 32 * REV2_WARPS, smem, st>>>(
                            c->pol, c->rw, c->gp.p, theta, goals, B, T, w.tape_x, w.tape_A, w.tape_act, w.tape_delta,
                            invB, c->gp.abs_target ? 0.0f : 1.0f, c->tcs.dbg3)));
  } else {
    DISPATCH_D(c->gp.d, (k_reverse2<D, false><<<cdiv(B, REV2_WARPS), 32 * REV2_WARPS, smem, st>>>(
                            c->pol, c->rw, c->gp.p, theta, goals, B, T, w.tape_x, w.tape_A, w.tape_act, w.tape_delta,
                            invB, c->gp.abs_target ? 0.0f : 1.0f, c->tcs.dbg3)));
  }
  *nblk_out = ro_theta_blocks(c, B, T);
  return 1;
}

int ro_theta_grad(const bagel_ctx* c, int B, int T, int nblk, cudaStream_t st) {
  const Workspace& w = c->ws;
  if (theta_tc_enabled(c->pol))  // wide policies: the delta^T H contraction on the tensor cores
    return theta_grad_tc(c->pol, (long long)T * B, w.tape_act, w.tape_delta, w.theta_colmax, w.theta_part, st);
  int njobs = 0;
  for (int l = 0; l < c->pol.n_layers; ++l)
    njobs += ((c->pol.sizes[l + 1] + 3) / 4) * ((c->pol.sizes[l] + 3) / 4 + 1);
  if (njobs > 2 * TG_THREADS * 2)
    k_theta_grad<2, 8, 8><<<nblk, TG_THREADS, ro_theta_grad_smem(c->pol), st>>>(
        c->pol, (long long)T * B, tg_chunk_rows(c->pol), w.tape_act, w.tape_delta, w.theta_part);
  else
    k_theta_grad<2, 4, 4><<<nblk, TG_THREADS, ro_theta_grad_smem(c->pol), st>>>(
        c->pol, (long long)T * B, tg_chunk_rows(c->pol), w.tape_act, w.tape_delta, w.theta_part);
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
