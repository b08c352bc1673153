// policy_rows.cuh -- per-row pieces of the rollout shared by the step-epilogue kernel
// (rollout.cu) and the pass-2 kernel with the epilogue fused in (gp_step_tc.cu):
//   reward r(x, g) (Alg.1), the tanh-MLP policy u = pi(x, g) (R13/R14) evaluated by
//   one warp for R rows, and the step epilogue of R rows (J^v from the pass-2 sums, eps by
//   Philox, x' = x + mu + sigma eps (Eq.9-10), G += r(x', g), the reverse-pass tapes, next action).
#pragma once
#include "bagel_internal.h"
#include "philox.cuh"

namespace rows {

constexpr int P2_LD = 1 + BAGEL_MAX_D;

__device__ __forceinline__ float reward_fn(const RewardDesc& rw, const float* x, const float* g, int p) {
  float q = 0.0f;
  for (int c = 0; c < p; ++c) {
    const float df = x[c] - g[c];
    q = fmaf(rw.Q[c] * df, df, q);
  }
  return expf(-q * rw.inv_two_sr2);
}

// rows r < nr <= R of this warp: x[r], g[r] (p each); u_out[r] (q each).  buf: R x 2 x BAGEL_MAX_WIDTH.
// act_out (nullable): every activation of row r, [phi | h_1 | ... | u] (segments at P.aoff,
// row stride P.act_ld), the reverse pass's tape.
template <int R>
__device__ void warp_policy(const PolicyDesc& P, int p, const float* th_s, const float* x, const float* g, int nr,
                            float* buf, float* u_out, float* __restrict__ act_out = nullptr) {
  const int lane = threadIdx.x % 32;
  constexpr int W2 = 2 * BAGEL_MAX_WIDTH;
  for (int r = 0; r < R; ++r)
    for (int i = lane; i < P.sizes[0]; i += 32) {
      float v = 0.0f;
      if (r < nr) {
        const float* xr = x + r * p;
        const float* gr = g + r * p;
        if (i < p) v = xr[i];
        else if (i < 2 * p) v = gr[i - p];
        else v = gr[i - 2 * p] - xr[i - 2 * p];
        if (act_out) act_out[(size_t)r * P.act_ld + i] = v;
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
        float acc[R][2];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          acc[r][0] = bb[o];
          acc[r][1] = 0.0f;
        }
        int i = 0;
        for (; i + 2 <= in; i += 2) {
          const float w0 = Wt[i * out + o], w1 = Wt[(i + 1) * out + o];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            acc[r][0] = fmaf(w0, buf[r * W2 + cur + i], acc[r][0]);
            acc[r][1] = fmaf(w1, buf[r * W2 + cur + i + 1], acc[r][1]);
          }
        }
        if (i < in) {
          const float w0 = Wt[i * out + o];
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r][0] = fmaf(w0, buf[r * W2 + cur + i], acc[r][0]);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float h = tanhf(acc[r][0] + acc[r][1]);
          buf[r * W2 + nxt + o] = h;
          if (act_out && r < nr) act_out[(size_t)r * P.act_ld + P.aoff[l + 1] + o] = h;
        }
      }
    } else {
      // narrow layer (e.g. the action head): lanes over inputs, butterfly reduction
      for (int o = 0; o < out; ++o) {
        float acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0.0f;
        for (int i = lane; i < in; i += 32) {
          const float wv = Wt[i * out + o];
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r] = fmaf(wv, buf[r * W2 + cur + i], acc[r]);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
          for (int sh = 16; sh > 0; sh >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], sh);
          if (lane == 0) {
            const float h = tanhf(acc[r] + bb[o]);
            buf[r * W2 + nxt + o] = h;
            if (act_out && r < nr) act_out[(size_t)r * P.act_ld + P.aoff[l + 1] + o] = h;
          }
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


// Per-warp scratch of epi_warp_rows (floats)
template <int D, int R>
__host__ __device__ constexpr int epi_scratch_floats() {
  return R * BAGEL_MAX_P * (D + 1) + 2 * R * BAGEL_MAX_P + R * BAGEL_MAX_D + R * BAGEL_MAX_P * BAGEL_MAX_D +
         R * BAGEL_MAX_D;
}

// The step epilogue (step t; e.t is ignored) of rows b0 .. b0 + nr - 1 (nr <= R) by one warp, in
// two halves so that the first can overlap a grid barrier:
//   epi_pre   everything that needs only pass 1 of this step: eps (Philox), x' = x + mu + sigma eps,
//             the tapes of x', f = eps / (2 sigma), and the J^mu / x* rows into scratch;
//   epi_post  pass-2 sums -> J^v, A = J^mu + f J^v, r(x'), the next action.
// scratch: epi_scratch_floats<D, R>() floats; buf (post): R x 2 x BAGEL_MAX_WIDTH; th_s: theta^T
// (read when t + 1 < T).
template <int D, int R>
struct EpiScratch {
  float* psum;  // R x p x (D + 1)
  float* f_s;   // R x p
  float* xn_s;  // R x p
  float* us;    // R x MAX_D
  float* jmu;   // R x p x D
  float* xq;    // R x MAX_D (this step's x*)
  __device__ explicit EpiScratch(float* s) {
    psum = s;
    f_s = psum + R * BAGEL_MAX_P * (D + 1);
    xn_s = f_s + R * BAGEL_MAX_P;
    us = xn_s + R * BAGEL_MAX_P;
    jmu = us + R * BAGEL_MAX_D;
    xq = jmu + R * BAGEL_MAX_P * BAGEL_MAX_D;
  }
};

template <int D, int R>
__device__ void epi_pre(const EpiArgs& e, const int t, int b0, int nr, float* scratch) {
  const int lane = threadIdx.x % 32;
  const int p = e.g.p, B = e.B, d = e.g.d;
  EpiScratch<D, R> sc(scratch);
  const float* sig_t = e.tape_sig + (size_t)t * B * p;
  const float* tape_x_t = e.tape_x + (size_t)t * B * p;
  float* tape_x_next = e.tape_x + (size_t)(t + 1) * B * p;
  const float* jmu_t = e.tape_jmu + (size_t)t * B * p * d;
  float* trace_mu = e.trace_mu ? e.trace_mu + (size_t)t * B * p : nullptr;
  float* trace_var = e.trace_var ? e.trace_var + (size_t)t * B * p : nullptr;
  if (lane < nr * p) {
    const int r = lane / p, m = lane % p, b = b0 + r;
    const float4 e4 = bagel_rollout_eps4(e.seed, (uint32_t)(e.traj_offset + b), (uint32_t)t);
    const float sgr = sig_t[(size_t)b * p + m];
    const float sg = fabsf(sgr);
    const float ep = bagel_f4get(e4, m & 3);
    const float mum = e.mu[(size_t)m * B + b];
    const float xn = (e.g.abs_target ? 0.0f : tape_x_t[(size_t)b * p + m]) + mum + sg * ep;
    if (!isfinite(xn)) atomicMin(e.err_flag, t * B + b);
    tape_x_next[(size_t)b * p + m] = xn;
    sc.xn_s[r * p + m] = xn;
    // d x'/d sigma^2 = eps / (2 sigma) where the variance is not clamped (R19), else 0
    sc.f_s[r * p + m] = sgr > 0.0f ? ep / (2.0f * sgr) : 0.0f;
    if (trace_mu) trace_mu[(size_t)b * p + m] = mum;
    if (trace_var) trace_var[(size_t)b * p + m] = e.var[(size_t)m * B + b];
  }
  for (int i = lane; i < nr * p * D; i += 32) {
    const int r = i / (p * D), o = i % (p * D);
    sc.jmu[r * BAGEL_MAX_P * BAGEL_MAX_D + o] = jmu_t[(size_t)(b0 + r) * p * D + o];
  }
  for (int i = lane; i < nr * D; i += 32) {
    const int r = i / D, c = i % D;
    sc.xq[r * BAGEL_MAX_D + c] = e.xstar[(size_t)(b0 + r) * D + c];
  }
  __syncwarp();
}

template <int D, int R>
__device__ void epi_post(const EpiArgs& e, const int t, int b0, int nr, const float* th_s, float* buf,
                         float* scratch) {
  const int lane = threadIdx.x % 32;
  const int p = e.g.p, B = e.B, d = e.g.d;
  EpiScratch<D, R> sc(scratch);
  float* jv_t = e.tape_jv + (size_t)t * B * p * d;
  float* A_t = e.tape_A + (size_t)t * B * p * d;
  const bool policy_next = t + 1 < e.T;
  // lane = r * p * (D + 1) + m * (D + 1) + c: pass-2 partial of (row r, output m, column c)
  const int per_row = p * (D + 1);
  const int nl = nr * per_row;
  for (int base = 0; base < nl; base += 32) {
    const int li = base + lane;
    if (li < nl) {
      const int r = li / per_row, m = (li % per_row) / (D + 1), c = li % (D + 1);
      const int b = b0 + r;
      // sum of the S2 pass-2 partials in split order, 8 loads in flight
      float part = 0.0f;
      const float* src = e.P2 + ((size_t)m * B + b) * P2_LD + c;
      const size_t sstride = (size_t)p * B * P2_LD;
      for (int s0 = 0; s0 < e.S2; s0 += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = s0 + u < e.S2 ? __ldcg(src + (s0 + u) * sstride) : 0.0f;
#pragma unroll
        for (int u = 0; u < 8; ++u) part += v[u];
      }
      sc.psum[li] = part;
    }
  }
  __syncwarp();
  // J^v from the (r, m) row of sums [sum w k | sum w k (x*_c - X_c)]; tape A = J^mu + f J^v (reverse input)
  for (int li = lane; li < nl; li += 32) {
    const int r = li / per_row, m = (li % per_row) / (D + 1), c = li % (D + 1);
    if (c == 0) continue;
    const int b = b0 + r;
    // part = sum_n w_n k_n (x*_c - X_nc) (difference form)
    const float part = sc.psum[li];
    const float jv = 2.0f * e.g.ell2inv[m][c - 1] * part;
    const size_t o = ((size_t)b * p + m) * D + c - 1;
    jv_t[o] = jv;
    A_t[o] = fmaf(sc.f_s[r * p + m], jv, sc.jmu[r * BAGEL_MAX_P * BAGEL_MAX_D + m * D + c - 1]);
  }
  __syncwarp();
  const float* gb = e.goals + (size_t)b0 * p;
  if (lane < nr) e.G[b0 + lane] += (double)reward_fn(e.rw, &sc.xn_s[lane * p], gb + lane * p, p);
  if (!policy_next || e.policy_external) return;
  warp_policy<R>(e.P, p, th_s, sc.xn_s, gb, nr, buf, sc.us, e.tape_act + ((size_t)(t + 1) * B + b0) * e.P.act_ld);
  for (int i = lane; i < nr * D; i += 32) {
    const int r = i / D, c = i % D;
    e.xstar[(size_t)(b0 + r) * D + c] = c < p ? sc.xn_s[r * p + c] : sc.us[r * BAGEL_MAX_D + c - p];
  }
  __syncwarp();
}

template <int D, int R>
__device__ void epi_warp_rows(const EpiArgs& e, const int t, int b0, int nr, const float* th_s, float* buf,
                              float* scratch) {
  epi_pre<D, R>(e, t, b0, nr, scratch);
  epi_post<D, R>(e, t, b0, nr, th_s, buf, scratch);
}

}  // namespace rows
