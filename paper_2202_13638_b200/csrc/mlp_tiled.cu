// mlp_tiled.cu -- the policy MLP for WIDE policies (C3: 4-256-256-256-1, 133k parameters) as
// register-tiled fp32 GEMMs over blocks of trajectories.
//
// The warp-per-trajectory kernels (rollout.cu, policy_rows.cuh) keep theta in shared memory and
// are right for C1/C2/C4/C5 (<= 5k parameters).  With 256-wide layers each trajectory-step is
// ~133k FMAs and the weights no longer fit shared memory, so the work is organised as what it is
// there -- a dense [rows x in] x [in x out] contraction per layer:
//   k_mlp_fwd   one step of a1 (tanh hidden and output, R13/R14) for a block of
//               MLP_RB rows: phi(x, g) -> every layer -> u; writes the activation tape row and x*.
//   k_mlp_bwd   one step of the a9 adjoint recursion for a block of rows:
//               xs-bar = sum_m xbar_m A_t[m], delta_L = xs-bar[p:] (1 - u^2),
//               delta_{l-1} = (delta_l W_l) (1 - h_l^2) (delta tape written),
//               xbar_t = xbar_{t+1} + xs-bar[:p] + dphi/dx^T (delta_0 W_0) + d(r_t / B)/dx_t.
//   k_xbar_init xbar_T = (1/B) r(x_T) Q (x_T - g) / sigma_r^2.
// Thread tile: 4 rows x 8 output units (units o = lane + 32 j: conflict-free weight reads),
// weights streamed through shared memory in MLP_KC-deep chunks.  The same fp32 FMAs in a fixed
// order as the per-row kernels' reference semantics (results within fp32 rounding of them).
#include <algorithm>

#include "bagel_internal.h"
#include "policy_rows.cuh"

namespace {

constexpr int MLP_RB = 32;       // rows per CTA
constexpr int MLP_THREADS = 256; // 8 warps: warp w owns rows 4w .. 4w+3
constexpr int MLP_KC = 32;       // K depth of one staged weight chunk
constexpr int MLP_LD = BAGEL_MAX_WIDTH + 4;  // activation row stride (floats; 16-byte rows)
constexpr int MLP_WK = MLP_KC + 4;           // staged weight row stride: Ws[o][k], 16-byte aligned,
                                             // float4 reads by 8 consecutive units hit distinct banks

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// acc[r][j] (rows 4 ty + r, units tx + 32 j) = sum_k Hin[row][k] * W(k, unit), W(k, o) read as
// W[o * in + k] (forward: the layer's weight) or W[k * in + o] (backward: its transpose).  Weight
// chunks of MLP_KC k's are staged by cp.async into a double buffer (the next chunk is in flight
// while the current one is multiplied), 4 k's per float4 read of activations and weights.
template <bool FWD>
__device__ __forceinline__ void tile_gemm(const float* __restrict__ W, int K, int NO, int in, const float* Hin,
                                          float* Ws, float acc[4][8]) {
  const int tid = threadIdx.x, ty = tid / 32, tx = tid % 32;
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[r][j] = 0.0f;
  const int nch = (K + MLP_KC - 1) / MLP_KC;
  // 16-byte copies need every row start 16-byte aligned
  const bool vec16 = (in % 4 == 0) && ((reinterpret_cast<uintptr_t>(W) & 15) == 0);
  auto stage = [&](int c) {
    const int k0 = c * MLP_KC, kc = min(MLP_KC, K - k0);
    float* buf = Ws + (c & 1) * (BAGEL_MAX_WIDTH * MLP_WK);
    if (FWD && kc == MLP_KC && vec16) {
      // W[o][k] rows of 32 k as 8 x 16-byte copies: a warp covers 4 rows per instruction
      const int r4 = tx / 8, c4 = (tx % 8) * 4;
      for (int o = 4 * ty + r4; o < NO; o += 4 * (MLP_THREADS / 32))
        cp_async16(buf + o * MLP_WK + c4, W + (size_t)o * in + k0 + c4);
    } else if (FWD) {
      // W[o][k]: lane = k (coalesced 128-byte rows), warps step over o
      if (tx < kc)
        for (int o = ty; o < NO; o += MLP_THREADS / 32) cp_async4(buf + o * MLP_WK + tx, W + (size_t)o * in + k0 + tx);
    } else {
      // W[k][o]: thread = o (coalesced), loop over the chunk's k
      for (int o = tid; o < NO; o += MLP_THREADS)
        for (int kk = 0; kk < kc; ++kk) cp_async4(buf + o * MLP_WK + kk, W + (size_t)(k0 + kk) * in + o);
    }
    cp_async_commit();
  };
  __syncthreads();  // Hin written; the previous user of both weight buffers is done
  stage(0);
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) {
      stage(c + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();  // chunk c landed for every thread
    const int k0 = c * MLP_KC, kc = min(MLP_KC, K - k0);
    const float* buf = Ws + (c & 1) * (BAGEL_MAX_WIDTH * MLP_WK);
    int kk = 0;
    if (kc == MLP_KC) {
      // full chunk: compile-time trip count, fully unrolled so the next k-group's shared-memory
      // loads are issued ahead of the current FMAs (the kernel is shared-memory-latency bound at
      // 8 warps per SM); same FMA order as the general loop below
#pragma unroll
      for (int k4 = 0; k4 < MLP_KC; k4 += 4) {
        float4 h[4], w[8];
#pragma unroll
        for (int r = 0; r < 4; ++r) h[r] = *reinterpret_cast<const float4*>(Hin + (4 * ty + r) * MLP_LD + k0 + k4);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          w[j] = tx + 32 * j < NO ? *reinterpret_cast<const float4*>(buf + (tx + 32 * j) * MLP_WK + k4)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            acc[r][j] = fmaf(h[r].x, w[j].x, acc[r][j]);
            acc[r][j] = fmaf(h[r].y, w[j].y, acc[r][j]);
            acc[r][j] = fmaf(h[r].z, w[j].z, acc[r][j]);
            acc[r][j] = fmaf(h[r].w, w[j].w, acc[r][j]);
          }
      }
      kk = kc;
    }
    for (; kk + 4 <= kc; kk += 4) {
      float4 h[4], w[8];
#pragma unroll
      for (int r = 0; r < 4; ++r) h[r] = *reinterpret_cast<const float4*>(Hin + (4 * ty + r) * MLP_LD + k0 + kk);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        w[j] = tx + 32 * j < NO ? *reinterpret_cast<const float4*>(buf + (tx + 32 * j) * MLP_WK + kk)
                                : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          acc[r][j] = fmaf(h[r].x, w[j].x, acc[r][j]);
          acc[r][j] = fmaf(h[r].y, w[j].y, acc[r][j]);
          acc[r][j] = fmaf(h[r].z, w[j].z, acc[r][j]);
          acc[r][j] = fmaf(h[r].w, w[j].w, acc[r][j]);
        }
    }
    for (; kk < kc; ++kk) {
      float h[4], w[8];
#pragma unroll
      for (int r = 0; r < 4; ++r) h[r] = Hin[(4 * ty + r) * MLP_LD + k0 + kk];
#pragma unroll
      for (int j = 0; j < 8; ++j) w[j] = tx + 32 * j < NO ? buf[(tx + 32 * j) * MLP_WK + kk] : 0.0f;
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[r][j] = fmaf(h[r], w[j], acc[r][j]);
    }
    __syncthreads();  // done with buffer c & 1 before chunk c + 2 overwrites it
  }
}

// One policy evaluation for rows b0 .. b0 + MLP_RB - 1 at state x (B x p) and goals: the activation
// tape row (B x act_ld, may be null) and x* = [x, u] (B x D).
template <int D>
__global__ void __launch_bounds__(MLP_THREADS) k_mlp_fwd(PolicyDesc P, int p, const float* __restrict__ theta,
                                                         const float* __restrict__ x, const float* __restrict__ goals,
                                                         int B, float* __restrict__ act, float* __restrict__ xstar) {
  extern __shared__ __align__(16) float sm[];
  float* Ha = sm;                    // MLP_RB x MLP_LD
  float* Hb = Ha + MLP_RB * MLP_LD;  // MLP_RB x MLP_LD
  float* Ws = Hb + MLP_RB * MLP_LD;  // 2 x BAGEL_MAX_WIDTH x MLP_WK
  const int tid = threadIdx.x, ty = tid / 32, tx = tid % 32;
  const int b0 = blockIdx.x * MLP_RB;
  // phi = [x, g] or [x, g, g - x]
  const int n0 = P.sizes[0];
  for (int idx = tid; idx < MLP_RB * n0; idx += MLP_THREADS) {
    const int r = idx / n0, i = idx % n0, b = b0 + r;
    float v = 0.0f;
    if (b < B) {
      if (i < p) v = x[(size_t)b * p + i];
      else if (i < 2 * p) v = goals[(size_t)b * p + i - p];
      else v = goals[(size_t)b * p + i - 2 * p] - x[(size_t)b * p + i - 2 * p];
      if (act) act[(size_t)b * P.act_ld + i] = v;
    }
    Ha[r * MLP_LD + i] = v;
  }
  float* hin = Ha;
  float* hout = Hb;
  for (int l = 0; l < P.n_layers; ++l) {
    const int in = P.sizes[l], out = P.sizes[l + 1];
    float acc[4][8];
    tile_gemm<true>(theta + P.w_off[l], in, out, in, hin, Ws, acc);
    const float* bias = theta + P.b_off[l];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int o = tx + 32 * j;
      if (o >= out) continue;
      const float bb = __ldg(bias + o);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int rr = 4 * ty + r, b = b0 + rr;
        const float h = tanhf(acc[r][j] + bb);
        hout[rr * MLP_LD + o] = h;
        if (b < B) {
          if (act) act[(size_t)b * P.act_ld + P.aoff[l + 1] + o] = h;
          if (l == P.n_layers - 1) xstar[(size_t)b * D + p + o] = h;
        }
      }
    }
    float* tmp = hin;
    hin = hout;
    hout = tmp;
  }
  for (int idx = tid; idx < MLP_RB * p; idx += MLP_THREADS) {
    const int r = idx / p, c = idx % p, b = b0 + r;
    if (b < B) xstar[(size_t)b * D + c] = x[(size_t)b * p + c];
  }
}

__global__ void k_xbar_init(RewardDesc rw, int p, const float* __restrict__ xT, const float* __restrict__ goals,
                            int B, float invB, float* __restrict__ xbar) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  float q = 0.0f;
  for (int c = 0; c < p; ++c) {
    const float df = xT[(size_t)b * p + c] - goals[(size_t)b * p + c];
    q = fmaf(rw.Q[c] * df, df, q);
  }
  const float rr = expf(-q * rw.inv_two_sr2);
  const float inv_sr2 = 2.0f * rw.inv_two_sr2;
  for (int c = 0; c < p; ++c)
    xbar[(size_t)b * p + c] = invB * rr * rw.Q[c] * (xT[(size_t)b * p + c] - goals[(size_t)b * p + c]) * inv_sr2;
}

// One reverse step t for rows b0 .. b0 + MLP_RB - 1 (xbar: B x p, updated in place).
template <int D>
__global__ void __launch_bounds__(MLP_THREADS) k_mlp_bwd(PolicyDesc P, RewardDesc rw, int p,
                                                         const float* __restrict__ thetaT,  // per-layer W_l^T (k_transpose_theta)
                                                         const float* __restrict__ goals, int B,
                                                         const float* __restrict__ x_t, const float* __restrict__ A_t,
                                                         const float* __restrict__ act_t,
                                                         float* __restrict__ delta_t, float invB, float carry,
                                                         float* __restrict__ xbar) {
  extern __shared__ __align__(16) float sm[];
  float* Da = sm;                    // MLP_RB x MLP_LD: the current delta
  float* Db = Da + MLP_RB * MLP_LD;  // the next one
  float* Ws = Db + MLP_RB * MLP_LD;  // 2 x BAGEL_MAX_WIDTH x MLP_WK
  __shared__ float xs_s[MLP_RB][BAGEL_MAX_D];
  const int tid = threadIdx.x, ty = tid / 32, tx = tid % 32;
  const int b0 = blockIdx.x * MLP_RB;
  const int L = P.n_layers, q = P.sizes[L];
  // xs-bar_c = sum_m xbar_m A_t[m][c]
  for (int idx = tid; idx < MLP_RB * D; idx += MLP_THREADS) {
    const int r = idx / D, c = idx % D, b = b0 + r;
    float v = 0.0f;
    if (b < B)
      for (int m = 0; m < p; ++m) v = fmaf(xbar[(size_t)b * p + m], A_t[((size_t)b * p + m) * D + c], v);
    xs_s[r][c] = v;
  }
  __syncthreads();
  // delta_L = ubar (1 - u^2)
  for (int idx = tid; idx < MLP_RB * q; idx += MLP_THREADS) {
    const int r = idx / q, o = idx % q, b = b0 + r;
    float v = 0.0f;
    if (b < B) {
      const float u = act_t[(size_t)b * P.act_ld + P.aoff[L] + o];
      v = xs_s[r][p + o] * (1.0f - u * u);
    }
    Da[r * MLP_LD + o] = v;
  }
  float* dc = Da;
  float* dn = Db;
  for (int l = L - 1; l >= 0; --l) {
    const int in = P.sizes[l], out = P.sizes[l + 1];
    __syncthreads();
    for (int idx = tid; idx < MLP_RB * out; idx += MLP_THREADS) {
      const int r = idx / out, o = idx % out, b = b0 + r;
      if (b < B) delta_t[(size_t)b * P.d_ld + P.doff[l] + o] = dc[r * MLP_LD + o];
    }
    // hbar[r][i] = sum_o delta[r][o] W_l[o][i]
    float acc[4][8];
    // hbar = delta W_l = delta (W_l^T)^T: the forward-form GEMM on thetaT's W_l^T rows (in x out,
    // contiguous over o) -- coalesced, bank-conflict-free weight staging (the transposed staging
    // of theta was an 8-way shared-memory bank conflict per cp.async)
    tile_gemm<true>(thetaT + P.w_off[l], out, in, out, dc, Ws, acc);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = tx + 32 * j;
      if (i >= in) continue;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int rr = 4 * ty + r, b = b0 + rr;
        float v = acc[r][j];
        if (l > 0) {
          const float h = b < B ? act_t[(size_t)b * P.act_ld + P.aoff[l] + i] : 0.0f;
          v *= (1.0f - h * h);
        }
        dn[rr * MLP_LD + i] = v;
      }
    }
    float* tmp = dc;
    dc = dn;
    dn = tmp;
  }
  __syncthreads();
  // xbar_t = xbar_{t+1} + xs-bar[:p] + dphi/dx^T h0-bar + d(r_t / B)/dx_t
  const float inv_sr2 = 2.0f * rw.inv_two_sr2;
  for (int r = tid; r < MLP_RB; r += MLP_THREADS) {
    const int b = b0 + r;
    if (b >= B) continue;
    float qd = 0.0f;
    for (int c = 0; c < p; ++c) {
      const float df = x_t[(size_t)b * p + c] - goals[(size_t)b * p + c];
      qd = fmaf(rw.Q[c] * df, df, qd);
    }
    const float rr = expf(-qd * rw.inv_two_sr2);
    for (int c = 0; c < p; ++c) {
      float hb = dc[r * MLP_LD + c];
      if (P.phi_mode == 1) hb -= dc[r * MLP_LD + 2 * p + c];
      const float df = x_t[(size_t)b * p + c] - goals[(size_t)b * p + c];
      // carry = 1 for Delta targets, 0 for absolute targets (NEXT-4)
      xbar[(size_t)b * p + c] = carry * xbar[(size_t)b * p + c] + xs_s[r][c] + hb + invB * rr * rw.Q[c] * df * inv_sr2;
    }
  }
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

size_t mlp_smem() { return sizeof(float) * (2 * MLP_RB * MLP_LD + 2 * BAGEL_MAX_WIDTH * MLP_WK); }

void mlp_set_attrs() {
  static std::atomic<unsigned long long> devices{0};
  if (!bagel_first_on_device(devices)) return;
  for (int dv = 2; dv <= 8; ++dv) {
    DISPATCH_D(dv, ({
      bagel_set_smem_attr(k_mlp_fwd<D>, mlp_smem());
      bagel_set_smem_attr(k_mlp_bwd<D>, mlp_smem());
    }));
  }
}

}  // namespace

// Policy of step t for every row: x = tape_x[t]; writes tape_act[t] and x*.
int mlp_forward_step(const bagel_ctx* c, const float* theta, const float* goals, int B, int t, cudaStream_t st) {
  if (mlp_tc_enabled(c) && c->ws.mlp_wpk) return mlp_tc_forward_step(c, theta, goals, B, t, st);
  mlp_set_attrs();
  const Workspace& w = c->ws;
  const int p = c->gp.p;
  DISPATCH_D(c->gp.d, (k_mlp_fwd<D><<<cdiv(B, MLP_RB), MLP_THREADS, mlp_smem(), st>>>(
                          c->pol, p, theta, w.tape_x + (size_t)t * B * p, goals, B,
                          w.tape_act + (size_t)t * B * c->pol.act_ld, w.xstar)));
  return 1;
}

// The whole adjoint recursion, one launch per step (t = T-1 .. 0), plus the xbar_T initialisation.
int mlp_reverse(const bagel_ctx* c, const float* theta, const float* goals, int B, int T, long long B_global,
                cudaStream_t st) {
  mlp_set_attrs();
  const Workspace& w = c->ws;
  const int p = c->gp.p, d = c->gp.d;
  const float invB = (float)(1.0 / (double)B_global);
  k_xbar_init<<<cdiv(B, 128), 128, 0, st>>>(c->rw, p, w.tape_x + (size_t)T * B * p, goals, B, invB, w.xbar);
  const bool tcm = mlp_tc_enabled(c) && w.mlp_wpk;
  for (int t = T - 1; t >= 0; --t) {
    if (tcm) {
      mlp_tc_backward_step(c, goals, B, t, B_global, st);
      continue;
    }
    DISPATCH_D(d, (k_mlp_bwd<D><<<cdiv(B, MLP_RB), MLP_THREADS, mlp_smem(), st>>>(
                      c->pol, c->rw, p, w.thetaT, goals, B, w.tape_x + (size_t)t * B * p,
                      w.tape_A + (size_t)t * B * p * d, w.tape_act + (size_t)t * B * c->pol.act_ld,
                      w.tape_delta + (size_t)t * B * c->pol.d_ld, invB, c->gp.abs_target ? 0.0f : 1.0f, w.xbar)));
  }
  return 1 + T;
}
