// optim.cu -- the steps of Algorithm 1 around the hot path:
//   "Sample batch of initial states S_0^{b x d}" and goal-conditioned goals G
//   "sampled according to a distribution" (uniform within the data bounds),
//   and "Update theta via gradient descent" with Adam ("for which we will use
//   Adam [kingma2014adam]", lr 1e-2 P:151).
// Both are tiny next to the rollout; they run on the GPU so that one training iteration
// (sample -> rollout_cost_and_grad -> allreduce -> update) never round-trips theta or the
// batch through the host.
#include <math.h>
#include <stdint.h>

#include "bagel_internal.h"
#include "philox.cuh"

namespace {

// x[b][m] = lo_m + (hi_m - lo_m) u, u = u23(Philox4x32-10(key = seed, ctr = (traj_offset + b, 0,
// m >> 2, 2 + which))[m & 3]) -- the 4th counter word 2 (x0) / 3 (goals) keeps these streams
// disjoint from the rollout noise (word 0) and the Lanczos restarts (word 1, other key).
__global__ void k_sample_uniform(uint64_t seed, long long traj_offset, int B, int p, int which,
                                 const float* __restrict__ lo, const float* __restrict__ hi,
                                 float* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * p) return;
  const int b = i / p, m = i % p;
  const uint4 o = bagel_philox4x32_10(make_uint4((uint32_t)(traj_offset + b), 0u, (uint32_t)(m >> 2), 2u + (uint32_t)which),
                                      (uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32));
  const uint32_t w = (m & 3) == 0 ? o.x : ((m & 3) == 1 ? o.y : ((m & 3) == 2 ? o.z : o.w));
  const float u = bagel_u23(w);
  out[i] = lo[m] + (hi[m] - lo[m]) * u;
}

// Adam (Kingma & Ba, Algorithm 1, bias-corrected; the update of SPEC S:399-402):
//   m1 = b1 m1 + (1 - b1) g;  m2 = b2 m2 + (1 - b2) g^2;
//   theta -= lr (m1 / bc1) / (sqrt(m2 / bc2) + eps),  bc1 = 1 - b1^t, bc2 = 1 - b2^t.
// A non-finite gradient entry skips the whole update: one CTA checks every entry first,
// so the decision is the same for all parameters.  flag[0] = 1 when skipped, else 0.
constexpr int ADAM_THREADS = 1024;
__global__ void __launch_bounds__(ADAM_THREADS) k_adam(float* __restrict__ theta, const float* __restrict__ g,
                                                      float* __restrict__ m1, float* __restrict__ m2, int n,
                                                      float lr, float b1, float b2, float eps, float bc1, float bc2,
                                                      int* __restrict__ flag) {
  int mine = 0;
  for (int i = threadIdx.x; i < n; i += ADAM_THREADS) mine |= !isfinite(g[i]);
  if (__syncthreads_or(mine)) {
    if (threadIdx.x == 0) flag[0] = 1;
    return;
  }
  for (int i = threadIdx.x; i < n; i += ADAM_THREADS) {
    const float gi = g[i];
    const float a = b1 * m1[i] + (1.0f - b1) * gi;
    const float v = b2 * m2[i] + (1.0f - b2) * (gi * gi);
    m1[i] = a;
    m2[i] = v;
    theta[i] -= lr * (a / bc1) / (sqrtf(v / bc2) + eps);
  }
  if (threadIdx.x == 0) flag[0] = 0;
}

}  // namespace

int op_sample_uniform(uint64_t seed, long long traj_offset, int B, int p, int which, const float* lo, const float* hi,
                      float* out, cudaStream_t st) {
  const int n = B * p;
  if (n <= 0) return 0;
  k_sample_uniform<<<(n + 255) / 256, 256, 0, st>>>(seed, traj_offset, B, p, which, lo, hi, out);
  return 1;
}

int op_adam(float* theta, const float* g, float* m1, float* m2, int n, float lr, float b1, float b2, float eps,
            float bc1, float bc2, int* flag, cudaStream_t st) {
  k_adam<<<1, ADAM_THREADS, 0, st>>>(theta, g, m1, m2, n, lr, b1, b2, eps, bc1, bc2, flag);
  return 1;
}
