/*
 * bagel.h -- C ABI of libbagel.so, the B200 (sm_100a) hot path of BAGEL
 * (arXiv 2202.13638, "Policy optimization via Batch Automatic differentiation
 * of Gaussian process Evaluations using Lanczos variance estimates").
 *
 * Citations: PAPER.md line numbers are written P:NN, SPEC.md lines S:NN,
 * equations follow the paper's label order (Eq.1 dynamics ... Eq.11 batched
 * objective); readings are written R<n>.
 *
 * Conventions (all entry points):
 *   - return 0 on success, else one of the BAGEL_E_* codes below; no C++
 *     exception crosses the ABI; bagel_last_error() holds a one-line message
 *     naming the argument, its shape, or (step, row) for numerical faults.
 *   - array arguments are row-major float32 unless stated.  Pointers marked
 *     [dev|host] may be device memory or host memory (pageable or pinned);
 *     host buffers are staged through library-owned device memory with
 *     cudaMemcpyAsync on the context stream.  Pointers marked [dev] must be
 *     device memory, [host] host memory.
 *   - everything is enqueued on the stream given to bagel_create (or
 *     bagel_set_stream); calls that return host values synchronise it.
 *   - the library owns every internal buffer; caller buffers are never kept.
 *   - one context per GPU / rank; a context is not thread-safe.
 *   - no global state: two contexts never share memory.
 */
#ifndef BAGEL_H
#define BAGEL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bagel_ctx bagel_ctx;

/* Error classes mirror the specification's exit codes: 1 usage/config,
 * 2 numerical, 3 I/O or device.  BAGEL_E_STATE is a usage error (class 1). */
#define BAGEL_OK 0
#define BAGEL_E_ARG 1     /* bad argument value or shape                      */
#define BAGEL_E_NUMERIC 2 /* pivot <= 0, T not PD, non-finite state    */
#define BAGEL_E_CUDA 3    /* CUDA runtime failure or out of device memory      */
#define BAGEL_E_STATE 4   /* call out of order (no gp_load / cache / policy)   */

/* ------------------------------------------------------------------ context */

/* Create a context on CUDA device `device`.  `cuda_stream` is a cudaStream_t
 * (NULL = legacy default stream), typically torch.cuda.current_stream().
 * *out receives the context.  Errors: E_ARG (out NULL), E_CUDA. */
int bagel_create(bagel_ctx** out, int device, void* cuda_stream);

/* Free every library buffer (synchronises the context's stream first).  NULL is
 * accepted.  Errors: none (always BAGEL_OK). */
int bagel_destroy(bagel_ctx* ctx);

/* Re-target subsequent work to another stream on the same device (cuda_stream as
 * in bagel_create).  Errors: E_ARG for a NULL context. */
int bagel_set_stream(bagel_ctx* ctx, void* cuda_stream);

/* Message of the last failing call on this context ("" if none).  The pointer
 * stays valid until the next call on the context; "null context" for NULL.
 * Errors: none (returns a string). */
const char* bagel_last_error(const bagel_ctx* ctx);

/* SHA-256 (hex) of the sources, headers and compiler flags this library was
 * built from (paper_2202_13638_b200/build.py); the binding refuses a library
 * whose hash differs from the tree it is loaded from.  Errors: none. */
const char* bagel_build_hash(void);

/* --------------------------------------------------------------- GP model */

/* gp_load -- the GP transition model of Eq.1-4: one independent
 * SE-ARD GP per state dimension m = 0..p-1 (reading R7, R8), prior mean
 * 0 (R4), Delta targets (R6).
 *   X            [dev|host] N x d training inputs (x_k, u_k), d = p + q, already
 *                normalised by the caller (R22).
 *   y            [dev|host] N x p targets; column m is Delta x_m.
 *   lengthscales [dev|host] p x d, l_mc > 0; Lambda = diag(l^-2) (R1).
 *   outputscale  [dev|host] p, signal VARIANCE s_m = alpha^2 of Eq.4 (R2).
 *   noise        [dev|host] p, observation-noise VARIANCE sigma_n^2 >= 1e-8 (R3).
 * Copies everything into library memory; invalidates any LOVE cache.
 * Errors: E_ARG for N < 1, d < 2, p < 1, p >= d, p > 4, non-finite or
 * non-positive l or s, noise < 1e-8, non-finite X or y. */
int gp_load(bagel_ctx* ctx, const float* X, const float* y, int N, int d, int p,
            const float* lengthscales, const float* outputscale, const float* noise);

/* gp_target_mode -- what the GPs' targets y were ("each m-th GP can model
 * the one-step forward dynamics of one output y = x_{k+1} or the discrete
 * difference y = Delta x = x_{k+1} - x_k"):
 *   absolute = 0 (default, reading R6): Delta targets, x' = x + mu + sigma eps;
 *   absolute = 1 (NEXT-4): absolute targets, x' = mu + sigma eps, and the
 *   reverse pass drops the identity path dx'/dx = I.  The GP step then runs on
 *   the round-to-nearest CUDA-core kernels: with y = x_{k+1} the prior variance
 *   is the states' variance and v = s - ||z||^2 cancels to ~1e-6 s, below what
 *   the tensor core's truncating TMEM accumulation resolves (R38).
 * Applies to every later rollout / trace call; kept across gp_load.
 * Errors: E_ARG if absolute is not 0 or 1. */
int gp_target_mode(bagel_ctx* ctx, int absolute);

/* love_cache_build -- the one-time LOVE cache ("one-time caching
 * operation ... ~0.6s"), for every output m, in float64 on the GPU:
 *   alpha_m = Khat_m^-1 y_m by blocked Cholesky (Khat = K + sigma_n^2 I; R21),
 *   Lanczos(Khat_m, q1 = y_m/||y_m||, `rank` steps, classical Gram-Schmidt
 *   twice, Philox restart on breakdown; R20) -> Q, T;  R_m = L_T^-1 Q^T;
 *   then packs V_m = s_m [alpha_m | alpha_m o X | R_m^T] for the hot path.
 * Synchronous.  seconds_out [host, nullable] receives the wall time.
 * Errors: E_STATE without gp_load; E_ARG for rank < 1 or rank > N or rank >
 * 8192; E_NUMERIC if a Cholesky pivot <= 0 (message carries the pivot index)
 * or T is not positive definite; E_CUDA (incl. out of memory). */
int love_cache_build(bagel_ctx* ctx, int rank, double* seconds_out);

/* exact_cache_build -- the exact-GP variant of the cache (SURVEY.md §8(f)
 * NEXT-3; the paper's "AutoDiff on exact GPs" baseline): per
 * output, in float64 on the GPU, L = chol(Khat), alpha = Khat^-1 y and
 * R = L^-1 (N x N, blocked triangular inverse), installed as a rank-N cache,
 * so every rollout / predict call afterwards uses the exact Eq.3 variance
 * k** - ||L^-1 k||^2 instead of the LOVE estimate (K^-1 = R^T R exactly).
 * Synchronous; seconds_out [host, nullable].  Replaces any LOVE cache.
 * Errors: E_STATE without gp_load; E_ARG if N > 8192 (the largest rank the
 * cache accepts; the paper's exact baseline is n = 2200); E_NUMERIC if a Cholesky pivot <= 0; E_CUDA. */
int exact_cache_build(bagel_ctx* ctx, double* seconds_out);

/* ------------------------------------------------------- policy / reward */

/* policy_configure -- tanh MLP policy u = pi_theta(x, g) (P:104, P:129,
 * P:149 "bounded in [-1,1] using a saturating function"; R13).
 *   sizes [host] n_sizes = L + 1 layer widths (in, h1, ..., q).  in = 2p selects
 *   phi = [x, g], in = 3p selects phi = [x, g, g - x] (R14).  Last width = q = d - p.
 * theta layout (rollout_cost_and_grad): per layer l, W_l [out x in] row-major
 * then b_l [out] (PyTorch nn.Sequential(Linear, Tanh, ...) order).
 * Errors: E_STATE without gp_load; E_ARG for n_sizes < 2, a width < 1 or > 256,
 * in not in {2p, 3p}, q != d - p. */
int policy_configure(bagel_ctx* ctx, const int* sizes, int n_sizes);

/* reward_configure -- Eq.8: r = exp(-(1/(2 sigma_r^2)) (x-g)^T Q (x-g)).
 *   Q_diag [host] p non-negative weights (default diag{10, 0.1} for p = 2, P:149;
 *   R12 for other p); sigma_r > 0 (default 1, R11).
 * Errors: E_STATE without gp_load; E_ARG for negative/non-finite Q or sigma_r <= 0. */
int reward_configure(bagel_ctx* ctx, const float* Q_diag, float sigma_r);

/* ------------------------------------------------------------ hot path */

/* rollout_cost_and_grad -- one BAGEL iteration's forward + backward pass
 * (Alg.1 lines P:101-109, Eq.9-11):
 *   G_b = r(x0_b, g_b);  for t = 0..T-1: u = pi(x_t, g); x* = [x_t, u];
 *   mu_m = k(x*,X) alpha_m (Eq.2), v_m = s_m - ||R_m k(x*,X)||^2 (LOVE, Eq.3),
 *   x_{t+1,m} = x_{t,m} + mu_m + sqrt(max(v_m, 1e-12)) eps_{b,t,m} (Eq.9-10, R6, R19),
 *   G_b += r(x_{t+1}, g_b);
 *   L = -(1/B_global) sum_b G_b (R9), and dL/dtheta by reverse mode
 *   through the whole horizon (pathwise, R18).
 *   eps_{b,t,m} = BoxMuller(Philox4x32-10(key = (seed lo, seed hi),
 *   ctr = (traj_offset + b, t, m >> 2, 0)))[m & 3].
 * Arguments:
 *   policy_params [dev|host] |theta| floats, layout of policy_configure.
 *   x0, goals     [dev|host] B x p (normalised units; goals are constants, R23).
 *   B >= 1 trajectories on this rank; T >= 0 steps.
 *   seed          64-bit Philox key for this iteration (fresh per iteration, R17).
 *   traj_offset   global id of row 0 (rank r of G: r*B/G, P:142 batches sharded).
 *   B_global      the 1/b of Eq.11 (total trajectories over all ranks), >= B.
 *   mean_cost     [host] receives this rank's share of L (already / B_global).
 *   grad          [dev|host] |theta| floats, overwritten with this rank's dL/dtheta.
 * Synchronises the stream before returning.  T = 0 returns -mean r(x0) share
 * and a zero gradient.
 * Errors: E_STATE without cache or policy; E_ARG (B < 1, T < 0, B_global < B,
 * B or T beyond the workspace limits); E_NUMERIC on a non-finite state (message
 * "step t, row b"); E_CUDA. */
int rollout_cost_and_grad(bagel_ctx* ctx, const float* policy_params, const float* x0,
                          const float* goals, int B, int T, uint64_t seed, long long traj_offset,
                          long long B_global, double* mean_cost, float* grad);

/* ------------------------------------- Algorithm 1 around the hot path (NEXT-2) */

/* bagel_sample_states -- "Sample batch of initial states S_0" (Alg.1) and
 * goal-conditioned goals "sampled according to a distribution", uniform
 * within the data bounds:
 *   out[b][m] = lo[m] + (hi[m] - lo[m]) u,  u = ((o >> 9) + 0.5) 2^-23 (R29),
 *   o = Philox4x32-10(key = (seed lo, seed hi),
 *                     ctr = (traj_offset + b, 0, m >> 2, 2 + which))[m & 3].
 *   which = 0 draws S_0, 1 draws G (disjoint streams; the rollout noise uses ctr
 *   word 3 = 0).  lo, hi [host] p floats; out [dev] B x p.  Asynchronous.
 * Errors: E_ARG (B < 1, p not in [1, 4], which not in {0, 1}, lo > hi or
 * non-finite bounds, out not device memory, traj_offset + B >= 2^32). */
int bagel_sample_states(bagel_ctx* ctx, uint64_t seed, long long traj_offset, int B, int p, int which,
                        const float* lo, const float* hi, float* out);

/* policy_adam_step -- "Update theta via gradient descent" (Alg.1) with
 * Adam ("for which we will use Adam"; lr 1e-2), bias-corrected
 * (Kingma & Ba Alg.1), elementwise on n floats:
 *   m1 = b1 m1 + (1 - b1) g;  m2 = b2 m2 + (1 - b2) g^2;
 *   params -= lr (m1 / (1 - b1^step)) / (sqrt(m2 / (1 - b2^step)) + eps).
 * params, m1, m2 [dev] n floats updated in place (m1 = m2 = 0 before step 1);
 * grad [dev] n floats; step >= 1 counts updates (the caller increments it).
 * If any grad entry is non-finite, nothing is updated and *skipped = 1.
 * skipped [host, nullable]: when non-NULL the call synchronises the stream and
 * reports; when NULL the update is only enqueued.
 * Errors: E_ARG (n < 1, step < 1, lr < 0, beta outside [0, 1), eps <= 0,
 * non-device arrays). */
int policy_adam_step(bagel_ctx* ctx, float* params, const float* grad, float* m1, float* m2, int n,
                     long long step, float lr, float beta1, float beta2, float eps, int* skipped);

/* gp_log_marginal_likelihood -- "Learn GP transition dynamics using D" (Alg.1
 * P:98): the exact log marginal likelihood of output GP m and its gradient in
 * the log-hyperparameters (Eq.5-6, reading R33 -- Eq.5 is written up
 * to a factor 2 and a constant, Eq.6 is garbled):
 *   log p(y_m | X, phi) = -1/2 y^T Khat^-1 y - 1/2 log|Khat| - N/2 log(2 pi),
 *   d/dphi_j = 1/2 tr((alpha alpha^T - Khat^-1) dKhat/dphi_j),  alpha = Khat^-1 y,
 * phi = [log l_1 .. log l_d, log s, log sigma_n^2] ("Adam on
 * log-parameters"), computed in float64 on the GPU (Cholesky, triangular
 * inverse, Khat^-1 formed tile by tile inside the gradient reduction).
 *   m        output index in [0, p); uses the X and column m of y of gp_load.
 *   log_hyp  [host, nullable] d + 2 doubles; NULL = the hyperparameters of gp_load.
 *   mll      [host] receives the log marginal likelihood.
 *   grad     [host, nullable] d + 2 doubles; NULL skips the gradient (O(N^3) less).
 * Synchronous.  Workspace 2 N^2 float64 (kept for the next call at the same N).
 * Does not change the loaded model or its LOVE cache.
 * Errors: E_STATE without gp_load; E_ARG (m out of range, non-finite log_hyp,
 * noise < 1e-8, workspace > 120 GB); E_NUMERIC if a Cholesky pivot <= 0; E_CUDA. */
int gp_log_marginal_likelihood(bagel_ctx* ctx, int m, const double* log_hyp, double* mll, double* grad);

/* gp_log_marginal_likelihood_bbmm -- the same quantities estimated the way the
 * paper's GP library does it at scale (GPyTorch; "blackbox matrix-matrix"
 * inference, reading R39), in float64 on the GPU without any factorisation:
 *   one batched conjugate-gradient run of exactly n_iter iterations (no
 *   preconditioner) on Khat [u_0 .. u_t] = [y z_1 .. z_t], z_i Rademacher with
 *   z_i[n] = sign bit of Philox4x32-10(key = (seed lo, seed hi),
 *   ctr = (i, n >> 2, 0x4242424D, 4))[n & 3] (set -> -1, clear -> +1), i = 0..t-1;
 *   log|Khat| ~ (1/t) sum_i N e_1^T log(T_i) e_1 with T_i the Lanczos tridiagonal
 *   of probe i from its CG coefficients (stochastic Lanczos quadrature);
 *   y^T Khat^-1 y ~ y^T u_0;  tr(Khat^-1 dK) ~ (1/t) sum_i u_i^T dK z_i;
 *   mll = -1/2 y^T u_0 - 1/2 log|Khat| - N/2 log(2 pi);
 *   grad_j = 1/2 u_0^T dK_j u_0 - 1/2 (1/t) sum_i u_i^T dK_j z_i.
 * A column whose residual reaches exactly 0 stops early (its T_i is smaller).
 * precond_rank k in [0, min(N, 64)]: k > 0 adds GPyTorch's preconditioner (reading
 * R40): a greedy rank-k pivoted Cholesky L L^T of Khat - sn2 I (pivot = the largest
 * residual diagonal, lowest index on ties; it stops early at a non-positive
 * residual), P = L L^T + sn2 I applied by Woodbury; probes become Gaussian,
 * z_i = L g_i[0..k) + sqrt(sn2) g_i[k..k+N), g_i[j] = Box-Muller word j & 3 of
 * Philox4x32-10(key = seed, ctr = (i, j >> 2, 0x4242424E, 5)); the CG is
 * preconditioned, log|Khat| ~ log|P| + (1/t) sum_i (z_i^T P^-1 z_i) e_1^T
 * log(T_i) e_1 and tr(Khat^-1 dK) ~ (1/t) sum_i u_i^T dK P^-1 z_i.
 *   m, log_hyp, mll, grad  as gp_log_marginal_likelihood.
 *   n_probes t in [1, 16];  n_iter J in [1, min(N, 4096)];  seed  probe stream.
 *   logdet   [host, nullable] receives the log-det estimate.
 * Synchronous.  Cost O(J N^2) for the solves plus O(t N^2 d) for the gradient;
 * workspace N^2 + 5 (t + 1) N float64 (kept for later calls).  Deterministic:
 * every reduction runs in a fixed order.  Does not change the loaded model.
 * Errors: E_STATE without gp_load; E_ARG (m, t, J, k out of range, non-finite
 * log_hyp, noise < 1e-8, workspace > 120 GB); E_NUMERIC when the estimate is
 * non-finite (Khat too ill-conditioned for J iterations) or sn2 I + L^T L is not
 * positive definite; E_CUDA. */
int gp_log_marginal_likelihood_bbmm(bagel_ctx* ctx, int m, const double* log_hyp, int n_probes, int n_iter,
                                    int precond_rank, uint64_t seed, double* mll, double* grad, double* logdet);

/* Number of kernel launches the last rollout_cost_and_grad enqueued: launches [host]
 * (the bench's gpu_launches count).  Errors: E_ARG for NULL pointers. */
int bagel_last_launch_count(const bagel_ctx* ctx, int* launches);

/* Per-kernel device timing for the roofline report (bench.py).  While enabled,
 * every hot-path launch is bracketed by cudaEvents on the context stream and
 * its duration is accumulated per kernel class:
 *   0 gp_pass1 (a2+a3 contraction), 1 gp_reduce1 (a4), 2 gp_pass2 (a5),
 *   3 step_epilogue (a6-a8 + next a1), 4 init (a1 + a7 at t = 0),
 *   5 reverse (a9: the adjoint recursion), 6 reduce (a10), 7 theta_grad (a9: the
 *   parameter-gradient contraction over the adjoint tape).
 * bagel_profile(ctx, 1) enables and clears, bagel_profile(ctx, 0) disables.
 * bagel_profile_get: total_ms [host] and launches [host] of class `kernel`
 * since the last enable (synchronises the stream).  Errors: E_ARG. */
#define BAGEL_PROFILE_CLASSES 8
int bagel_profile(bagel_ctx* ctx, int enable);
int bagel_profile_get(bagel_ctx* ctx, int kernel, double* total_ms, long long* launches);

/* ------------------------------------------------------- test-only exports */

/* One GP query per row of xstar [dev] M x d with the LOVE variance and input
 * Jacobians (Appendix B of SURVEY.md; the autodiff of Eq.2-3):
 *   mean, var [dev] M x p; dmean, dvar [dev] M x p x d (dvar uses the unclamped v).
 * Runs the same kernels as the rollout's GP step.  Errors: E_STATE without a cache;
 * E_ARG (NULL pointers, M < 1); E_CUDA. */
int bagel_gp_predict(bagel_ctx* ctx, const float* xstar, int M, float* mean, float* var,
                     float* dmean, float* dvar);

/* Forward rollout with per-step traces (same kernels as rollout_cost_and_grad,
 * Alg.1; Eq.9-10):
 *   x [dev] (T+1) x B x p states, mu / var [dev] T x B x p GP moments,
 *   ret [dev] B returns G_b.  Any trace pointer may be NULL.  Other arguments and
 *   errors as rollout_cost_and_grad (E_STATE, E_ARG, E_NUMERIC, E_CUDA). */
int bagel_rollout_trace(bagel_ctx* ctx, const float* policy_params, const float* x0,
                        const float* goals, int B, int T, uint64_t seed, long long traj_offset,
                        float* x, float* mu, float* var, float* ret);

/* Raw Philox4x32-10 (Salmon et al., SC'11; the generator of reading R29 / DESIGN.md
 * "Philox"): ctr [dev] n x 4 u32, key [host] 2 u32, out [dev] n x 4 u32.
 * Synchronous.  Errors: E_ARG for NULL pointers or n < 0; E_CUDA. */
int bagel_philox4x32_10(bagel_ctx* ctx, const uint32_t* ctr, const uint32_t* key, int n,
                        uint32_t* out);

/* Rollout noise as the rollout draws it (Eq.9, reparameterised, R18): out [dev]
 * T x B x p floats, out[t][b][m] = eps_{traj_offset + b, t, m} for `seed`.
 * Synchronous.  Errors: E_ARG (out NULL, B < 1, T < 1, p not in [1, 4]); E_CUDA. */
int bagel_philox_normals(bagel_ctx* ctx, uint64_t seed, long long traj_offset, int B, int T,
                         int p, float* out);

/* LOVE cache of output m as float64 device arrays: alpha [dev] N,
 * R [dev] rank x N.  bagel_cache_rank returns the rank k (0 if no cache) in
 * rank [host].  Errors: E_ARG (NULL pointers, m out of range); E_STATE without a
 * cache; E_CUDA. */
int bagel_cache_rank(const bagel_ctx* ctx, int* rank);
int bagel_cache_get(bagel_ctx* ctx, int m, double* alpha, double* R);

/* Install an externally computed cache (isolates hot-path parity from the
 * cache build).  Call once per output m = 0..p-1 with the same rank; the
 * packed hot-path operand V_m is rebuilt for that output.
 *   alpha [dev] N float64, R [dev] rank x N float64.
 * Errors: E_STATE without gp_load; E_ARG for m out of range, rank change. */
int bagel_cache_set(bagel_ctx* ctx, int m, int rank, const double* alpha, const double* R);

/* GP-step implementation selector (bench / A-B parity tests):
 *   1 (default) tcgen05 tensor-core kernels (csrc/gp_step_tc.cu),
 *   0 the v0 CUDA-core FFMA kernels (csrc/gp_step.cu), kept as a reference.
 * bagel_get_gp_kernel reports the path the next call will take (1 unless
 * absolute targets are selected, gp_target_mode).  Errors: E_ARG. */
int bagel_set_gp_kernel(bagel_ctx* ctx, int version);
int bagel_get_gp_kernel(const bagel_ctx* ctx, int* version);

/* Tensor-core probe: one CTA computes D[128 x N] = A[128 x K] . B[N x K]^T with
 * fp16 operands (tcgen05.mma kind::f16, fp32 accumulate in TMEM).  B is a [dev]
 * fp16 array in the canonical no-swizzle K-major packing of csrc/tc.cuh
 * (element (r, k) at ((r/8)(K/8) + k/8) 64 + (r%8) 8 + k%8).  mode 0: A [dev]
 * in the same packing, read from shared memory; mode 1: A [dev] row-major
 * 128 x K, placed in TMEM and read by the TS form of tcgen05.mma.
 * D [dev] row-major 128 x N float32.  N in {16, 32, ..., 256}, K in {16, 32, ...},
 * (128 + N) K 2 bytes <= 200 KB.  Errors: E_ARG, E_CUDA. */
int bagel_tc_selftest(bagel_ctx* ctx, const void* A, const void* B, int N, int K, int mode, float* D);

/* CTA-pair probe (tcgen05.mma.cta_group::2): a 2-CTA cluster computes D[256 x N] = A[256 x K] .
 * B[N x K]^T, A and B [dev] fp16 given as two halves each in the canonical packing above (A rows
 * 0-127 | 128-255; B rows 0..N/2-1 | N/2..N-1), D [dev] 256 x N fp32 row-major.  mode 0: A from
 * shared memory; mode 1: A from each CTA's TMEM (A [dev] then also carries the 256 x K rows
 * row-major after the packed halves).  N in {32, 64, ..., 256}, (128 + N/2) K 2 bytes <= 200 KB.
 * Synchronous.  Errors: E_ARG, E_CUDA. */
int bagel_tc_selftest2(bagel_ctx* ctx, const void* A, const void* B, int N, int K, int mode, float* D);

/* Debug copy of an internal per-step buffer into host memory dst [host] (bytes <= its size):
 * 0 pass-1 mean-column partials, 1 pass-1 z partials, 2 pass-2 partials, 3 step means.
 * Layouts are internal (csrc/gp_step_tc.cu).  Errors: E_ARG. */
int bagel_debug_buffer(bagel_ctx* ctx, int which, void* dst, size_t bytes);

/* Enable (1) / disable (0) per-CTA %globaltimer event stamps of the tensor-core GP kernels
 * (16 per CTA, up to 4096 CTAs; read with bagel_debug_buffer 4 = pass 1, 5 = pass 2).
 * Errors: E_CUDA (stamp buffer allocation). */
int bagel_debug_trace(bagel_ctx* ctx, int enable);

/* Tensor-core issue-rate microbenchmark: `ctas` CTAs (one per SM) each issue `iters`
 * back-to-back tcgen05.mma (M = 128, N, K = 16; mode 0: A from shared memory, 1: A from
 * TMEM) and write the elapsed SM cycles to cycles [dev] (ctas int64).  mode 64: `ctas` CTA
 * pairs (<= 74), each leader issuing tcgen05.mma.cta_group::2 (M = 256, N, both operands from
 * shared memory; 65: A from TMEM).  Errors: E_ARG. */
int bagel_tc_bench(bagel_ctx* ctx, int N, int iters, int mode, int ctas, long long* cycles);

#ifdef __cplusplus
}
#endif

#endif /* BAGEL_H */
