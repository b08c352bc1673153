// bagel_internal.h -- context layout and launcher prototypes shared by the
// CUDA translation units of libbagel.so.  Not part of the ABI (see include/bagel.h).
#pragma once

#include <cuda_runtime.h>
#include <atomic>
#include <stdint.h>

#include <string>
#include <vector>

#define BAGEL_MAX_P 4        // one Philox call per (b, t) carries the p <= 4 normals
#define BAGEL_MAX_D 8        // d = p + q <= 8
#define BAGEL_MAX_WIDTH 256  // widest MLP layer
#define BAGEL_MAX_LAYERS 8
#define BAGEL_MAX_RANK 8192  // tensor-core kernels tile any k (256-column z tiles, 256-j pass-2 tiles)
#define BAGEL_VAR_FLOOR 1e-12f
#define BAGEL_BARRIER_TIMEOUT (-2)  // err_flag value: a grid barrier timed out (grid not co-resident)  // S:252 clamp (reading R19)

// sqrt(0.5 * log2(e)): x_hat = x * KAPPA / l so that exp(-1/2 sum (dx/l)^2) = exp2(-||x_hat - X_hat||^2)
#define BAGEL_KAPPA 0.84932180028801907f

struct PolicyDesc {
  int n_layers;
  int sizes[BAGEL_MAX_LAYERS + 1];
  int w_off[BAGEL_MAX_LAYERS];  // offset of W_l in theta
  int b_off[BAGEL_MAX_LAYERS];  // offset of b_l in theta
  int phi_mode;                 // 0: [x, g]; 1: [x, g, g - x]
  int n_params;
  int max_width;
  int act_total;                // sum of all layer widths (activations per row)
  // reverse-pass tapes: every segment padded to a multiple of 4 floats (16-byte aligned rows)
  int aoff[BAGEL_MAX_LAYERS + 1];  // activation tape: offset of layer l's activations (l = 0: phi)
  int act_ld;                      // activation tape row length
  int doff[BAGEL_MAX_LAYERS];      // adjoint tape: offset of delta_l (layer l's outputs)
  int d_ld;                        // adjoint tape row length
};

struct RewardDesc {
  float Q[BAGEL_MAX_P];
  float inv_two_sr2;  // 1 / (2 sigma_r^2)
};

// Problem geometry of one GP step, passed by value to kernels.
struct GpDesc {
  int N, d, p, k;
  int C;     // 1 + d + k columns of V = [s alpha | s alpha o X | s R^T]
  int Cld;   // leading dimension of V rows (C rounded up to the column tile)
  float ell2inv[BAGEL_MAX_P][BAGEL_MAX_D];  // 1 / l_mc^2
  float qscale[BAGEL_MAX_P][BAGEL_MAX_D];   // KAPPA / l_mc
  float s[BAGEL_MAX_P];
  int abs_target;  // 0: Delta targets x' = x + f (R6, default); 1: absolute targets x' = f (NEXT-4)
};

// Arguments of the step epilogue (policy_rows.cuh epi_warp_rows) for step t of T: pass-2
// partial sums -> J^v, eps, x' = x + mu + sigma eps, G += r, tapes (x, J^v, A, activations),
// next action.  Tape pointers are the bases of the whole rollout; step t's rows are derived.
struct EpiArgs {
  PolicyDesc P;
  RewardDesc rw;
  GpDesc g;
  const float* thetaT;
  const float* goals;
  int B, t, T, S2;
  const float* P2;       // S2 x p x B x (1 + MAX_D)
  const float* mu;       // p x B
  const float* var;      // p x B
  float* tape_x;         // (T + 1) x B x p
  const float* tape_sig; // T x B x p (negative: clamped)
  float* tape_jv;        // T x B x p x d
  const float* tape_jmu; // T x B x p x d
  float* tape_A;         // T x B x p x d
  float* tape_act;       // T x B x act_ld
  double* G;             // B
  float* xstar;          // B x d (read: this step's query; written: the next one)
  uint64_t seed;
  long long traj_offset;
  int* err_flag;
  float* trace_mu;       // nullable, T x B x p
  float* trace_var;      // nullable, T x B x p
  int policy_external;   // 1: the next action is computed by mlp_forward_step (wide policies)
};

// Tensor-core (tcgen05) path state: packed operand tiles (cache-build time) and
// its per-step buffers (see gp_step_tc.cu for layouts).
struct TcState {
  uint8_t* tiles1 = nullptr;  // p x t1_stride bytes
  uint8_t* tiles2 = nullptr;  // p x t2_stride bytes
  size_t t1_stride = 0, t2_stride = 0;
  float* colscale = nullptr;      // p x k  (2^e_j)
  float* colscale_inv = nullptr;  // p x k  (2^-e_j)
  float* qscale = nullptr;        // p x MAX_D
  float* P1z = nullptr;           // S1 x p x nct x NZ x B
  float* P1h = nullptr;           // S1 x p x B x (1 + d)
  uint8_t* Zp = nullptr;          // packed pass-2 A operand
  float* zrow_inv = nullptr;      // p x B
  unsigned long long* gbar = nullptr;  // grid-barrier counter of the fused pass 1 (monotonic)
  unsigned long long* dbg1 = nullptr;  // optional per-CTA event stamps (bagel_debug_trace)
  unsigned long long* dbg2 = nullptr;
  unsigned long long* dbg3 = nullptr;  // step epilogue (t = 50 of a rollout)
  double* zz_part = nullptr;      // p x (k/32) x B partial ||z||^2
  float* zmax_part = nullptr;     // p x (k/32) x B partial max|z|
};

struct Workspace {
  int B = 0, T = 0;         // capacity
  int S1 = 0, S2 = 0;       // N-splits of pass 1 / pass 2 (v0 FFMA path)
  int S1tc = 0, S2tc = 0, tps1 = 0, tps2 = 0;  // tcgen05 path splits / tiles per split
  int p1_fused = 0;  // pass 1 launched cooperatively with reduce 1 fused in (k_p1_tc<D, true>)
  int S2eff = 0;            // number of pass-2 partial slices the epilogue sums
  float* xstar = nullptr;   // B x d
  float* theta_colmax = nullptr;  // theta_tc.cu: per K block, max |delta| per tape column + max |phi|
  size_t theta_colmax_cap = 0;
  float* P1 = nullptr;      // S1 x p x B x Cld partial [mu | k a X | z]
  float* Z = nullptr;       // p x B x k
  float* P2 = nullptr;      // S2 x p x B x (1 + MAX_D) partial [sum w k | sum w k X_c]
  float* mu = nullptr;      // p x B  (step moments)
  float* var = nullptr;     // p x B
  // tape (a8): x (T+1) x B x p, sig T x B x p (negative = clamped), Jmu / Jv T x B x p x d
  float* tape_x = nullptr;
  float* tape_sig = nullptr;
  float* tape_jmu = nullptr;
  float* tape_jv = nullptr;
  // reverse-pass tape: A = J^mu + (eps / 2 sigma) J^v  T x B x p x d; every policy activation
  // T x B x act_total; the adjoints delta_l T x B x (act_total - sizes[0])
  float* tape_A = nullptr;
  float* tape_act = nullptr;
  float* tape_delta = nullptr;
  size_t tape_pol_cap = 0;      // rows (T x B) the activation / delta tapes hold
  float* xbar = nullptr;        // B x p adjoint state (tiled reverse of wide policies)
  double* G = nullptr;      // B returns
  float* theta_part = nullptr;  // nblk x n_params reverse partials
  int theta_part_cap = 0;
  float* grad_tmp = nullptr;    // n_params (host-grad staging)
  float* thetaT = nullptr;      // n_params: per-layer transposed weights (coalesced policy forward)
  double* cost_dev = nullptr;   // 1
  int* err_flag = nullptr;      // first (t * B + b) + 1 with a non-finite state, else 0
  // host staging of [dev|host] inputs
  float* stage = nullptr;
  size_t stage_cap = 0;
  uint8_t* mlp_wpk = nullptr;   // wide policies: packed hi/lo weight chunks of the tensor-core MLP (mlp_tc.cu)
  size_t mlp_wpk_cap = 0;
};

struct bagel_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  // GP data (gp_load)
  int N = 0, d = 0, p = 0;
  float* X = nullptr;   // N x d
  float* Y = nullptr;   // N x p
  std::vector<float> ell, s, noise;
  // LOVE cache
  int k = 0;
  std::vector<int> cache_ok;
  double* alpha64 = nullptr;  // p x N
  double* R64 = nullptr;      // p x k x N
  float* V = nullptr;         // p x N x Cld (fp32 packed hot-path operand)
  float* Xs = nullptr;        // p x N x d   (X * KAPPA / l)
  GpDesc gp{};
  // policy / reward
  bool policy_ok = false, reward_ok = false;
  PolicyDesc pol{};
  RewardDesc rw{};
  Workspace ws;
  TcState tcs;
  int* op_flag = nullptr;     // Adam skip flag (device int, optim.cu)
  float* op_bounds = nullptr; // 2 x MAX_P sampling bounds (lo | hi)
  double* mll_K = nullptr;    // N x N: Khat, then its Cholesky factor (mll.cu)
  double* mll_Li = nullptr;   // N x N: L^-1
  double* mll_vec = nullptr;  // alpha (N) | scalars (2) | grad (MAX_D + 2) | tile partials
  int mll_N = 0;
  double* bbmm_ws = nullptr;  // BBMM workspace (bbmm.cu): Khat | rhs, u, r, p, q columns | CG coefficients | partials
  size_t bbmm_ws_n = 0;
  int* bbmm_its = nullptr;     // CG iterations per column
  int abs_target = 0;         // gp_target_mode
  int gp_kernel = 1;  // 1: tcgen05 path (default), 0: v0 FFMA path (reference / A-B tests)
  int last_launches = 0;
  int num_sms = 148;
  // per-kernel-class event timing (bagel_profile)
  struct ProfEvent {
    cudaEvent_t a, b;
    int cls;
  };
  bool prof_on = false;
  std::vector<ProfEvent> prof_pending;
  std::vector<cudaEvent_t> prof_pool;
  double prof_ms[8] = {};
  long long prof_n[8] = {};
};

// True the first time it is called for the current device: kernel attributes such as the
// dynamic shared-memory opt-in are set per device, so a process driving several GPUs (one
// context each) sets them once on every device, not once per process.
inline bool bagel_first_on_device(std::atomic<unsigned long long>& devices) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  return !(devices.fetch_or(bit) & bit);
}

// Opt a kernel into the largest dynamic shared memory the device allows next to its
// static shared memory (capped at `want`); never leaves a pending CUDA error behind.
template <class K>
inline void bagel_set_smem_attr(K kernel, size_t want) {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, kernel) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  size_t cap = optin > (int)fa.sharedSizeBytes ? (size_t)optin - fa.sharedSizeBytes : 0;
  if (want > cap) want = cap;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
  cudaGetLastError();
}

// ----------------------------------------------------------------- launchers
// Every launcher returns the number of kernels it enqueued (for gpu_launches).

// cache_build.cu
int cb_build_khat(const float* X, int N, int d, const float* ell_dev, double s, double noise,
                  double* K, cudaStream_t st);
// blocked Cholesky in place (lower); pivot_flag[0] = first failing pivot + 1 (0 if ok)
int cb_cholesky(double* K, int N, int* pivot_flag, cudaStream_t st);
// alpha = L^-T L^-1 y  (y float32 column, stride ystride)
int cb_cholesky_solve(const double* L, int N, const float* y, int ystride, double* alpha,
                      double* tmp, cudaStream_t st);
// Lanczos pieces (fp64)
int cb_symv(const double* K, int N, const double* q, double* v, cudaStream_t st);
int cb_dot(const double* a, const double* b, int N, double* out, cudaStream_t st);
int cb_gemv_t(const double* Q, int nq, int N, const double* v, double* c, cudaStream_t st);  // c = Q v
int cb_gemv_sub(const double* Q, int nq, int N, const double* c, double* v, cudaStream_t st); // v -= Q^T c
int cb_scale_copy(const double* v, double scale_inv, double* q, int N, cudaStream_t st);
int cb_probe_from_y(const float* Y, int ystride, int N, double* v, cudaStream_t st);
int cb_restart_vector(uint32_t restart_idx, int m, int N, double* v, cudaStream_t st);
int cb_love_R(const double* Q, const double* ld, const double* le, int k, int N, double* R,
              cudaStream_t st);
int cb_pack(const float* X, const double* alpha, const double* R, int N, int d, int k, float s,
            const float* qscale_host, int Cld, float* V, float* Xs, cudaStream_t st);

// gp_step.cu
int gs_pass1(const bagel_ctx* c, const float* xstar, int B, cudaStream_t st);
int gs_reduce1(const bagel_ctx* c, const float* xstar, int B, float* jmu_out, float* sig_out,
               cudaStream_t st);
int gs_pass2(const bagel_ctx* c, const float* xstar, int B, cudaStream_t st);
int gs_finish_predict(const bagel_ctx* c, const float* xstar, int B, float* mean, float* var,
                      float* dmean, float* dvar, cudaStream_t st);
void gs_choose_splits(const bagel_ctx* c, int B, int* S1, int* S2);

// rollout.cu
int ro_init(const bagel_ctx* c, const float* theta, const float* x0, const float* goals, int B,
            cudaStream_t st);
EpiArgs ro_epi_args(const bagel_ctx* c, const float* goals, int B, int t, int T, uint64_t seed, long long traj_offset,
                    float* trace_mu, float* trace_var);
int ro_step_epilogue(const bagel_ctx* c, const float* theta, const float* goals, int B, int t, int T,
                     uint64_t seed, long long traj_offset, float* trace_mu, float* trace_var, cudaStream_t st);
int ro_reverse(const bagel_ctx* c, const float* theta, const float* goals, int B, int T,
               uint64_t seed, long long traj_offset, long long B_global, int* nblk_out,
               cudaStream_t st);
int ro_reduce(const bagel_ctx* c, int nblk, int B, long long B_global, float* grad,
              cudaStream_t st);
int ro_copy_returns(const bagel_ctx* c, int B, float* ret, cudaStream_t st);
int ro_philox_raw(const uint32_t* ctr, uint32_t k0, uint32_t k1, int n, uint32_t* out,
                  cudaStream_t st);
int ro_philox_normals(uint64_t seed, long long traj_offset, int B, int T, int p, float* out,
                      cudaStream_t st);
int ro_theta_blocks(const bagel_ctx* c, int B, int T);
bool ro_wide_policy(const PolicyDesc& P);
bool mlp_tc_enabled(const bagel_ctx* c);
int mlp_tc_pack(bagel_ctx* c, const float* theta, cudaStream_t st);
int mlp_tc_backward_step(const bagel_ctx* c, const float* goals, int B, int t, long long B_global, cudaStream_t st);
int mlp_tc_forward_step(const bagel_ctx* c, const float* theta, const float* goals, int B, int t, cudaStream_t st);
int mlp_forward_step(const bagel_ctx* c, const float* theta, const float* goals, int B, int t, cudaStream_t st);
int mlp_reverse(const bagel_ctx* c, const float* theta, const float* goals, int B, int T, long long B_global,
                cudaStream_t st);
int ro_theta_grad(const bagel_ctx* c, int B, int T, int nblk, cudaStream_t st);
size_t ro_theta_grad_smem(const PolicyDesc& P);

// gp_step_tc.cu
bool tc_supported(const bagel_ctx* c);
size_t tc_tiles1_bytes(const bagel_ctx* c);
size_t tc_tiles2_bytes(const bagel_ctx* c);
int tc_pack(bagel_ctx* c, int m, cudaStream_t st);
void tc_choose_splits(const bagel_ctx* c, int B, int* S1, int* S2, int* tps1, int* tps2, int* p1_fused);
int op_sample_uniform(uint64_t seed, long long traj_offset, int B, int p, int which, const float* lo,
                      const float* hi, float* out, cudaStream_t st);
int op_adam(float* theta, const float* g, float* m1, float* m2, int n, float lr, float b1, float b2, float eps,
            float bc1, float bc2, int* flag, cudaStream_t st);
int mll_part_count(int N);
size_t bbmm_workspace_doubles(int N, int nc, int J);
int bbmm_launch(const float* X, const float* Y, int ystride, int N, int d, const double* log_hyp, int t, int J,
                int kp, uint64_t seed, double* ws, int* its_dev, double* logdet, double* quad, double* grad,
                int* rank_out, cudaStream_t st);
int exact_launch(const float* X, const float* Y, int ystride, int N, int d, const float* ell, float s, float noise,
                 double* K, double* Li, double* alpha, int* pivot_flag, cudaStream_t st);
int mll_launch(const float* X, const float* Y, int ystride, int N, int d, const double* log_hyp, double* K,
               double* Li, double* alpha, double* sc, double* part, double* grad, int* pivot_flag, bool want_grad,
               cudaStream_t st);
size_t tc_p1z_floats(const bagel_ctx* c, int B, int S1);
size_t tc_zp_bytes(const bagel_ctx* c, int B);
int tc_njt(const bagel_ctx* c);
int tc_pair_row_tiles(int B);  // row tiles rounded up to whole CTA pairs
// theta_tc.cu: the parameter gradient of wide policies on the tensor cores
bool theta_tc_enabled(const PolicyDesc& P);
int theta_tc_blocks(long long K);
size_t theta_tc_colmax_floats(const PolicyDesc& P, long long K);
int theta_grad_tc(const PolicyDesc& P, long long K, const float* act, const float* delta, float* colmax, float* part,
                  cudaStream_t st);
size_t tc_zpart_count(const bagel_ctx* c, int B);
size_t tc_gbar_count();
int tc_pass1(const bagel_ctx* c, const float* xstar, int B, float* jmu_out, float* sig_out, cudaStream_t st);
int tc_reduce1(const bagel_ctx* c, const float* xstar, int B, float* jmu_out, float* sig_out, cudaStream_t st);
int tc_pass2(const bagel_ctx* c, const float* xstar, int B, const EpiArgs* epi, cudaStream_t st);
bool tc_pass2_epi_ok(const bagel_ctx* c, int B);
