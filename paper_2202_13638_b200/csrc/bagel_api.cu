// bagel_api.cu -- the C ABI of include/bagel.h: context, validation, workspace,
// staging of host buffers, and the host-side orchestration of the hot path
// (rollout_cost_and_grad, Alg.1) and of the one-time LOVE cache
// build.  No exception crosses the ABI.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <new>
#include <string>
#include <vector>

#include "../../include/bagel.h"
#include "bagel_internal.h"

size_t gs_pass2_smem(int k, int d);
size_t ro_reverse_smem(const PolicyDesc& P, int p, int d);
size_t ro_epilogue_smem(const PolicyDesc& P);
size_t ro_policy_smem(const PolicyDesc& P);
int tc_selftest_launch(const void* A, const void* B, int N, int K, float* D, int mode, cudaStream_t st);
int tc_selftest2_launch(const void* A, const void* B, int N, int K, float* D, int ts, cudaStream_t st);
int tc_bench_launch(int N, int iters, int mode, int ctas, long long* cycles, cudaStream_t st);

namespace {

const int kErrNone = 0x7f7f7f7f;  // err_flag sentinel (memset byte 0x7f)

struct Fail {
  int code;
};

void set_err(bagel_ctx* c, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
void set_err(bagel_ctx* c, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  c->err = buf;
}

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      set_err(c, "CUDA error %s at %s:%d (%s)", cudaGetErrorString(e_), __FILE__, __LINE__, #call); \
      throw Fail{BAGEL_E_CUDA};                                                       \
    }                                                                                 \
  } while (0)

#define REQUIRE(cond, code, ...)     \
  do {                               \
    if (!(cond)) {                   \
      set_err(c, __VA_ARGS__);       \
      throw Fail{code};              \
    }                                \
  } while (0)

template <class F>
int guarded(bagel_ctx* c, F&& f) {
  if (!c) return BAGEL_E_ARG;
  c->err.clear();
  try {
    cudaSetDevice(c->device);
    f();
    return BAGEL_OK;
  } catch (const Fail& e) {
    return e.code;
  } catch (const std::bad_alloc&) {
    c->err = "host out of memory";
    return BAGEL_E_CUDA;
  } catch (...) {
    c->err = "unexpected internal exception";
    return BAGEL_E_CUDA;
  }
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

template <class T>
void dev_free(T*& p) {
  if (p) cudaFree((void*)p);
  p = nullptr;
}

template <class T>
void dev_alloc(bagel_ctx* c, T*& p, size_t n) {
  dev_free(p);
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc((void**)&p, n * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    p = nullptr;
    set_err(c, "cudaMalloc of %zu bytes failed (%s)", n * sizeof(T), cudaGetErrorString(e));
    throw Fail{BAGEL_E_CUDA};
  }
}

// Copy n floats from a [dev|host] pointer to host memory.
std::vector<float> to_host(bagel_ctx* c, const float* p, size_t n) {
  std::vector<float> h(n);
  if (n) CK(cudaMemcpyAsync(h.data(), p, n * sizeof(float), cudaMemcpyDefault, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return h;
}

// Device view of a [dev|host] float array; host data goes to ws.stage + offset.
const float* stage_in(bagel_ctx* c, const float* p, size_t n, size_t& off) {
  if (is_device_ptr(p)) return p;
  float* dst = c->ws.stage + off;
  off += (n + 63) & ~(size_t)63;
  if (n) CK(cudaMemcpyAsync(dst, p, n * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  return dst;
}

void ensure_stage(bagel_ctx* c, size_t n) {
  if (c->ws.stage_cap >= n) return;
  dev_alloc(c, c->ws.stage, n);
  c->ws.stage_cap = n;
}

void free_cache(bagel_ctx* c) {
  dev_free(c->alpha64);
  dev_free(c->R64);
  dev_free(c->V);
  dev_free(c->Xs);
  dev_free(c->tcs.tiles1);
  dev_free(c->tcs.tiles2);
  dev_free(c->tcs.colscale);
  dev_free(c->tcs.colscale_inv);
  dev_free(c->tcs.qscale);
  c->k = 0;
  c->cache_ok.assign(c->p, 0);
}

void free_workspace(bagel_ctx* c) {
  Workspace& w = c->ws;
  dev_free(w.xstar); dev_free(w.P1); dev_free(w.Z); dev_free(w.P2); dev_free(w.mu); dev_free(w.var);
  dev_free(w.tape_x); dev_free(w.tape_sig); dev_free(w.tape_jmu); dev_free(w.tape_jv); dev_free(w.G);
  dev_free(w.tape_A); dev_free(w.tape_act); dev_free(w.tape_delta); dev_free(w.xbar);
  w.tape_pol_cap = 0;
  dev_free(w.theta_part); dev_free(w.grad_tmp); dev_free(w.thetaT); dev_free(w.cost_dev); dev_free(w.err_flag);
  dev_free(c->tcs.P1z); dev_free(c->tcs.P1h); dev_free(c->tcs.Zp); dev_free(c->tcs.zrow_inv);
  dev_free(c->tcs.zz_part); dev_free(c->tcs.zmax_part);
  dev_free(w.mlp_wpk);
  w.mlp_wpk_cap = 0;
  w.B = w.T = 0;
  w.S1 = w.S2 = 0;
  w.theta_part_cap = 0;
  dev_free(w.theta_colmax);
  w.theta_colmax_cap = 0;
}

int round_up(int a, int b) { return (a + b - 1) / b * b; }

void setup_gpdesc(bagel_ctx* c, int k) {
  GpDesc& g = c->gp;
  g = GpDesc{};
  g.N = c->N;
  g.d = c->d;
  g.p = c->p;
  g.k = k;
  g.C = 1 + c->d + k;
  g.Cld = round_up(g.C, 64);
  g.abs_target = c->abs_target;
  for (int m = 0; m < c->p; ++m) {
    g.s[m] = c->s[m];
    for (int j = 0; j < c->d; ++j) {
      const float l = c->ell[(size_t)m * c->d + j];
      g.ell2inv[m][j] = (float)(1.0 / ((double)l * (double)l));
      g.qscale[m][j] = (float)((double)BAGEL_KAPPA / (double)l);
    }
  }
}

// Workspace for B trajectories and T steps (the tape and the step buffers).
void ensure_workspace(bagel_ctx* c, int B, int T) {
  Workspace& w = c->ws;
  int S1, S2;
  gs_choose_splits(c, B, &S1, &S2);
  int S1t = 0, S2t = 0, tps1 = 0, tps2 = 0, fused = 0;
  const bool tc = tc_supported(c);
  if (tc) tc_choose_splits(c, B, &S1t, &S2t, &tps1, &tps2, &fused);
  const bool same = w.B >= B && w.T >= T && w.B > 0 && w.S1 == S1 && w.S2 == S2 && w.B == B && w.S1tc == S1t &&
                    w.S2tc == S2t && w.p1_fused == fused && w.tps1 == tps1;
  const int nblk = ro_theta_blocks(c, B, T);
  if (!same) {
    free_workspace(c);
    const int p = c->p, d = c->d;
    const size_t Bs = (size_t)B, Ts = (size_t)std::max(T, 1);
    dev_alloc(c, w.xstar, Bs * d);
    dev_alloc(c, w.P1, (size_t)S1 * p * Bs * c->gp.Cld);
    dev_alloc(c, w.Z, (size_t)p * Bs * c->gp.k);
    const size_t s2max = std::max((size_t)S2, (size_t)S2t * (tc ? tc_njt(c) : 1));
    dev_alloc(c, w.P2, s2max * p * Bs * (1 + BAGEL_MAX_D));
    if (tc) {
      dev_alloc(c, c->tcs.P1z, tc_p1z_floats(c, (B + 127) / 128 * 128, S1t));  // fused layout pads row tiles
      dev_alloc(c, c->tcs.P1h, (size_t)S1t * p * Bs * (1 + d));
      dev_alloc(c, c->tcs.Zp, tc_zp_bytes(c, B));
      CK(cudaMemsetAsync(c->tcs.Zp, 0, tc_zp_bytes(c, B), c->stream));  // padding rows / j stay zero
      dev_alloc(c, c->tcs.zrow_inv, (size_t)p * Bs);
      if (!c->tcs.gbar) dev_alloc(c, c->tcs.gbar, 2 * tc_gbar_count());  // pass 1 | pass 2
      // the barrier's counters assume a fixed grid: restart them with every new split layout
      CK(cudaMemsetAsync(c->tcs.gbar, 0, 2 * tc_gbar_count() * sizeof(unsigned long long), c->stream));
      dev_alloc(c, c->tcs.zz_part, tc_zpart_count(c, B));
      dev_alloc(c, c->tcs.zmax_part, tc_zpart_count(c, B));
    }
    dev_alloc(c, w.mu, (size_t)p * Bs);
    dev_alloc(c, w.var, (size_t)p * Bs);
    dev_alloc(c, w.tape_x, (Ts + 1) * Bs * p);
    dev_alloc(c, w.tape_sig, Ts * Bs * p);
    dev_alloc(c, w.tape_jmu, Ts * Bs * p * d);
    dev_alloc(c, w.tape_jv, Ts * Bs * p * d);
    dev_alloc(c, w.tape_A, Ts * Bs * p * d);
    dev_alloc(c, w.xbar, Bs * p);
    dev_alloc(c, w.G, Bs);
    dev_alloc(c, w.cost_dev, 1);
    dev_alloc(c, w.err_flag, 1);
    w.B = B;
    w.T = std::max(T, 1);
    w.S1 = S1;
    w.S2 = S2;
    w.S1tc = S1t;
    w.S2tc = S2t;
    w.tps1 = tps1;
    w.tps2 = tps2;
    w.p1_fused = fused;
  }
  if (c->policy_ok) {
    const int need = nblk * c->pol.n_params;
    if (w.theta_part_cap < need) {
      dev_alloc(c, w.theta_part, (size_t)need);
      w.theta_part_cap = need;
    }
    const size_t rows = (size_t)std::max(w.T, 1) * w.B;
    if (w.tape_pol_cap < rows) {
      dev_alloc(c, w.tape_act, rows * c->pol.act_ld);
      dev_alloc(c, w.tape_delta, rows * c->pol.d_ld);
      w.tape_pol_cap = rows;
    }
    if (theta_tc_enabled(c->pol)) {
      const size_t cm = theta_tc_colmax_floats(c->pol, (long long)std::max(w.T, 1) * w.B);
      if (w.theta_colmax_cap < cm) {
        dev_alloc(c, w.theta_colmax, cm);
        w.theta_colmax_cap = cm;
      }
    }
    if (!w.grad_tmp) dev_alloc(c, w.grad_tmp, (size_t)c->pol.n_params + 64);
    if (!w.thetaT) dev_alloc(c, w.thetaT, (size_t)c->pol.n_params + 64);
  }
}

void require_ready(bagel_ctx* c, bool need_policy) {
  REQUIRE(c->N > 0, BAGEL_E_STATE, "no GP loaded: call gp_load first");
  REQUIRE(c->k > 0, BAGEL_E_STATE, "no LOVE cache: call love_cache_build (or bagel_cache_set) first");
  for (int m = 0; m < c->p; ++m)
    REQUIRE(c->cache_ok[m], BAGEL_E_STATE, "LOVE cache of output %d is missing", m);
  if (need_policy) {
    REQUIRE(c->policy_ok, BAGEL_E_STATE, "no policy: call policy_configure first");
    REQUIRE(c->reward_ok, BAGEL_E_STATE, "no reward: call reward_configure first");
  }
}

void check_numeric(bagel_ctx* c, int B) {
  int flag = kErrNone;
  CK(cudaMemcpyAsync(&flag, c->ws.err_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (flag == BAGEL_BARRIER_TIMEOUT) {
    set_err(c, "grid barrier timed out: the one-wave GP-step grid was not co-resident (other work on the "
               "GPU?); set BAGEL_COOP=1 for cooperative launches");
    throw Fail{BAGEL_E_CUDA};
  }
  if (flag != kErrNone) {
    set_err(c, "non-finite state at step %d, row %d", flag / B, flag % B);
    throw Fail{BAGEL_E_NUMERIC};
  }
}

enum { PC_PASS1 = 0, PC_REDUCE1, PC_PASS2, PC_EPI, PC_INIT, PC_REVERSE, PC_REDUCE, PC_THETA };

cudaEvent_t prof_event(bagel_ctx* c) {
  if (!c->prof_pool.empty()) {
    cudaEvent_t e = c->prof_pool.back();
    c->prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  return e;
}

// Run a launcher; with profiling on, bracket it with events on the context stream.
template <class F>
int timed(bagel_ctx* c, int cls, F&& f) {
  if (!c->prof_on) return f();
  cudaEvent_t a = prof_event(c), b = prof_event(c);
  CK(cudaEventRecord(a, c->stream));
  const int n = f();
  CK(cudaEventRecord(b, c->stream));
  c->prof_pending.push_back({a, b, cls});
  c->prof_n[cls] += n;
  return n;
}

void prof_drain(bagel_ctx* c) {
  if (c->prof_pending.empty()) return;
  CK(cudaStreamSynchronize(c->stream));
  for (auto& e : c->prof_pending) {
    float ms = 0.0f;
    CK(cudaEventElapsedTime(&ms, e.a, e.b));
    c->prof_ms[e.cls] += ms;
    c->prof_pool.push_back(e.a);
    c->prof_pool.push_back(e.b);
  }
  c->prof_pending.clear();
}

// The tensor-core GP step is THE path; the v0 CUDA-core kernels run only when a test selects them
// explicitly (bagel_set_gp_kernel(0), a precision cross-check).  A shape the tensor-core kernels
// cannot hold is an error, never a silent switch to another implementation.
//
// Absolute targets (gp_target_mode(1)) run on the v0 kernels: the tensor core accumulates in
// TMEM with truncation (~1 ulp of the accumulator per MMA step, scripts/diag_tmem_acc.py), which
// biases ||z|| low by ~steps x 2^-24 relative; with y = x_{k+1} the prior variance s is the states'
// variance, v / s falls to ~1e-6 and v = s - ||z||^2 loses all accuracy (measured: gradient 7.5e-3
// off at T = 40 vs 5.3e-4 for the round-to-nearest FFMA path; R38).
bool use_tc(bagel_ctx* c) {
  if (c->gp_kernel != 1 || c->gp.abs_target) return false;
  REQUIRE(tc_supported(c), BAGEL_E_ARG, "GP shape (N=%d, d=%d, k=%d) exceeds the tensor-core kernels' shared memory",
          c->N, c->d, c->k);
  return true;
}

// Forward rollout (shared by rollout_cost_and_grad and bagel_rollout_trace).
int forward(bagel_ctx* c, const float* theta, const float* x0, const float* goals, int B, int T,
            uint64_t seed, long long traj_offset, float* trace_mu, float* trace_var) {
  cudaStream_t st = c->stream;
  Workspace& w = c->ws;
  const int p = c->p, d = c->d;
  int launches = 0;
  CK(cudaMemsetAsync(w.err_flag, 0x7f, sizeof(int), st));
  launches += timed(c, PC_INIT, [&] { return ro_init(c, theta, x0, goals, B, st); });
  if (ro_wide_policy(c->pol) && mlp_tc_enabled(c)) {
    // wide policies: this iteration's weights as the tensor-core MLP's hi/lo operand (mlp_tc.cu)
    const int r = mlp_tc_pack(c, theta, st);
    REQUIRE(r > 0, BAGEL_E_CUDA, "rollout: out of device memory for the packed policy weights");
    launches += r;
  }
  const bool tc = use_tc(c);
  w.S2eff = tc ? w.S2tc * tc_njt(c) : w.S2;
  const bool fuse_epi = tc && tc_pass2_epi_ok(c, B);
  for (int t = 0; t < T; ++t) {
    float* jm = w.tape_jmu + (size_t)t * B * p * d;
    float* sg = w.tape_sig + (size_t)t * B * p;
    launches += timed(c, PC_PASS1, [&] { return tc ? tc_pass1(c, w.xstar, B, jm, sg, st) : gs_pass1(c, w.xstar, B, st); });
    if (!(tc && w.p1_fused))
      launches += timed(c, PC_REDUCE1, [&] {
        return tc ? tc_reduce1(c, w.xstar, B, jm, sg, st) : gs_reduce1(c, w.xstar, B, jm, sg, st);
      });
    if (fuse_epi) {
      const EpiArgs e = ro_epi_args(c, goals, B, t, T, seed, traj_offset, trace_mu, trace_var);
      launches += timed(c, PC_PASS2, [&] { return tc_pass2(c, w.xstar, B, &e, st); });
    } else {
      launches += timed(c, PC_PASS2, [&] { return tc ? tc_pass2(c, w.xstar, B, nullptr, st) : gs_pass2(c, w.xstar, B, st); });
      launches += timed(c, PC_EPI, [&] {
        return ro_step_epilogue(c, theta, goals, B, t, T, seed, traj_offset, trace_mu, trace_var, st);
      });
    }
  }
  CK(cudaGetLastError());
  return launches;
}

void load_common_rollout_args(bagel_ctx* c, const float* theta, const float* x0, const float* goals, int B,
                              int T, const float** th_d, const float** x0_d, const float** g_d) {
  require_ready(c, true);
  REQUIRE(B >= 1, BAGEL_E_ARG, "B must be >= 1 (got %d)", B);
  REQUIRE(T >= 0, BAGEL_E_ARG, "T must be >= 0 (got %d)", T);
  // the numeric-fault report encodes (step, row) as one int (t * B + b)
  REQUIRE((long long)B * (long long)(T + 1) < 2147483647LL, BAGEL_E_ARG,
          "B * (T + 1) must be < 2^31 (got B = %d, T = %d)", B, T);
  REQUIRE(theta && x0 && goals, BAGEL_E_ARG, "policy_params, x0 and goals must be non-NULL");
  const size_t np = (size_t)c->pol.n_params, bp = (size_t)B * c->p;
  ensure_stage(c, np + 2 * bp + 256);
  ensure_workspace(c, B, T);
  size_t off = 0;
  *th_d = stage_in(c, theta, np, off);
  *x0_d = stage_in(c, x0, bp, off);
  *g_d = stage_in(c, goals, bp, off);
}

}  // namespace

// ====================================================================== ABI

extern "C" int bagel_create(bagel_ctx** out, int device, void* cuda_stream) {
  if (!out) return BAGEL_E_ARG;
  *out = nullptr;
  bagel_ctx* c = new (std::nothrow) bagel_ctx();
  if (!c) return BAGEL_E_CUDA;
  c->device = device;
  c->stream = (cudaStream_t)cuda_stream;
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    delete c;
    return BAGEL_E_CUDA;
  }
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess && sms > 0)
    c->num_sms = sms;
  *out = c;
  return BAGEL_OK;
}

extern "C" int bagel_destroy(bagel_ctx* c) {
  if (!c) return BAGEL_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  free_workspace(c);
  free_cache(c);
  for (auto& e : c->prof_pending) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  for (auto e : c->prof_pool) cudaEventDestroy(e);
  dev_free(c->tcs.dbg1);
  dev_free(c->tcs.dbg2);
  dev_free(c->tcs.dbg3);
  dev_free(c->tcs.gbar);
  dev_free(c->X);
  dev_free(c->Y);
  dev_free(c->ws.stage);
  dev_free(c->op_flag);
  dev_free(c->op_bounds);
  dev_free(c->mll_K);
  dev_free(c->mll_Li);
  dev_free(c->mll_vec);
  dev_free(c->bbmm_ws);
  dev_free(c->bbmm_its);
  delete c;
  return BAGEL_OK;
}

extern "C" int bagel_set_stream(bagel_ctx* c, void* cuda_stream) {
  return guarded(c, [&] { c->stream = (cudaStream_t)cuda_stream; });
}

extern "C" const char* bagel_last_error(const bagel_ctx* c) { return c ? c->err.c_str() : "null context"; }

#ifndef BAGEL_SRC_HASH
#define BAGEL_SRC_HASH "unknown"
#endif
extern "C" const char* bagel_build_hash(void) { return BAGEL_SRC_HASH; }

extern "C" int gp_load(bagel_ctx* c, const float* X, const float* y, int N, int d, int p,
                       const float* lengthscales, const float* outputscale, const float* noise) {
  return guarded(c, [&] {
    REQUIRE(X && y && lengthscales && outputscale && noise, BAGEL_E_ARG, "gp_load: NULL array argument");
    REQUIRE(N >= 1, BAGEL_E_ARG, "gp_load: N must be >= 1 (got %d)", N);
    REQUIRE(p >= 1 && p <= BAGEL_MAX_P, BAGEL_E_ARG, "gp_load: p must be in [1, %d] (got %d)", BAGEL_MAX_P, p);
    REQUIRE(d > p && d <= BAGEL_MAX_D && d >= 2, BAGEL_E_ARG,
            "gp_load: d must satisfy p < d <= %d (got d=%d, p=%d)", BAGEL_MAX_D, d, p);
    std::vector<float> hX = to_host(c, X, (size_t)N * d), hy = to_host(c, y, (size_t)N * p);
    std::vector<float> hl = to_host(c, lengthscales, (size_t)p * d), hs = to_host(c, outputscale, p),
                       hn = to_host(c, noise, p);
    for (size_t i = 0; i < hX.size(); ++i)
      REQUIRE(isfinite(hX[i]), BAGEL_E_ARG, "gp_load: X[%zu][%zu] is not finite (X is %d x %d)", i / d, i % d, N, d);
    for (size_t i = 0; i < hy.size(); ++i)
      REQUIRE(isfinite(hy[i]), BAGEL_E_ARG, "gp_load: y[%zu][%zu] is not finite (y is %d x %d)", i / p, i % p, N, p);
    for (size_t i = 0; i < hl.size(); ++i)
      REQUIRE(isfinite(hl[i]) && hl[i] > 0.0f, BAGEL_E_ARG, "gp_load: lengthscales[%zu][%zu] = %g must be finite and > 0",
              i / d, i % d, (double)hl[i]);
    for (int m = 0; m < p; ++m) {
      REQUIRE(isfinite(hs[m]) && hs[m] > 0.0f, BAGEL_E_ARG, "gp_load: outputscale[%d] = %g must be finite and > 0", m,
              (double)hs[m]);
      REQUIRE(isfinite(hn[m]) && hn[m] >= 1e-8f, BAGEL_E_ARG, "gp_load: noise[%d] = %g must be >= 1e-8", m,
              (double)hn[m]);
    }
    free_cache(c);
    free_workspace(c);
    dev_alloc(c, c->X, (size_t)N * d);
    dev_alloc(c, c->Y, (size_t)N * p);
    CK(cudaMemcpyAsync(c->X, hX.data(), hX.size() * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->Y, hy.data(), hy.size() * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->N = N;
    c->d = d;
    c->p = p;
    c->ell = hl;
    c->s = hs;
    c->noise = hn;
    c->cache_ok.assign(p, 0);
    c->policy_ok = false;
    c->reward_ok = false;
  });
}

namespace {

void alloc_cache(bagel_ctx* c, int k) {
  free_cache(c);
  free_workspace(c);
  setup_gpdesc(c, k);
  dev_alloc(c, c->alpha64, (size_t)c->p * c->N);
  dev_alloc(c, c->R64, (size_t)c->p * k * c->N);
  dev_alloc(c, c->V, (size_t)c->p * c->N * c->gp.Cld);
  dev_alloc(c, c->Xs, (size_t)c->p * c->N * c->d);
  c->k = k;
  if (tc_supported(c)) {
    c->tcs.t1_stride = tc_tiles1_bytes(c);
    c->tcs.t2_stride = tc_tiles2_bytes(c);
    dev_alloc(c, c->tcs.tiles1, (size_t)c->p * c->tcs.t1_stride);
    dev_alloc(c, c->tcs.tiles2, (size_t)c->p * c->tcs.t2_stride);
    dev_alloc(c, c->tcs.colscale, (size_t)c->p * k);
    dev_alloc(c, c->tcs.colscale_inv, (size_t)c->p * k);
    dev_alloc(c, c->tcs.qscale, (size_t)c->p * BAGEL_MAX_D);
  }
  c->cache_ok.assign(c->p, 0);
}

void pack_output(bagel_ctx* c, int m) {
  cb_pack(c->X, c->alpha64 + (size_t)m * c->N, c->R64 + (size_t)m * c->k * c->N, c->N, c->d, c->k, c->s[m],
          c->gp.qscale[m], c->gp.Cld, c->V + (size_t)m * c->N * c->gp.Cld, c->Xs + (size_t)m * c->N * c->d,
          c->stream);
  if (tc_supported(c)) tc_pack(c, m, c->stream);
  CK(cudaGetLastError());
}

}  // namespace

extern "C" int love_cache_build(bagel_ctx* c, int rank, double* seconds_out) {
  return guarded(c, [&] {
    REQUIRE(c->N > 0, BAGEL_E_STATE, "love_cache_build: no GP loaded (call gp_load first)");
    REQUIRE(rank >= 1 && rank <= c->N && rank <= BAGEL_MAX_RANK, BAGEL_E_ARG,
            "love_cache_build: rank must be in [1, min(N=%d, %d)] (got %d)", c->N, BAGEL_MAX_RANK, rank);
    const auto t0 = std::chrono::steady_clock::now();
    const int N = c->N, k = rank;
    cudaStream_t st = c->stream;
    alloc_cache(c, k);
    double *K = nullptr, *Q = nullptr, *v = nullptr, *cs = nullptr, *sc = nullptr, *ldd = nullptr, *led = nullptr;
    int* piv = nullptr;
    struct Guard {
      bagel_ctx* c;
      double** ps[7];
      int** pi;
      ~Guard() {
        for (auto p : ps) dev_free(*p);
        dev_free(*pi);
      }
    } guard{c, {&K, &Q, &v, &cs, &sc, &ldd, &led}, &piv};
    dev_alloc(c, K, (size_t)N * N);
    dev_alloc(c, Q, (size_t)k * N);
    dev_alloc(c, v, (size_t)N);
    dev_alloc(c, cs, (size_t)k + 1);
    dev_alloc(c, sc, 4);
    dev_alloc(c, ldd, (size_t)k);
    dev_alloc(c, led, (size_t)k);
    dev_alloc(c, piv, 1);
    for (int m = 0; m < c->p; ++m) {
      cb_build_khat(c->X, N, c->d, c->ell.data() + (size_t)m * c->d, (double)c->s[m], (double)c->noise[m], K, st);
      // ---- Lanczos (reading R20)
      std::vector<double> a(k), b(k, 0.0);
      uint32_t restart_idx = 0;
      double h[2];
      cb_probe_from_y(c->Y + m, c->p, N, v, st);
      cb_dot(v, v, N, sc, st);
      CK(cudaMemcpyAsync(h, sc, sizeof(double), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      double ny = sqrt(h[0]);
      if (!(ny > 0.0)) {
        cb_restart_vector(restart_idx++, m, N, v, st);
        cb_dot(v, v, N, sc, st);
        CK(cudaMemcpyAsync(h, sc, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        ny = sqrt(h[0]);
      }
      cb_scale_copy(v, 1.0 / ny, Q, N, st);
      double amax = 0.0;
      for (int j = 0; j < k; ++j) {
        const double* qj = Q + (size_t)j * N;
        cb_symv(K, N, qj, v, st);
        cb_dot(qj, v, N, sc, st);
        for (int pass = 0; pass < 2; ++pass) {
          cb_gemv_t(Q, j + 1, N, v, cs, st);
          cb_gemv_sub(Q, j + 1, N, cs, v, st);
        }
        cb_dot(v, v, N, sc + 1, st);
        CK(cudaMemcpyAsync(h, sc, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        a[j] = h[0];
        amax = std::max(amax, fabs(h[0]));
        const double bj = sqrt(h[1]);
        if (j < k - 1) {
          double* qn = Q + (size_t)(j + 1) * N;
          if (bj <= 1e-10 * amax) {
            cb_restart_vector(restart_idx++, m, N, v, st);
            for (int pass = 0; pass < 2; ++pass) {
              cb_gemv_t(Q, j + 1, N, v, cs, st);
              cb_gemv_sub(Q, j + 1, N, cs, v, st);
            }
            cb_dot(v, v, N, sc, st);
            CK(cudaMemcpyAsync(h, sc, sizeof(double), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            cb_scale_copy(v, 1.0 / sqrt(h[0]), qn, N, st);
            b[j] = 0.0;
          } else {
            cb_scale_copy(v, 1.0 / bj, qn, N, st);
            b[j] = bj;
          }
        }
      }
      // ---- L_T = chol(T), bidiagonal; R = L_T^-1 Q^T
      std::vector<double> ld(k), le(k, 0.0);
      for (int j = 0; j < k; ++j) {
        double dj = a[j];
        if (j > 0) {
          le[j] = b[j - 1] / ld[j - 1];
          dj -= le[j] * le[j];
        }
        REQUIRE(dj > 0.0, BAGEL_E_NUMERIC, "love_cache_build: Lanczos T of output %d is not positive definite at row %d", m, j);
        ld[j] = sqrt(dj);
      }
      CK(cudaMemcpyAsync(ldd, ld.data(), k * sizeof(double), cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(led, le.data(), k * sizeof(double), cudaMemcpyHostToDevice, st));
      cb_love_R(Q, ldd, led, k, N, c->R64 + (size_t)m * k * N, st);
      // ---- alpha = Khat^-1 y by blocked Cholesky (in place on K)
      CK(cudaMemsetAsync(piv, 0, sizeof(int), st));
      cb_cholesky(K, N, piv, st);
      int pv = 0;
      CK(cudaMemcpyAsync(&pv, piv, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      REQUIRE(pv == 0, BAGEL_E_NUMERIC, "love_cache_build: Cholesky pivot %d of output %d is <= 0 (Khat not SPD)", pv - 1, m);
      cb_cholesky_solve(K, N, c->Y + m, c->p, c->alpha64 + (size_t)m * N, nullptr, st);
      CK(cudaGetLastError());
      pack_output(c, m);
      c->cache_ok[m] = 1;
    }
    CK(cudaStreamSynchronize(st));
    if (seconds_out)
      *seconds_out = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

extern "C" int exact_cache_build(bagel_ctx* c, double* seconds_out) {
  return guarded(c, [&] {
    REQUIRE(c->N > 0, BAGEL_E_STATE, "exact_cache_build: no GP loaded (call gp_load first)");
    REQUIRE(c->N <= BAGEL_MAX_RANK, BAGEL_E_ARG,
            "exact_cache_build: the exact variance is the LOVE query at rank N, supported for N <= %d (N=%d)",
            BAGEL_MAX_RANK, c->N);
    const auto t0 = std::chrono::steady_clock::now();
    const int N = c->N;
    cudaStream_t st = c->stream;
    alloc_cache(c, N);
    double* K = nullptr;
    int* piv = nullptr;
    struct Guard {
      bagel_ctx* c;
      double** K;
      int** piv;
      ~Guard() {
        dev_free(*K);
        dev_free(*piv);
      }
    } guard{c, &K, &piv};
    dev_alloc(c, K, (size_t)N * N);
    dev_alloc(c, piv, 1);
    for (int m = 0; m < c->p; ++m) {
      CK(cudaMemsetAsync(piv, 0, sizeof(int), st));
      exact_launch(c->X, c->Y + m, c->p, N, c->d, c->ell.data() + (size_t)m * c->d, c->s[m], c->noise[m], K,
                   c->R64 + (size_t)m * N * N, c->alpha64 + (size_t)m * N, piv, st);
      int pv = 0;
      CK(cudaMemcpyAsync(&pv, piv, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      REQUIRE(pv == 0, BAGEL_E_NUMERIC, "exact_cache_build: Cholesky pivot %d of output %d is <= 0 (Khat not SPD)", pv - 1,
              m);
      pack_output(c, m);
      c->cache_ok[m] = 1;
    }
    CK(cudaStreamSynchronize(st));
    if (seconds_out)
      *seconds_out = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

extern "C" int policy_configure(bagel_ctx* c, const int* sizes, int n_sizes) {
  return guarded(c, [&] {
    REQUIRE(c->N > 0, BAGEL_E_STATE, "policy_configure: no GP loaded (call gp_load first)");
    REQUIRE(sizes && n_sizes >= 2 && n_sizes <= BAGEL_MAX_LAYERS + 1, BAGEL_E_ARG,
            "policy_configure: need 2..%d layer sizes (got %d)", BAGEL_MAX_LAYERS + 1, n_sizes);
    PolicyDesc P{};
    P.n_layers = n_sizes - 1;
    int off = 0, mw = 0, at = 0;
    for (int i = 0; i < n_sizes; ++i) {
      REQUIRE(sizes[i] >= 1 && sizes[i] <= BAGEL_MAX_WIDTH, BAGEL_E_ARG,
              "policy_configure: width %d of layer %d must be in [1, %d]", sizes[i], i, BAGEL_MAX_WIDTH);
      P.sizes[i] = sizes[i];
      mw = std::max(mw, sizes[i]);
      at += sizes[i];
    }
    REQUIRE(sizes[0] == 2 * c->p || sizes[0] == 3 * c->p, BAGEL_E_ARG,
            "policy_configure: input width %d must be 2p=%d ([x,g]) or 3p=%d ([x,g,g-x])", sizes[0], 2 * c->p, 3 * c->p);
    REQUIRE(sizes[n_sizes - 1] == c->d - c->p, BAGEL_E_ARG, "policy_configure: output width %d must be q = d - p = %d",
            sizes[n_sizes - 1], c->d - c->p);
    for (int l = 0; l < P.n_layers; ++l) {
      P.w_off[l] = off;
      off += P.sizes[l] * P.sizes[l + 1];
      P.b_off[l] = off;
      off += P.sizes[l + 1];
    }
    P.n_params = off;
    P.max_width = mw;
    P.act_total = at;
    {
      int ao = 0, dof = 0;
      for (int l = 0; l <= P.n_layers; ++l) {
        P.aoff[l] = ao;
        ao += (P.sizes[l] + 3) & ~3;
        if (l < P.n_layers) {
          P.doff[l] = dof;
          dof += (P.sizes[l + 1] + 3) & ~3;
        }
      }
      P.act_ld = ao;
      P.d_ld = dof;
    }
    P.phi_mode = sizes[0] == 3 * c->p ? 1 : 0;
    REQUIRE(ro_reverse_smem(P, c->p, c->d) <= 200 * 1024 && ro_policy_smem(P) <= 200 * 1024 &&
                ro_theta_grad_smem(P) <= 200 * 1024, BAGEL_E_ARG,
            "policy_configure: policy with %d parameters exceeds the kernels' shared-memory budget", P.n_params);
    c->pol = P;
    c->policy_ok = true;
    c->ws.theta_part_cap = 0;
    dev_free(c->ws.theta_part);
    c->ws.tape_pol_cap = 0;
    dev_free(c->ws.tape_act);
    dev_free(c->ws.tape_delta);
    dev_free(c->ws.grad_tmp);
    dev_free(c->ws.thetaT);
  });
}

extern "C" int reward_configure(bagel_ctx* c, const float* Q_diag, float sigma_r) {
  return guarded(c, [&] {
    REQUIRE(c->N > 0, BAGEL_E_STATE, "reward_configure: no GP loaded (call gp_load first)");
    REQUIRE(Q_diag, BAGEL_E_ARG, "reward_configure: Q_diag is NULL");
    REQUIRE(isfinite(sigma_r) && sigma_r > 0.0f, BAGEL_E_ARG, "reward_configure: sigma_r = %g must be > 0",
            (double)sigma_r);
    RewardDesc r{};
    for (int m = 0; m < c->p; ++m) {
      REQUIRE(isfinite(Q_diag[m]) && Q_diag[m] >= 0.0f, BAGEL_E_ARG, "reward_configure: Q[%d] = %g must be >= 0", m,
              (double)Q_diag[m]);
      r.Q[m] = Q_diag[m];
    }
    r.inv_two_sr2 = (float)(1.0 / (2.0 * (double)sigma_r * (double)sigma_r));
    c->rw = r;
    c->reward_ok = true;
  });
}

extern "C" int rollout_cost_and_grad(bagel_ctx* c, const float* policy_params, const float* x0,
                                     const float* goals, int B, int T, uint64_t seed, long long traj_offset,
                                     long long B_global, double* mean_cost, float* grad) {
  return guarded(c, [&] {
    REQUIRE(mean_cost && grad, BAGEL_E_ARG, "rollout_cost_and_grad: mean_cost and grad must be non-NULL");
    REQUIRE(B_global >= B && traj_offset >= 0 && traj_offset + B <= 0xffffffffLL, BAGEL_E_ARG,
            "rollout_cost_and_grad: need B_global >= B and 0 <= traj_offset, traj_offset + B < 2^32 "
            "(B=%d, B_global=%lld, traj_offset=%lld)", B, B_global, traj_offset);
    const float *th, *xd, *gd;
    load_common_rollout_args(c, policy_params, x0, goals, B, T, &th, &xd, &gd);
    cudaStream_t st = c->stream;
    int launches = forward(c, th, xd, gd, B, T, seed, traj_offset, nullptr, nullptr);
    const bool dev_grad = is_device_ptr(grad);
    float* gout = dev_grad ? grad : c->ws.grad_tmp;
    int nblk = 0;
    launches += timed(c, PC_REVERSE, [&] { return ro_reverse(c, th, gd, B, T, seed, traj_offset, B_global, &nblk, st); });
    {
      const int n = timed(c, PC_THETA, [&] { return ro_theta_grad(c, B, T, nblk, st); });
      REQUIRE(n > 0, BAGEL_E_CUDA, "rollout: could not encode the tensor maps of the theta-gradient contraction");
      launches += n;
    }
    launches += timed(c, PC_REDUCE, [&] { return ro_reduce(c, nblk, B, B_global, gout, st); });
    CK(cudaGetLastError());
    double cost = 0.0;
    CK(cudaMemcpyAsync(&cost, c->ws.cost_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
    if (!dev_grad)
      CK(cudaMemcpyAsync(grad, gout, (size_t)c->pol.n_params * sizeof(float), cudaMemcpyDeviceToHost, st));
    check_numeric(c, B);  // synchronises
    prof_drain(c);
    *mean_cost = cost;
    c->last_launches = launches;
  });
}

extern "C" int bagel_last_launch_count(const bagel_ctx* c, int* launches) {
  if (!c || !launches) return BAGEL_E_ARG;
  *launches = c->last_launches;
  return BAGEL_OK;
}

extern "C" int bagel_gp_predict(bagel_ctx* c, const float* xstar, int M, float* mean, float* var, float* dmean,
                                float* dvar) {
  return guarded(c, [&] {
    require_ready(c, false);
    REQUIRE(M >= 1 && xstar, BAGEL_E_ARG, "bagel_gp_predict: need M >= 1 and xstar non-NULL");
    ensure_workspace(c, M, 1);
    cudaStream_t st = c->stream;
    CK(cudaMemsetAsync(c->ws.err_flag, 0x7f, sizeof(int), st));  // barrier watchdog report
    float* jmu = dmean ? dmean : c->ws.tape_jmu;
    const bool tc = use_tc(c);
    c->ws.S2eff = tc ? c->ws.S2tc * tc_njt(c) : c->ws.S2;
    int n = 0;
    n += tc ? tc_pass1(c, xstar, M, jmu, c->ws.tape_sig, st) : gs_pass1(c, xstar, M, st);
    if (!(tc && c->ws.p1_fused))
      n += tc ? tc_reduce1(c, xstar, M, jmu, c->ws.tape_sig, st) : gs_reduce1(c, xstar, M, jmu, c->ws.tape_sig, st);
    n += tc ? tc_pass2(c, xstar, M, nullptr, st) : gs_pass2(c, xstar, M, st);
    n += gs_finish_predict(c, xstar, M, mean, var, dmean, dvar, st);
    CK(cudaGetLastError());
    check_numeric(c, M);  // synchronises; only the barrier watchdog can fire here
    c->last_launches = n;
  });
}

extern "C" int bagel_rollout_trace(bagel_ctx* c, const float* policy_params, const float* x0, const float* goals,
                                   int B, int T, uint64_t seed, long long traj_offset, float* x, float* mu,
                                   float* var, float* ret) {
  return guarded(c, [&] {
    const float *th, *xd, *gd;
    load_common_rollout_args(c, policy_params, x0, goals, B, T, &th, &xd, &gd);
    cudaStream_t st = c->stream;
    int n = forward(c, th, xd, gd, B, T, seed, traj_offset, mu, var);
    if (x)
      CK(cudaMemcpyAsync(x, c->ws.tape_x, (size_t)(T + 1) * B * c->p * sizeof(float), cudaMemcpyDeviceToDevice, st));
    if (ret) n += ro_copy_returns(c, B, ret, st);
    check_numeric(c, B);
    c->last_launches = n;
  });
}

extern "C" int bagel_philox4x32_10(bagel_ctx* c, const uint32_t* ctr, const uint32_t* key, int n, uint32_t* out) {
  return guarded(c, [&] {
    REQUIRE(ctr && key && out && n >= 0, BAGEL_E_ARG, "bagel_philox4x32_10: bad arguments");
    if (n == 0) return;
    ro_philox_raw(ctr, key[0], key[1], n, out, c->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
  });
}

extern "C" int bagel_philox_normals(bagel_ctx* c, uint64_t seed, long long traj_offset, int B, int T, int p,
                                    float* out) {
  return guarded(c, [&] {
    REQUIRE(out && B >= 1 && T >= 1 && p >= 1 && p <= BAGEL_MAX_P, BAGEL_E_ARG, "bagel_philox_normals: bad arguments");
    ro_philox_normals(seed, traj_offset, B, T, p, out, c->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
  });
}

extern "C" int bagel_cache_rank(const bagel_ctx* c, int* rank) {
  if (!c || !rank) return BAGEL_E_ARG;
  *rank = c->k;
  return BAGEL_OK;
}

extern "C" int bagel_cache_get(bagel_ctx* c, int m, double* alpha, double* R) {
  return guarded(c, [&] {
    REQUIRE(c->k > 0 && m >= 0 && m < c->p && c->cache_ok[m], BAGEL_E_STATE, "bagel_cache_get: no cache for output %d", m);
    if (alpha)
      CK(cudaMemcpyAsync(alpha, c->alpha64 + (size_t)m * c->N, (size_t)c->N * sizeof(double), cudaMemcpyDefault, c->stream));
    if (R)
      CK(cudaMemcpyAsync(R, c->R64 + (size_t)m * c->k * c->N, (size_t)c->k * c->N * sizeof(double), cudaMemcpyDefault,
                         c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

extern "C" int bagel_cache_set(bagel_ctx* c, int m, int rank, const double* alpha, const double* R) {
  return guarded(c, [&] {
    REQUIRE(c->N > 0, BAGEL_E_STATE, "bagel_cache_set: no GP loaded");
    REQUIRE(m >= 0 && m < c->p, BAGEL_E_ARG, "bagel_cache_set: output %d out of range [0, %d)", m, c->p);
    REQUIRE(rank >= 1 && rank <= c->N && rank <= BAGEL_MAX_RANK, BAGEL_E_ARG, "bagel_cache_set: bad rank %d", rank);
    REQUIRE(alpha && R, BAGEL_E_ARG, "bagel_cache_set: alpha and R must be non-NULL");
    if (c->k != rank) {
      bool any = false;
      for (int i = 0; i < c->p; ++i) any = any || c->cache_ok[i];
      REQUIRE(!any, BAGEL_E_ARG, "bagel_cache_set: rank %d differs from the installed rank %d", rank, c->k);
      alloc_cache(c, rank);
    }
    CK(cudaMemcpyAsync(c->alpha64 + (size_t)m * c->N, alpha, (size_t)c->N * sizeof(double), cudaMemcpyDefault, c->stream));
    CK(cudaMemcpyAsync(c->R64 + (size_t)m * rank * c->N, R, (size_t)rank * c->N * sizeof(double), cudaMemcpyDefault,
                       c->stream));
    pack_output(c, m);
    CK(cudaStreamSynchronize(c->stream));
    c->cache_ok[m] = 1;
  });
}

extern "C" int bagel_profile(bagel_ctx* c, int enable) {
  return guarded(c, [&] {
    prof_drain(c);
    c->prof_on = enable != 0;
    if (enable)
      for (int i = 0; i < 8; ++i) {
        c->prof_ms[i] = 0.0;
        c->prof_n[i] = 0;
      }
  });
}

extern "C" int bagel_profile_get(bagel_ctx* c, int kernel, double* total_ms, long long* launches) {
  return guarded(c, [&] {
    REQUIRE(kernel >= 0 && kernel < BAGEL_PROFILE_CLASSES && total_ms && launches, BAGEL_E_ARG,
            "bagel_profile_get: kernel class %d out of range [0, %d)", kernel, BAGEL_PROFILE_CLASSES);
    prof_drain(c);
    *total_ms = c->prof_ms[kernel];
    *launches = c->prof_n[kernel];
  });
}

extern "C" int bagel_tc_selftest(bagel_ctx* c, const void* A, const void* B, int N, int K, int mode, float* D) {
  return guarded(c, [&] {
    REQUIRE(A && B && D && N >= 16 && N <= 256 && N % 16 == 0 && K >= 16 && K % 16 == 0 &&
                (size_t)(128 + N) * K * 2 <= 200 * 1024 && (mode == 0 || (mode == 1 && N + K / 2 <= 512)),
            BAGEL_E_ARG, "bagel_tc_selftest: bad shape N=%d K=%d mode=%d", N, K, mode);
    tc_selftest_launch(A, B, N, K, D, mode, c->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
  });
}

extern "C" int bagel_tc_selftest2(bagel_ctx* c, const void* A, const void* B, int N, int K, int mode, float* D) {
  return guarded(c, [&] {
    REQUIRE(A && B && D && N >= 32 && N <= 256 && N % 32 == 0 && K >= 16 && K % 16 == 0 &&
                (size_t)(128 + N / 2) * K * 2 <= 200 * 1024 && (mode == 0 || (mode == 1 && N + K / 2 <= 512)),
            BAGEL_E_ARG, "bagel_tc_selftest2: bad shape N=%d K=%d mode=%d", N, K, mode);
    tc_selftest2_launch(A, B, N, K, D, mode, c->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
  });
}

extern "C" int bagel_set_gp_kernel(bagel_ctx* c, int version) {
  return guarded(c, [&] {
    REQUIRE(version == 0 || version == 1, BAGEL_E_ARG, "bagel_set_gp_kernel: version must be 0 or 1 (got %d)", version);
    c->gp_kernel = version;
  });
}

extern "C" int bagel_get_gp_kernel(const bagel_ctx* c, int* version) {
  if (!c || !version) return BAGEL_E_ARG;
  *version = (c->gp_kernel == 1 && !c->gp.abs_target && (c->k == 0 || tc_supported(c))) ? 1 : 0;
  return BAGEL_OK;
}

extern "C" int bagel_tc_bench(bagel_ctx* c, int N, int iters, int mode, int ctas, long long* cycles) {
  return guarded(c, [&] {
    REQUIRE(cycles && N >= 16 && N <= 256 && N % 16 == 0 && iters >= 1 && ctas >= 1 && mode >= 0 &&
                (mode < 32 || ((mode == 64 || mode == 65) && N % 32 == 0 && ctas <= 74)),
            BAGEL_E_ARG, "bagel_tc_bench: bad arguments");
    tc_bench_launch(N, iters, mode, ctas, cycles, c->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
  });
}

extern "C" int bagel_debug_buffer(bagel_ctx* c, int which, void* dst, size_t bytes) {
  return guarded(c, [&] {
    const void* src = nullptr;
    size_t have = 0;
    const Workspace& w = c->ws;
    switch (which) {
      case 0: src = c->tcs.P1h; have = (size_t)w.S1tc * c->p * w.B * (1 + c->d) * sizeof(float); break;
      case 1: src = c->tcs.P1z; have = c->tcs.P1z ? tc_p1z_floats(c, w.B, w.S1tc) * sizeof(float) : 0; break;
      case 2: src = w.P2; have = (size_t)w.S2eff * c->p * w.B * (1 + BAGEL_MAX_D) * sizeof(float); break;
      case 3: src = w.mu; have = (size_t)c->p * w.B * sizeof(float); break;
      case 4: src = c->tcs.dbg1; have = c->tcs.dbg1 ? 16 * 4096 * sizeof(unsigned long long) : 0; break;
      case 6: src = c->tcs.dbg3; have = c->tcs.dbg3 ? 16 * 4096 * sizeof(unsigned long long) : 0; break;
      case 5: src = c->tcs.dbg2; have = c->tcs.dbg2 ? 16 * 4096 * sizeof(unsigned long long) : 0; break;
      default: break;
    }
    REQUIRE(src && dst && bytes <= have, BAGEL_E_ARG, "bagel_debug_buffer: buffer %d unavailable or %zu > %zu bytes",
            which, bytes, have);
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

extern "C" int bagel_debug_trace(bagel_ctx* c, int enable) {
  return guarded(c, [&] {
    dev_free(c->tcs.dbg1);
    dev_free(c->tcs.dbg2);
    dev_free(c->tcs.dbg3);
    if (enable) {
      dev_alloc(c, c->tcs.dbg3, (size_t)16 * 4096);
      CK(cudaMemsetAsync(c->tcs.dbg3, 0, 16 * 4096 * sizeof(unsigned long long), c->stream));
      dev_alloc(c, c->tcs.dbg1, (size_t)16 * 4096);
      dev_alloc(c, c->tcs.dbg2, (size_t)16 * 4096);
      CK(cudaMemsetAsync(c->tcs.dbg1, 0, 16 * 4096 * sizeof(unsigned long long), c->stream));
      CK(cudaMemsetAsync(c->tcs.dbg2, 0, 16 * 4096 * sizeof(unsigned long long), c->stream));
    }
  });
}

// ------------------------------------------------------------ Algorithm 1 around the hot path
extern "C" int bagel_sample_states(bagel_ctx* c, uint64_t seed, long long traj_offset, int B, int p, int which,
                                   const float* lo, const float* hi, float* out) {
  return guarded(c, [&] {
    REQUIRE(lo && hi && out, BAGEL_E_ARG, "bagel_sample_states: NULL argument");
    REQUIRE(B >= 1 && p >= 1 && p <= BAGEL_MAX_P && (which == 0 || which == 1), BAGEL_E_ARG,
            "bagel_sample_states: need B >= 1, 1 <= p <= %d, which in {0, 1} (B=%d, p=%d, which=%d)", BAGEL_MAX_P, B,
            p, which);
    REQUIRE(traj_offset >= 0 && traj_offset + B <= 0xffffffffLL, BAGEL_E_ARG,
            "bagel_sample_states: need 0 <= traj_offset, traj_offset + B < 2^32");
    REQUIRE(is_device_ptr(out), BAGEL_E_ARG, "bagel_sample_states: out must be device memory");
    float hb[2 * BAGEL_MAX_P];
    for (int m = 0; m < p; ++m) {
      REQUIRE(isfinite(lo[m]) && isfinite(hi[m]) && lo[m] <= hi[m], BAGEL_E_ARG,
              "bagel_sample_states: bounds[%d] = [%g, %g] must be finite with lo <= hi", m, (double)lo[m], (double)hi[m]);
      hb[m] = lo[m];
      hb[BAGEL_MAX_P + m] = hi[m];
    }
    if (!c->op_bounds) dev_alloc(c, c->op_bounds, 2 * BAGEL_MAX_P);
    CK(cudaMemcpyAsync(c->op_bounds, hb, sizeof hb, cudaMemcpyHostToDevice, c->stream));
    op_sample_uniform(seed, traj_offset, B, p, which, c->op_bounds, c->op_bounds + BAGEL_MAX_P, out, c->stream);
    CK(cudaGetLastError());
  });
}

extern "C" int policy_adam_step(bagel_ctx* c, float* params, const float* grad, float* m1, float* m2, int n,
                                long long step, float lr, float beta1, float beta2, float eps, int* skipped) {
  return guarded(c, [&] {
    REQUIRE(params && grad && m1 && m2, BAGEL_E_ARG, "policy_adam_step: NULL array argument");
    REQUIRE(n >= 1 && step >= 1, BAGEL_E_ARG, "policy_adam_step: need n >= 1 and step >= 1 (n=%d, step=%lld)", n, step);
    REQUIRE(isfinite(lr) && lr >= 0.0f && beta1 >= 0.0f && beta1 < 1.0f && beta2 >= 0.0f && beta2 < 1.0f &&
                isfinite(eps) && eps > 0.0f,
            BAGEL_E_ARG, "policy_adam_step: need lr >= 0, 0 <= beta1, beta2 < 1, eps > 0 (lr=%g b1=%g b2=%g eps=%g)",
            (double)lr, (double)beta1, (double)beta2, (double)eps);
    REQUIRE(is_device_ptr(params) && is_device_ptr(grad) && is_device_ptr(m1) && is_device_ptr(m2), BAGEL_E_ARG,
            "policy_adam_step: params, grad, m1 and m2 must be device memory");
    if (!c->op_flag) dev_alloc(c, c->op_flag, 1);
    // bias corrections in float64 on the host, rounded once
    const float bc1 = (float)(1.0 - pow((double)beta1, (double)step));
    const float bc2 = (float)(1.0 - pow((double)beta2, (double)step));
    op_adam(params, grad, m1, m2, n, lr, beta1, beta2, eps, bc1, bc2, c->op_flag, c->stream);
    CK(cudaGetLastError());
    if (skipped) {
      int f = 0;
      CK(cudaMemcpyAsync(&f, c->op_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      *skipped = f;
    }
  });
}

// ------------------------------------------------------------ GP hyperparameter learning (NEXT-1)
extern "C" int gp_log_marginal_likelihood(bagel_ctx* c, int m, const double* log_hyp, double* mll, double* grad) {
  return guarded(c, [&] {
    REQUIRE(c->N > 0, BAGEL_E_STATE, "gp_log_marginal_likelihood: no GP loaded (call gp_load first)");
    REQUIRE(m >= 0 && m < c->p, BAGEL_E_ARG, "gp_log_marginal_likelihood: output m=%d out of range [0, %d)", m, c->p);
    REQUIRE(mll, BAGEL_E_ARG, "gp_log_marginal_likelihood: mll must be non-NULL");
    const int N = c->N, d = c->d;
    REQUIRE((double)N * N * 8.0 * 2.0 < 120e9, BAGEL_E_ARG,
            "gp_log_marginal_likelihood: N=%d needs 2 N^2 float64 (%.1f GB) of workspace, above the 120 GB limit", N,
            (double)N * N * 16.0 / 1e9);
    double h[BAGEL_MAX_D + 2];
    for (int i = 0; i < d; ++i) h[i] = log_hyp ? log_hyp[i] : log((double)c->ell[(size_t)m * d + i]);
    h[d] = log_hyp ? log_hyp[d] : log((double)c->s[m]);
    h[d + 1] = log_hyp ? log_hyp[d + 1] : log((double)c->noise[m]);
    for (int i = 0; i < d + 2; ++i)
      REQUIRE(isfinite(h[i]) && fabs(h[i]) < 700.0, BAGEL_E_ARG, "gp_log_marginal_likelihood: log_hyp[%d] = %g out of range",
              i, h[i]);
    REQUIRE(exp(h[d + 1]) >= 1e-8, BAGEL_E_ARG, "gp_log_marginal_likelihood: noise exp(log_hyp[%d]) = %g must be >= 1e-8",
            d + 1, exp(h[d + 1]));
    const size_t nvec = (size_t)N + 2 + (BAGEL_MAX_D + 2) + (size_t)mll_part_count(N);
    if (c->mll_N != N) {
      dev_free(c->mll_K);
      dev_free(c->mll_Li);
      dev_free(c->mll_vec);
      c->mll_N = 0;
      dev_alloc(c, c->mll_K, (size_t)N * N);
      dev_alloc(c, c->mll_Li, (size_t)N * N);
      dev_alloc(c, c->mll_vec, nvec);
      c->mll_N = N;
    }
    if (!c->op_flag) dev_alloc(c, c->op_flag, 1);
    double* alpha = c->mll_vec;
    double* sc = alpha + N;
    double* g = sc + 2;
    double* part = g + BAGEL_MAX_D + 2;
    cudaStream_t st = c->stream;
    CK(cudaMemsetAsync(c->op_flag, 0, sizeof(int), st));
    mll_launch(c->X, c->Y + m, c->p, N, d, h, c->mll_K, c->mll_Li, alpha, sc, part, g, c->op_flag, grad != nullptr, st);
    CK(cudaGetLastError());
    int pv = 0;
    double hs[2 + BAGEL_MAX_D + 2];
    CK(cudaMemcpyAsync(&pv, c->op_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hs, sc, (2 + (size_t)(grad ? d + 2 : 0)) * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    REQUIRE(pv == 0, BAGEL_E_NUMERIC, "gp_log_marginal_likelihood: Cholesky pivot %d of output %d is <= 0 (Khat not SPD)",
            pv - 1, m);
    *mll = -0.5 * hs[1] - hs[0] - 0.5 * N * log(2.0 * M_PI);
    if (grad)
      for (int i = 0; i < d + 2; ++i) grad[i] = hs[2 + i];
  });
}

extern "C" int gp_log_marginal_likelihood_bbmm(bagel_ctx* c, int m, const double* log_hyp, int n_probes, int n_iter,
                                               int precond_rank, uint64_t seed, double* mll, double* grad,
                                               double* logdet) {
  return guarded(c, [&] {
    REQUIRE(c->N > 0, BAGEL_E_STATE, "gp_log_marginal_likelihood_bbmm: no GP loaded (call gp_load first)");
    REQUIRE(m >= 0 && m < c->p, BAGEL_E_ARG, "gp_log_marginal_likelihood_bbmm: output m=%d out of range [0, %d)", m, c->p);
    REQUIRE(mll, BAGEL_E_ARG, "gp_log_marginal_likelihood_bbmm: mll must be non-NULL");
    REQUIRE(n_probes >= 1 && n_probes <= 16, BAGEL_E_ARG, "gp_log_marginal_likelihood_bbmm: n_probes=%d not in [1, 16]",
            n_probes);
    const int N = c->N, d = c->d;
    REQUIRE(n_iter >= 1 && n_iter <= N && n_iter <= 4096, BAGEL_E_ARG,
            "gp_log_marginal_likelihood_bbmm: n_iter=%d not in [1, min(N=%d, 4096)]", n_iter, N);
    REQUIRE(precond_rank >= 0 && precond_rank <= 64 && precond_rank <= N, BAGEL_E_ARG,
            "gp_log_marginal_likelihood_bbmm: precond_rank=%d not in [0, min(N=%d, 64)]", precond_rank, N);
    const size_t need = bbmm_workspace_doubles(N, n_probes + 1, n_iter);
    REQUIRE((double)need * 8.0 < 120e9, BAGEL_E_ARG,
            "gp_log_marginal_likelihood_bbmm: N=%d needs %.1f GB of float64 workspace, above the 120 GB limit", N,
            (double)need * 8.0 / 1e9);
    double h[BAGEL_MAX_D + 2];
    for (int i = 0; i < d; ++i) h[i] = log_hyp ? log_hyp[i] : log((double)c->ell[(size_t)m * d + i]);
    h[d] = log_hyp ? log_hyp[d] : log((double)c->s[m]);
    h[d + 1] = log_hyp ? log_hyp[d + 1] : log((double)c->noise[m]);
    for (int i = 0; i < d + 2; ++i)
      REQUIRE(isfinite(h[i]) && fabs(h[i]) < 700.0, BAGEL_E_ARG,
              "gp_log_marginal_likelihood_bbmm: log_hyp[%d] = %g out of range", i, h[i]);
    REQUIRE(exp(h[d + 1]) >= 1e-8, BAGEL_E_ARG,
            "gp_log_marginal_likelihood_bbmm: noise exp(log_hyp[%d]) = %g must be >= 1e-8", d + 1, exp(h[d + 1]));
    if (c->bbmm_ws_n < need) {
      dev_free(c->bbmm_ws);
      c->bbmm_ws_n = 0;
      dev_alloc(c, c->bbmm_ws, need);
      c->bbmm_ws_n = need;
    }
    if (!c->bbmm_its) dev_alloc(c, c->bbmm_its, 32);
    double ld = 0.0, quad = 0.0;
    int rank = 0;
    const int rc = bbmm_launch(c->X, c->Y + m, c->p, N, d, h, n_probes, n_iter, precond_rank, seed, c->bbmm_ws,
                               c->bbmm_its, &ld, &quad, grad, &rank, c->stream);
    CK(cudaGetLastError());
    REQUIRE(rc != -2, BAGEL_E_CUDA, "gp_log_marginal_likelihood_bbmm: cuTensorMapEncodeTiled failed for the Khat tiles");
    REQUIRE(rc != -3, BAGEL_E_NUMERIC, "gp_log_marginal_likelihood_bbmm: sn2 I + L^T L of the preconditioner is not SPD");
    REQUIRE(rc == 0, BAGEL_E_CUDA, "gp_log_marginal_likelihood_bbmm: stream error");
    REQUIRE(isfinite(ld) && isfinite(quad), BAGEL_E_NUMERIC,
            "gp_log_marginal_likelihood_bbmm: non-finite estimate (log-det %g, quadratic form %g): Khat too "
            "ill-conditioned for %d CG iterations",
            ld, quad, n_iter);
    *mll = -0.5 * quad - 0.5 * ld - 0.5 * N * log(2.0 * M_PI);
    if (logdet) *logdet = ld;
  });
}

extern "C" int gp_target_mode(bagel_ctx* c, int absolute) {
  return guarded(c, [&] {
    REQUIRE(absolute == 0 || absolute == 1, BAGEL_E_ARG, "gp_target_mode: absolute must be 0 or 1 (got %d)", absolute);
    c->abs_target = absolute;
    c->gp.abs_target = absolute;
  });
}
