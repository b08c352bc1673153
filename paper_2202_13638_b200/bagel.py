"""Thin ctypes binding of libbagel.so (include/bagel.h) -- argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module only
turns torch tensors / numpy arrays into pointers, sizes and the current CUDA
stream.  There is no CPU fallback: if libbagel.so is missing or fails to load,
``lib()`` raises.  Method names follow the C ABI.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np
import torch

from . import build as _build
from .build import LIB

_lock = threading.Lock()
_lib = None

E_ARG, E_NUMERIC, E_CUDA, E_STATE = 1, 2, 3, 4
_vp = C.c_void_p


class BagelError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[bagel error {code}] {msg}")
        self.code = code


def lib() -> C.CDLL:
    """Load libbagel.so (built in-tree by __graft_entry__.build()); never falls back."""
    global _lib
    with _lock:
        if _lib is None:
            # content-hash check: a stale library (sources changed since it was built) is rebuilt
            # with nvcc, never silently used; no nvcc and no library -> loud failure
            in_tree = LIB == _build.LIB
            if in_tree:
                try:
                    _build.ensure_built()
                except (OSError, subprocess.CalledProcessError) as e:
                    raise RuntimeError(f"{LIB} is missing or stale and could not be rebuilt ({e}); build it with "
                                       "`python -c 'import __graft_entry__ as g; g.build()'`") from e
            if not os.path.exists(LIB):
                raise RuntimeError(f"{LIB} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
            L = C.CDLL(LIB)
            L.bagel_build_hash.restype = C.c_char_p
            got, want = L.bagel_build_hash().decode(), _build.source_hash()
            if in_tree and got != want:
                raise RuntimeError(f"{LIB} was built from other sources (hash {got[:12]} != tree {want[:12]})")
            L.bagel_create.argtypes = [C.POINTER(_vp), C.c_int, _vp]
            L.bagel_destroy.argtypes = [_vp]
            L.bagel_set_stream.argtypes = [_vp, _vp]
            L.bagel_last_error.argtypes = [_vp]
            L.bagel_last_error.restype = C.c_char_p
            L.gp_load.argtypes = [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp]
            L.love_cache_build.argtypes = [_vp, C.c_int, C.POINTER(C.c_double)]
            L.exact_cache_build.argtypes = [_vp, C.POINTER(C.c_double)]
            L.gp_target_mode.argtypes = [_vp, C.c_int]
            L.policy_configure.argtypes = [_vp, C.POINTER(C.c_int), C.c_int]
            L.reward_configure.argtypes = [_vp, C.POINTER(C.c_float), C.c_float]
            L.rollout_cost_and_grad.argtypes = [_vp, _vp, _vp, _vp, C.c_int, C.c_int, C.c_uint64, C.c_longlong,
                                                C.c_longlong, C.POINTER(C.c_double), _vp]
            L.bagel_last_launch_count.argtypes = [_vp, C.POINTER(C.c_int)]
            L.bagel_gp_predict.argtypes = [_vp, _vp, C.c_int, _vp, _vp, _vp, _vp]
            L.bagel_rollout_trace.argtypes = [_vp, _vp, _vp, _vp, C.c_int, C.c_int, C.c_uint64, C.c_longlong,
                                              _vp, _vp, _vp, _vp]
            L.bagel_philox4x32_10.argtypes = [_vp, _vp, C.POINTER(C.c_uint32), C.c_int, _vp]
            L.bagel_philox_normals.argtypes = [_vp, C.c_uint64, C.c_longlong, C.c_int, C.c_int, C.c_int, _vp]
            L.bagel_cache_rank.argtypes = [_vp, C.POINTER(C.c_int)]
            L.bagel_cache_get.argtypes = [_vp, C.c_int, _vp, _vp]
            L.bagel_cache_set.argtypes = [_vp, C.c_int, C.c_int, _vp, _vp]
            L.bagel_profile.argtypes = [_vp, C.c_int]
            L.bagel_profile_get.argtypes = [_vp, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_longlong)]
            L.bagel_tc_selftest.argtypes = [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, _vp]
            L.bagel_set_gp_kernel.argtypes = [_vp, C.c_int]
            L.bagel_tc_selftest2.argtypes = [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, _vp]
            L.bagel_tc_bench.argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp]
            L.bagel_debug_buffer.argtypes = [_vp, C.c_int, _vp, C.c_size_t]
            L.bagel_debug_trace.argtypes = [_vp, C.c_int]
            L.bagel_get_gp_kernel.argtypes = [_vp, C.POINTER(C.c_int)]
            L.bagel_sample_states.argtypes = [_vp, C.c_uint64, C.c_longlong, C.c_int, C.c_int, C.c_int,
                                              C.POINTER(C.c_float), C.POINTER(C.c_float), _vp]
            L.gp_log_marginal_likelihood.argtypes = [_vp, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                                     C.POINTER(C.c_double)]
            L.gp_log_marginal_likelihood_bbmm.argtypes = [_vp, C.c_int, C.POINTER(C.c_double), C.c_int, C.c_int,
                                                          C.c_int, C.c_uint64, C.POINTER(C.c_double),
                                                          C.POINTER(C.c_double), C.POINTER(C.c_double)]
            L.policy_adam_step.argtypes = [_vp, _vp, _vp, _vp, _vp, C.c_int, C.c_longlong, C.c_float, C.c_float,
                                           C.c_float, C.c_float, C.POINTER(C.c_int)]
            _lib = L
    return _lib


EXPORTS = ["bagel_create", "bagel_destroy", "bagel_set_stream", "bagel_last_error", "bagel_build_hash", "gp_load", "love_cache_build",
           "policy_configure", "reward_configure", "rollout_cost_and_grad", "bagel_last_launch_count",
           "bagel_gp_predict", "bagel_rollout_trace", "bagel_philox4x32_10", "bagel_philox_normals",
           "bagel_cache_rank", "bagel_cache_get", "bagel_cache_set", "bagel_profile", "bagel_profile_get", "bagel_tc_selftest",
           "bagel_set_gp_kernel", "bagel_get_gp_kernel", "bagel_tc_bench", "bagel_tc_selftest2",
           "bagel_debug_buffer", "bagel_debug_trace", "bagel_sample_states", "policy_adam_step",
           "gp_log_marginal_likelihood", "gp_log_marginal_likelihood_bbmm", "exact_cache_build",
           "gp_target_mode"]

PROFILE_CLASSES = ["gp_pass1", "gp_reduce1", "gp_pass2", "step_epilogue", "init", "reverse", "reduce", "theta_grad"]


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    raise TypeError(type(t))


def _f32(a, device=None):
    """Contiguous float32 tensor (kept on its device unless `device` is given)."""
    if isinstance(a, np.ndarray):
        a = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
    t = a.to(dtype=torch.float32) if a.dtype != torch.float32 else a
    if device is not None:
        t = t.to(device)
    return t.contiguous()


class Context:
    """One bagel_ctx per GPU / rank (not thread-safe)."""

    def __init__(self, device: int | None = None, stream: torch.cuda.Stream | None = None):
        self.L = lib()
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.dev = torch.device("cuda", self.device)
        self.stream = stream or torch.cuda.current_stream(self.dev)
        h = _vp()
        self._check(self.L.bagel_create(C.byref(h), self.device, _vp(self.stream.cuda_stream)), ctx=None)
        self.h = h
        self.p = self.d = self.N = 0
        self.n_params = 0

    def close(self):
        if getattr(self, "h", None):
            self.L.bagel_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int, ctx=True):
        if rc != 0:
            msg = self.L.bagel_last_error(self.h).decode() if ctx and self.h else "bagel_create failed"
            raise BagelError(rc, msg)

    def set_stream(self, stream: torch.cuda.Stream):
        self.stream = stream
        self._check(self.L.bagel_set_stream(self.h, _vp(stream.cuda_stream)))

    # ------------------------------------------------------------ model
    def gp_load(self, X, Y, lengthscales, outputscale, noise):
        X, Y = _f32(X, self.dev), _f32(Y, self.dev)
        ell, s, sn = _f32(lengthscales, self.dev), _f32(outputscale, self.dev), _f32(noise, self.dev)
        N, d = X.shape
        p = Y.shape[1]
        self._check(self.L.gp_load(self.h, _ptr(X), _ptr(Y), N, d, p, _ptr(ell), _ptr(s), _ptr(sn)))
        self.N, self.d, self.p = N, d, p
        self._ell = ell.double().cpu().numpy().reshape(p, d)
        self._s = s.double().cpu().numpy().reshape(p)
        self._noise = sn.double().cpu().numpy().reshape(p)

    def love_cache_build(self, rank: int) -> float:
        sec = C.c_double(0.0)
        self._check(self.L.love_cache_build(self.h, int(rank), C.byref(sec)))
        return sec.value

    def gp_target_mode(self, absolute: bool):
        """False (default): Delta targets, x' = x + f; True: absolute targets, x' = f."""
        self._check(self.L.gp_target_mode(self.h, int(bool(absolute))))

    def exact_cache_build(self) -> float:
        """Exact-GP cache (R = L^-1 at rank N, N <= 8192): exact Eq.3 variances from here on."""
        sec = C.c_double(0.0)
        self._check(self.L.exact_cache_build(self.h, C.byref(sec)))
        return sec.value

    def policy_configure(self, sizes):
        arr = (C.c_int * len(sizes))(*[int(s) for s in sizes])
        self._check(self.L.policy_configure(self.h, arr, len(sizes)))
        self.n_params = int(sum((sizes[i] + 1) * sizes[i + 1] for i in range(len(sizes) - 1)))

    def reward_configure(self, Q, sigma_r: float = 1.0):
        q = np.ascontiguousarray(Q, dtype=np.float32)
        self._check(self.L.reward_configure(self.h, q.ctypes.data_as(C.POINTER(C.c_float)), float(sigma_r)))

    # ------------------------------------------------------------ hot path
    def rollout_cost_and_grad(self, theta, x0, goals, T: int, seed: int, traj_offset: int = 0,
                              B_global: int | None = None, grad=None):
        """Returns (this rank's share of L, dL/dtheta).  Tensors may live on the GPU or on the host
        (host buffers are staged by the library); `grad` (optional) is written in place."""
        B = int(x0.shape[0])
        if B_global is None:
            B_global = B
        if grad is None:
            grad = torch.empty(self.n_params, dtype=torch.float32, device=self.dev)
        cost = C.c_double(0.0)
        self._check(self.L.rollout_cost_and_grad(self.h, _ptr(theta), _ptr(x0), _ptr(goals), B, int(T),
                                                 int(seed) & 0xFFFFFFFFFFFFFFFF, int(traj_offset), int(B_global),
                                                 C.byref(cost), _ptr(grad)))
        return cost.value, grad

    def loaded_log_hyp(self, m: int) -> np.ndarray:
        """phi of output m as loaded by gp_load: [log l (d) | log s | log sn2]."""
        return np.log(np.r_[self._ell[m], self._s[m], self._noise[m]]).astype(np.float64)

    def log_marginal_likelihood(self, m: int, log_hyp=None, want_grad: bool = True):
        """(log p(y_m | X, phi), d/dphi) with phi = [log l (d) | log s | log sn2] (Eq.5-6);
        log_hyp None = the loaded hyperparameters.  The gradient is None unless want_grad."""
        dp = C.POINTER(C.c_double)
        h = None if log_hyp is None else np.ascontiguousarray(log_hyp, dtype=np.float64)
        if h is not None and h.shape != (self.d + 2,):
            raise ValueError(f"log_hyp must have d + 2 = {self.d + 2} entries")
        val = C.c_double(0.0)
        g = np.zeros(self.d + 2) if want_grad else None
        self._check(self.L.gp_log_marginal_likelihood(self.h, int(m), None if h is None else h.ctypes.data_as(dp),
                                                      C.byref(val), None if g is None else g.ctypes.data_as(dp)))
        return val.value, g

    def log_marginal_likelihood_bbmm(self, m: int, log_hyp=None, n_probes: int = 8, n_iter: int = 100,
                                     seed: int = 0, want_grad: bool = True, precond_rank: int = 0):
        """BBMM estimate (readings R39 / R40) of (log p(y_m | X, phi), d/dphi, log|Khat|): one batched
        (preconditioned) CG of exactly n_iter iterations on [y | z_1 .. z_t], SLQ log-det, Hutchinson trace;
        precond_rank k > 0 adds GPyTorch's rank-k pivoted-Cholesky preconditioner (Gaussian probes)."""
        dp = C.POINTER(C.c_double)
        h = None if log_hyp is None else np.ascontiguousarray(log_hyp, dtype=np.float64)
        if h is not None and h.shape != (self.d + 2,):
            raise ValueError(f"log_hyp must have d + 2 = {self.d + 2} entries")
        val, ld = C.c_double(0.0), C.c_double(0.0)
        g = np.zeros(self.d + 2) if want_grad else None
        self._check(self.L.gp_log_marginal_likelihood_bbmm(
            self.h, int(m), None if h is None else h.ctypes.data_as(dp), int(n_probes), int(n_iter),
            int(precond_rank), int(seed) & 0xFFFFFFFFFFFFFFFF, C.byref(val), None if g is None else g.ctypes.data_as(dp), C.byref(ld)))
        return val.value, g, ld.value

    # ------------------------------------------------------------ Algorithm 1 around the path
    def sample_states(self, seed: int, traj_offset: int, B: int, lo, hi, which: int = 0, out=None):
        """S_0 (which = 0) or goals (which = 1) uniform in [lo, hi] per state column."""
        lo = np.ascontiguousarray(lo, dtype=np.float32).reshape(-1)
        hi = np.ascontiguousarray(hi, dtype=np.float32).reshape(-1)
        p = lo.shape[0]
        if out is None:
            out = torch.empty(B, p, dtype=torch.float32, device=self.dev)
        fp = C.POINTER(C.c_float)
        self._check(self.L.bagel_sample_states(self.h, int(seed) & 0xFFFFFFFFFFFFFFFF, int(traj_offset), int(B), p,
                                               int(which), lo.ctypes.data_as(fp), hi.ctypes.data_as(fp), _ptr(out)))
        return out

    def adam_step(self, params, grad, m1, m2, step: int, lr: float = 1e-2, beta1: float = 0.9,
                  beta2: float = 0.999, eps: float = 1e-8, report_skip: bool = False):
        """In-place Adam update of device tensors.  Returns True if the update was skipped
        because of a non-finite gradient (only when report_skip, which synchronises)."""
        sk = C.c_int(0)
        self._check(self.L.policy_adam_step(self.h, _ptr(params), _ptr(grad), _ptr(m1), _ptr(m2), int(params.numel()),
                                            int(step), float(lr), float(beta1), float(beta2), float(eps),
                                            C.byref(sk) if report_skip else None))
        return bool(sk.value)

    def last_launch_count(self) -> int:
        n = C.c_int(0)
        self._check(self.L.bagel_last_launch_count(self.h, C.byref(n)))
        return n.value

    def profile(self, enable: bool):
        self._check(self.L.bagel_profile(self.h, int(bool(enable))))

    def profile_get(self) -> dict:
        """{kernel class: (total device ms, launches)} since profile(True)."""
        out = {}
        for i, name in enumerate(PROFILE_CLASSES):
            ms, n = C.c_double(0.0), C.c_longlong(0)
            self._check(self.L.bagel_profile_get(self.h, i, C.byref(ms), C.byref(n)))
            out[name] = (ms.value, n.value)
        return out

    # ------------------------------------------------------------ test exports
    def gp_predict(self, xstar):
        xs = _f32(xstar, self.dev)
        M = xs.shape[0]
        mean = torch.empty(M, self.p, device=self.dev)
        var = torch.empty(M, self.p, device=self.dev)
        dmean = torch.empty(M, self.p, self.d, device=self.dev)
        dvar = torch.empty(M, self.p, self.d, device=self.dev)
        self._check(self.L.bagel_gp_predict(self.h, _ptr(xs), M, _ptr(mean), _ptr(var), _ptr(dmean), _ptr(dvar)))
        return mean, var, dmean, dvar

    def rollout_trace(self, theta, x0, goals, T: int, seed: int, traj_offset: int = 0):
        th, x0d, gd = _f32(theta, self.dev), _f32(x0, self.dev), _f32(goals, self.dev)
        B = x0d.shape[0]
        x = torch.empty(T + 1, B, self.p, device=self.dev)
        mu = torch.empty(max(T, 1), B, self.p, device=self.dev)
        var = torch.empty(max(T, 1), B, self.p, device=self.dev)
        ret = torch.empty(B, device=self.dev)
        self._check(self.L.bagel_rollout_trace(self.h, _ptr(th), _ptr(x0d), _ptr(gd), B, int(T), int(seed),
                                               int(traj_offset), _ptr(x), _ptr(mu), _ptr(var), _ptr(ret)))
        return dict(x=x, mu=mu[:T], var=var[:T], ret=ret)

    def philox4x32_10(self, ctr, key):
        c = torch.as_tensor(np.ascontiguousarray(ctr, dtype=np.uint32).view(np.int32)).to(self.dev)
        n = c.numel() // 4
        out = torch.empty_like(c)
        k = (C.c_uint32 * 2)(*[int(v) for v in key])
        self._check(self.L.bagel_philox4x32_10(self.h, _ptr(c), k, n, _ptr(out)))
        return out.cpu().numpy().view(np.uint32).reshape(-1, 4)

    def philox_normals(self, seed: int, traj_offset: int, B: int, T: int, p: int):
        out = torch.empty(T, B, p, device=self.dev)
        self._check(self.L.bagel_philox_normals(self.h, int(seed), int(traj_offset), B, T, p, _ptr(out)))
        return out

    def set_gp_kernel(self, version: int):
        """1: tcgen05 tensor-core GP step (default); 0: v0 CUDA-core FFMA reference."""
        self._check(self.L.bagel_set_gp_kernel(self.h, int(version)))

    def gp_kernel(self) -> int:
        v = C.c_int(0)
        self._check(self.L.bagel_get_gp_kernel(self.h, C.byref(v)))
        return v.value

    def tc_selftest(self, A: torch.Tensor, B_packed: torch.Tensor, N: int, K: int, mode: int = 0) -> torch.Tensor:
        D = torch.empty(128, N, dtype=torch.float32, device=self.dev)
        self._check(self.L.bagel_tc_selftest(self.h, _ptr(A), _ptr(B_packed), int(N), int(K), int(mode), _ptr(D)))
        return D

    def tc_selftest2(self, A_packed: torch.Tensor, B_packed: torch.Tensor, N: int, K: int, mode: int = 0) -> torch.Tensor:
        D = torch.empty(256, N, dtype=torch.float32, device=self.dev)
        self._check(self.L.bagel_tc_selftest2(self.h, _ptr(A_packed), _ptr(B_packed), int(N), int(K), int(mode),
                                              _ptr(D)))
        return D

    def tc_bench(self, N: int, iters: int, mode: int = 0, ctas: int = 1) -> np.ndarray:
        cyc = torch.zeros(ctas, dtype=torch.int64, device=self.dev)
        self._check(self.L.bagel_tc_bench(self.h, int(N), int(iters), int(mode), int(ctas), _ptr(cyc)))
        return cyc.cpu().numpy()

    def debug_buffer(self, which: int, n_floats: int) -> np.ndarray:
        out = np.empty(n_floats, dtype=np.float32)
        self._check(self.L.bagel_debug_buffer(self.h, int(which), out.ctypes.data, out.nbytes))
        return out

    def debug_trace(self, enable: bool):
        self._check(self.L.bagel_debug_trace(self.h, int(bool(enable))))

    def debug_stamps(self, which: int) -> np.ndarray:
        out = np.empty(16 * 4096, dtype=np.uint64)
        self._check(self.L.bagel_debug_buffer(self.h, int(which), out.ctypes.data, out.nbytes))
        return out.reshape(4096, 16)

    def cache_rank(self) -> int:
        k = C.c_int(0)
        self._check(self.L.bagel_cache_rank(self.h, C.byref(k)))
        return k.value

    def cache_get(self, m: int):
        k = self.cache_rank()
        alpha = torch.empty(self.N, dtype=torch.float64, device=self.dev)
        R = torch.empty(k, self.N, dtype=torch.float64, device=self.dev)
        self._check(self.L.bagel_cache_get(self.h, int(m), _ptr(alpha), _ptr(R)))
        return alpha, R

    def cache_set(self, m: int, alpha, R):
        a = torch.as_tensor(alpha, dtype=torch.float64).to(self.dev).contiguous()
        r = torch.as_tensor(R, dtype=torch.float64).to(self.dev).contiguous()
        self._check(self.L.bagel_cache_set(self.h, int(m), int(r.shape[0]), _ptr(a), _ptr(r)))


def setup(wl, rank: int | None = None, device: int | None = None, build_cache: bool = True) -> Context:
    """Context with the workload's GP, LOVE cache, policy and reward configured."""
    ctx = Context(device)
    ctx.gp_load(wl.X, wl.Y, wl.ell, wl.s, wl.noise)
    if build_cache:
        ctx.cache_seconds = ctx.love_cache_build(wl.rank if rank is None else rank)
    ctx.policy_configure(wl.sizes)
    ctx.reward_configure(wl.Q, wl.sigma_r)
    return ctx
