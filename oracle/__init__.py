"""float64 CPU oracle for BAGEL's hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.  The product package
(paper_2202_13638_b200) never imports it and shares no code with it.

This module is argument marshalling (numpy <-> ctypes) around
``bagel_oracle.c``; the arithmetic and its paper citations live there.

Parity pins: see tests/test_oracle_*.py.  Unpinned parts: end-to-end rollout
values at full size (no worked example in PAPER.md; pinned only through the
invariants and closed forms listed in DESIGN.md §Oracle).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bagel_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_up = C.POINTER(C.c_uint32)


def build(force: bool = False) -> str:
    """Compile liboracle.so (generic x86-64, IEEE fp64: no -ffast-math, no -march=native)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-fno-fast-math", "-ffp-contract=off", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class GP(C.Structure):
    _fields_ = [("N", C.c_int), ("d", C.c_int), ("p", C.c_int), ("k", C.c_int),
                ("X", _dp), ("ell", _dp), ("s", _dp), ("alpha", _dp), ("R", _dp), ("abs_target", C.c_int)]


class Policy(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("sizes", _ip), ("phi_mode", C.c_int), ("theta", _dp)]


class Reward(C.Structure):
    _fields_ = [("Q", _dp), ("sigma_r", C.c_double)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            L.orc_philox4x32_10.argtypes = [_up, _up, _up]
            L.orc_box_muller4.argtypes = [_up, _dp]
            L.orc_rollout_eps.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_int]
            L.orc_rollout_eps.restype = C.c_double
            L.orc_kernel_matrix.argtypes = [_dp, C.c_int, _dp, C.c_int, C.c_int, _dp, C.c_double, _dp]
            L.orc_cholesky.argtypes = [_dp, C.c_int]
            L.orc_cholesky.restype = C.c_int
            L.orc_exact_fit.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, C.c_double, C.c_double, _dp, _dp]
            L.orc_exact_fit.restype = C.c_int
            L.orc_exact_predict.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_double, _dp, _dp, _dp,
                                            C.c_int, _dp, _dp]
            L.orc_love_build.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, C.c_double, C.c_double,
                                         C.c_int, C.c_int, _dp, _dp, _dp, _ip]
            L.orc_love_build.restype = C.c_int
            L.orc_love_predict.argtypes = [C.POINTER(GP), _dp, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp]
            L.orc_reward_fn.argtypes = [C.POINTER(Reward), C.c_int, _dp, _dp]
            L.orc_reward_fn.restype = C.c_double
            L.orc_policy_act.argtypes = [C.POINTER(Policy), C.c_int, _dp, _dp, C.c_int, _dp]
            L.orc_rollout.argtypes = [C.POINTER(GP), C.POINTER(Policy), C.POINTER(Reward), _dp, _dp,
                                      C.c_int, C.c_int, C.c_uint64, C.c_longlong, C.c_longlong,
                                      C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, C.c_int, C.c_uint64]
            L.orc_rollout.restype = C.c_int
            L.orc_sample_states.argtypes = [C.c_uint64, C.c_longlong, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]
            L.orc_adam_step.argtypes = [_dp, _dp, _dp, _dp, C.c_int, C.c_longlong, C.c_double, C.c_double,
                                        C.c_double, C.c_double]
            L.orc_adam_step.restype = C.c_int
            L.orc_mll.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, _dp, _dp]
            L.orc_mll.restype = C.c_int
            L.orc_mll_bbmm.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, C.c_int, C.c_int, C.c_uint64, _dp, _dp, _dp, _dp]
            L.orc_mll_bbmm.restype = C.c_int
            L.orc_bbmm_probe.argtypes = [C.c_uint64, C.c_int, C.c_int]
            L.orc_bbmm_probe.restype = C.c_double
            L.orc_mll_bbmm_pc.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, C.c_int, C.c_int, C.c_int, C.c_uint64, _dp,
                                          _dp, _dp, _dp, C.POINTER(C.c_int)]
            L.orc_mll_bbmm_pc.restype = C.c_int
            L.orc_bbmm_gauss.argtypes = [C.c_uint64, C.c_int, C.c_int]
            L.orc_bbmm_gauss.restype = C.c_double
            L.orc_pivoted_cholesky.argtypes = [_dp, C.c_int, C.c_int, _dp, C.POINTER(C.c_int)]
            L.orc_pivoted_cholesky.restype = C.c_int
            L.orc_num_threads.restype = C.c_int
            L.orc_set_num_threads.argtypes = [C.c_int]
            _lib = L
    return _lib


def _d(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray, t=_dp):
    return a.ctypes.data_as(t) if a is not None else None


# ---------------------------------------------------------------- Philox
def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_ptr(c, _up), _ptr(k, _up), _ptr(out, _up))
    return out


def box_muller4(o) -> np.ndarray:
    o = np.ascontiguousarray(o, dtype=np.uint32)
    e = np.zeros(4)
    lib().orc_box_muller4(_ptr(o, _up), _ptr(e))
    return e


def rollout_eps(seed: int, b_global: int, t: int, m: int) -> float:
    return lib().orc_rollout_eps(seed, b_global, t, m)


# ---------------------------------------------------------------- GP
def kernel_matrix(A, B, ell, s) -> np.ndarray:
    A, B, ell = _d(A), _d(B), _d(ell)
    K = np.zeros((A.shape[0], B.shape[0]))
    lib().orc_kernel_matrix(_ptr(A), A.shape[0], _ptr(B), B.shape[0], A.shape[1], _ptr(ell), float(s), _ptr(K))
    return K


def cholesky(A):
    A = _d(A).copy()
    rc = lib().orc_cholesky(_ptr(A), A.shape[0])
    return A, rc


def exact_fit(X, y, ell, s, noise, want_L=True):
    X, y, ell = _d(X), _d(y), _d(ell)
    N, d = X.shape
    alpha = np.zeros(N)
    L = np.zeros((N, N)) if want_L else None
    rc = lib().orc_exact_fit(_ptr(X), N, d, _ptr(y), _ptr(ell), float(s), float(noise), _ptr(alpha), _ptr(L))
    if rc != 0:
        raise ArithmeticError(f"oracle Cholesky failed at pivot {rc - 1}")
    return alpha, L


def exact_predict(X, ell, s, L, alpha, xs):
    X, ell, L, alpha, xs = _d(X), _d(ell), _d(L), _d(alpha), _d(xs)
    M = xs.shape[0]
    mean, var = np.zeros(M), np.zeros(M)
    lib().orc_exact_predict(_ptr(X), X.shape[0], X.shape[1], _ptr(ell), float(s), _ptr(L), _ptr(alpha),
                            _ptr(xs), M, _ptr(mean), _ptr(var))
    return mean, var


def love_build(X, y, ell, s, noise, k, m_index=0):
    """Returns (R [k x N], a [k], b [k-1], restarts)."""
    X, y, ell = _d(X), _d(y), _d(ell)
    N, d = X.shape
    R = np.zeros((k, N))
    a = np.zeros(k)
    b = np.zeros(max(k - 1, 1))
    nr = C.c_int(0)
    rc = lib().orc_love_build(_ptr(X), N, d, _ptr(y), _ptr(ell), float(s), float(noise), m_index, k,
                              _ptr(R), _ptr(a), _ptr(b), C.byref(nr))
    if rc != 0:
        raise ArithmeticError(f"oracle LOVE build failed (rc={rc})")
    return R, a, b[: k - 1], nr.value


class Model:
    """The oracle's GP dynamics model: fp64 copies of X, hyperparameters, alpha and R."""

    def __init__(self, X, ell, s, alpha, R, abs_target=False):
        self.X = _d(X)
        self.ell = _d(ell)
        self.s = _d(s).reshape(-1)
        self.alpha = _d(alpha)
        self.R = _d(R)
        self.N, self.d = self.X.shape
        self.p = self.s.shape[0]
        self.k = self.R.shape[1]
        assert self.alpha.shape == (self.p, self.N)
        assert self.R.shape == (self.p, self.k, self.N)
        self.abs_target = bool(abs_target)  # targets y = x_{k+1} instead of Delta x
        self.struct = GP(self.N, self.d, self.p, self.k, _ptr(self.X), _ptr(self.ell), _ptr(self.s),
                         _ptr(self.alpha), _ptr(self.R), int(self.abs_target))

    @classmethod
    def build(cls, X, Y, ell, s, noise, k, abs_target=False):
        """Exact alpha (Cholesky) and naive LOVE R for every output (one-time cache)."""
        X, Y, ell, s, noise = _d(X), _d(Y), _d(ell), _d(s), _d(noise)
        p = Y.shape[1]
        alphas, Rs, restarts = [], [], []
        for m in range(p):
            a, _ = exact_fit(X, Y[:, m], ell[m], s[m], noise[m], want_L=False)
            R, _, _, nr = love_build(X, Y[:, m], ell[m], s[m], noise[m], k, m_index=m)
            alphas.append(a)
            Rs.append(R)
            restarts.append(nr)
        mdl = cls(X, ell, s, np.stack(alphas), np.stack(Rs), abs_target)
        mdl.restarts = restarts
        return mdl

    def predict(self, xs):
        """LOVE query with Jacobians: mean, var (M x p), jmu, jv (M x p x d), mbound, vbound (M x p)."""
        xs = _d(xs)
        M = xs.shape[0]
        p, d = self.p, self.d
        out = [np.zeros((M, p)), np.zeros((M, p)), np.zeros((M, p, d)), np.zeros((M, p, d)),
               np.zeros((M, p)), np.zeros((M, p))]
        lib().orc_love_predict(C.byref(self.struct), _ptr(xs), M, *[_ptr(o) for o in out])
        return tuple(out)


def reward(Q, sigma_r, x, g) -> float:
    Q, x, g = _d(Q), _d(x), _d(g)
    rw = Reward(_ptr(Q), float(sigma_r))
    return lib().orc_reward_fn(C.byref(rw), x.shape[0], _ptr(x), _ptr(g))


def policy_act(sizes, phi_mode, theta, x, g) -> np.ndarray:
    """u = pi(x, g) for every row (the oracle's tanh MLP, PyTorch nn.Sequential parameter order)."""
    x, g, theta = _d(np.atleast_2d(x)), _d(np.atleast_2d(g)), _d(theta)
    B, p = x.shape
    sz = np.ascontiguousarray(sizes, dtype=np.int32)
    pm = {"xg": 0, "xgd": 1}[phi_mode] if isinstance(phi_mode, str) else int(phi_mode)
    pol = Policy(len(sizes) - 1, sz.ctypes.data_as(_ip), pm, _ptr(theta))
    u = np.zeros((B, int(sizes[-1])))
    lib().orc_policy_act(C.byref(pol), p, _ptr(x), _ptr(g), B, _ptr(u))
    return u


def rollout(model: Model, sizes, phi_mode, theta, Q, sigma_r, x0, goals, T, seed, traj_offset=0,
            B_global=None, eps_mode=0, want_grad=True, trace=False, perturb_mode=0, perturb_seed=0):
    """Returns dict(cost, grad, ret, [x, mu, var]).  phi_mode: 'xg' or 'xgd'.
    perturb_mode (fp32-sensitivity mode): 0 exact; 1 every kernel value x (1 + U(+-2^-22));
    2 only the mean path (mu, J^mu); 3 only the variance path (z, J^v)."""
    x0, goals, theta, Q = _d(x0), _d(goals), _d(theta), _d(Q)
    B, p = x0.shape
    if B_global is None:
        B_global = B
    sz = np.ascontiguousarray(sizes, dtype=np.int32)
    pm = {"xg": 0, "xgd": 1}[phi_mode] if isinstance(phi_mode, str) else int(phi_mode)
    pol = Policy(len(sizes) - 1, sz.ctypes.data_as(_ip), pm, _ptr(theta))
    rw = Reward(_ptr(Q), float(sigma_r))
    cost = C.c_double(0.0)
    grad = np.zeros(theta.shape[0])
    ret = np.zeros(B)
    tx = np.zeros((T + 1, B, p)) if trace else None
    tm = np.zeros((T, B, p)) if trace else None
    tv = np.zeros((T, B, p)) if trace else None
    rc = lib().orc_rollout(C.byref(model.struct), C.byref(pol), C.byref(rw), _ptr(x0), _ptr(goals), B, T,
                           int(seed), int(traj_offset), int(B_global), int(eps_mode), int(bool(want_grad)),
                           C.byref(cost), _ptr(grad), _ptr(tx), _ptr(tm), _ptr(tv), _ptr(ret),
                           int(perturb_mode), int(perturb_seed))
    if rc != 0:
        t, b = divmod(rc - 1, B)
        raise FloatingPointError(f"oracle rollout: non-finite state at step {t}, row {b}")
    out = dict(cost=cost.value, grad=grad, ret=ret)
    if trace:
        out.update(x=tx, mu=tm, var=tv)
    return out


def log_marginal_likelihood(X, y, log_hyp, want_grad=True):
    """(log p(y | X, phi), d/dphi) with phi = [log l (d) | log s | log sn2] (Eq.5-6, reading R33)."""
    X, y, h = _d(X), _d(y).reshape(-1), _d(log_hyp).reshape(-1)
    N, d = X.shape
    assert h.shape == (d + 2,) and y.shape == (N,)
    val = C.c_double(0.0)
    g = np.zeros(d + 2) if want_grad else None
    rc = lib().orc_mll(_ptr(X), N, d, _ptr(y), _ptr(h), C.byref(val), _ptr(g))
    if rc != 0:
        raise ArithmeticError(f"oracle Cholesky failed at pivot {rc - 1}")
    return val.value, g


def log_marginal_likelihood_bbmm(X, y, log_hyp, n_probes, n_iter, seed, want_grad=True):
    """BBMM estimate of (log p, d/dphi) -- mBCG with n_probes Rademacher probes and exactly n_iter CG
    iterations, SLQ log-det, Hutchinson trace (NEXT-1 at large N, reading R39).  Returns
    (mll, grad or None, logdet estimate, y^T u_0)."""
    X, y, h = _d(X), _d(y).reshape(-1), _d(log_hyp).reshape(-1)
    N, d = X.shape
    assert h.shape == (d + 2,) and y.shape == (N,)
    val, ld, qd = C.c_double(0.0), C.c_double(0.0), C.c_double(0.0)
    g = np.zeros(d + 2) if want_grad else None
    rc = lib().orc_mll_bbmm(_ptr(X), N, d, _ptr(y), _ptr(h), int(n_probes), int(n_iter), int(seed), C.byref(val),
                            _ptr(g), C.byref(ld), C.byref(qd))
    if rc != 0:
        raise MemoryError("oracle BBMM: allocation failed")
    return val.value, g, ld.value, qd.value


def log_marginal_likelihood_bbmm_pc(X, y, log_hyp, n_probes, n_iter, precond_rank, seed, want_grad=True):
    """BBMM with GPyTorch's rank-k pivoted-Cholesky preconditioner (reading R40): probes z ~ N(0, P),
    preconditioned CG of exactly n_iter iterations, log|P| + SLQ log-det, Hutchinson trace with P^-1 z.
    precond_rank 0 is log_marginal_likelihood_bbmm.  Returns (mll, grad or None, logdet, y^T u_0, rank)."""
    X, y, h = _d(X), _d(y).reshape(-1), _d(log_hyp).reshape(-1)
    N, d = X.shape
    assert h.shape == (d + 2,) and y.shape == (N,)
    val, ld, qd, rk = C.c_double(0.0), C.c_double(0.0), C.c_double(0.0), C.c_int(0)
    g = np.zeros(d + 2) if want_grad else None
    rc = lib().orc_mll_bbmm_pc(_ptr(X), N, d, _ptr(y), _ptr(h), int(n_probes), int(n_iter), int(precond_rank),
                               int(seed), C.byref(val), _ptr(g), C.byref(ld), C.byref(qd), C.byref(rk))
    if rc != 0:
        raise ArithmeticError(f"oracle preconditioned BBMM failed ({rc})")
    return val.value, g, ld.value, qd.value, rk.value


def pivoted_cholesky(Kf, k):
    """(L (N x rank), pivots) of the oracle's greedy pivoted Cholesky of a PSD matrix (reading R40)."""
    Kf = _d(Kf)
    N = Kf.shape[0]
    L = np.zeros((N, k))
    piv = (C.c_int * k)()
    r = lib().orc_pivoted_cholesky(_ptr(Kf), N, int(k), _ptr(L), piv)
    return L[:, :r], np.array(piv[:r])


def bbmm_gauss(seed, i, j) -> float:
    """Gaussian g_i[j] of the preconditioned probes (Philox, Box-Muller, reading R40)."""
    return lib().orc_bbmm_gauss(int(seed), int(i), int(j))


def bbmm_probes(seed, n_probes, N) -> np.ndarray:
    """The Rademacher probes of log_marginal_likelihood_bbmm (n_probes x N)."""
    return np.array([[lib().orc_bbmm_probe(int(seed), i, n) for n in range(N)] for i in range(n_probes)])


# ---------------------------------------------------------------- Algorithm 1 around the path
def sample_states(seed: int, traj_offset: int, B: int, lo, hi, which: int = 0) -> np.ndarray:
    """S_0 (which = 0) / goals (which = 1): uniform within [lo, hi] per column."""
    lo, hi = _d(lo).reshape(-1), _d(hi).reshape(-1)
    p = lo.shape[0]
    out = np.zeros((B, p))
    lib().orc_sample_states(int(seed) & 0xFFFFFFFFFFFFFFFF, int(traj_offset), int(B), p, int(which), _ptr(lo),
                            _ptr(hi), _ptr(out))
    return out


def adam_step(theta, g, m1, m2, t: int, lr=1e-2, b1=0.9, b2=0.999, eps=1e-8) -> bool:
    """In-place bias-corrected Adam on float64 arrays.  True if skipped (non-finite g)."""
    for a in (theta, g, m1, m2):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    return bool(lib().orc_adam_step(_ptr(theta), _ptr(g), _ptr(m1), _ptr(m2), theta.shape[0], int(t), float(lr),
                                    float(b1), float(b2), float(eps)))


def train(model: Model, sizes, phi_mode, theta0, Q, sigma_r, T, iters, B, lo, hi, seed0, lr=1e-2,
          x0=None, goals=None):
    """Algorithm 1's inner loop: per iteration i (seed0 + i) sample S_0 and G (unless fixed,
    P:144), rollout cost and gradient, Adam.  Returns (theta, [cost_i])."""
    theta = _d(theta0).copy()
    m1, m2 = np.zeros_like(theta), np.zeros_like(theta)
    costs, t = [], 0
    for i in range(iters):
        seed = seed0 + i
        xs = _d(x0) if x0 is not None else sample_states(seed, 0, B, lo, hi, 0)
        gs = _d(goals) if goals is not None else sample_states(seed, 0, B, lo, hi, 1)
        out = rollout(model, sizes, phi_mode, theta, Q, sigma_r, xs, gs, T, seed)
        costs.append(out["cost"])
        if not adam_step(theta, out["grad"], m1, m2, t + 1, lr):
            t += 1
    return theta, costs


def num_threads() -> int:
    return lib().orc_num_threads()


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))
