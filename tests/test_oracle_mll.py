"""Pins of the oracle's log marginal likelihood and its gradient (Eq.5-6; reading R33) --
no GPU: closed forms at N = 1 and N = 2, brute force at N = 8 against numpy's slogdet / inverse,
central finite differences, and the SPEC S:229 sign property."""
import math

import numpy as np
import pytest

import oracle as O
from conftest import small_gp_data

LOG2PI = math.log(2.0 * math.pi)


def test_n1_closed_form():
    """N = 1: Khat = s + sn2; log p = -y^2/(2 Khat) - log(Khat)/2 - log(2 pi)/2;
    d/dlog s = s/2 (y^2/Khat^2 - 1/Khat), d/dlog sn2 likewise with sn2, d/dlog l = 0 (r = 0)."""
    X, y = np.array([[0.3, -0.2, 1.1]]), np.array([0.7])
    ell, s, sn2 = np.array([0.8, 1.3, 0.4]), 0.2, 0.05
    val, g = O.log_marginal_likelihood(X, y, np.log(np.r_[ell, s, sn2]))
    Kh = s + sn2
    assert val == pytest.approx(-0.49 / (2 * Kh) - 0.5 * math.log(Kh) - 0.5 * LOG2PI, rel=1e-14)
    assert g[:3] == pytest.approx([0.0, 0.0, 0.0], abs=1e-300)
    assert g[3] == pytest.approx(0.5 * s * (0.49 / Kh ** 2 - 1 / Kh), rel=1e-13)
    assert g[4] == pytest.approx(0.5 * sn2 * (0.49 / Kh ** 2 - 1 / Kh), rel=1e-13)


def test_n2_closed_form():
    """N = 2: Khat = [[a, k], [k, a]], a = s + sn2, k = s exp(-r^2/2), r^2 = sum_c dx_c^2 / l_c^2.
    log|Khat| = log(a^2 - k^2); y^T Khat^-1 y = (a y1^2 - 2 k y1 y2 + a y2^2) / (a^2 - k^2);
    d/dlog l_c (only k moves, dk = k dx_c^2 / l_c^2): d log p = dk (y^T Khat^-1 E Khat^-1 y - tr(Khat^-1 E)) / 2
    with E = [[0, 1], [1, 0]]."""
    X = np.array([[0.1, 0.5], [-0.4, 0.9]])
    y = np.array([0.3, -0.8])
    ell, s, sn2 = np.array([0.7, 1.5]), 0.9, 0.1
    val, g = O.log_marginal_likelihood(X, y, np.log(np.r_[ell, s, sn2]))
    dx = X[0] - X[1]
    r2c = dx ** 2 / ell ** 2
    k = s * math.exp(-0.5 * r2c.sum())
    a = s + sn2
    det = a * a - k * k
    Kinv = np.array([[a, -k], [-k, a]]) / det
    quad = (a * y[0] ** 2 - 2 * k * y[0] * y[1] + a * y[1] ** 2) / det
    assert val == pytest.approx(-0.5 * quad - 0.5 * math.log(det) - LOG2PI, rel=1e-14)
    al = Kinv @ y
    E = np.array([[0.0, 1.0], [1.0, 0.0]])
    dE = al @ E @ al - np.trace(Kinv @ E)
    for c in range(2):
        assert g[c] == pytest.approx(0.5 * k * r2c[c] * dE, rel=1e-12)
    # d/dlog s: dKhat = K (off-diagonal k, diagonal s); d/dlog sn2: sn2 I
    Ks = np.array([[s, k], [k, s]])
    assert g[2] == pytest.approx(0.5 * (al @ Ks @ al - np.trace(Kinv @ Ks)), rel=1e-12)
    assert g[3] == pytest.approx(0.5 * sn2 * (al @ al - np.trace(Kinv)), rel=1e-12)


def test_brute_force_n8_against_numpy():
    X, Y, ell, s, noise = small_gp_data(N=8, d=3, p=1, seed=4)
    y = Y[:, 0]
    h = np.log(np.r_[ell[0], s[0], noise[0]])
    val, _ = O.log_marginal_likelihood(X, y, h)
    D = ((X[:, None, :] - X[None, :, :]) / ell[0]) ** 2
    Kh = s[0] * np.exp(-0.5 * D.sum(-1)) + noise[0] * np.eye(8)
    sign, ld = np.linalg.slogdet(Kh)
    assert sign > 0
    ref = -0.5 * y @ np.linalg.solve(Kh, y) - 0.5 * ld - 4 * LOG2PI
    assert val == pytest.approx(ref, rel=1e-12)


def test_gradient_matches_central_differences():
    X, Y, ell, s, noise = small_gp_data(N=40, d=3, p=2, seed=1)
    for m in range(2):
        h = np.log(np.r_[ell[m], s[m], noise[m]])
        _, g = O.log_marginal_likelihood(X, Y[:, m], h)
        for j in range(5):
            e = np.zeros(5)
            e[j] = 1e-5
            fp, _ = O.log_marginal_likelihood(X, Y[:, m], h + e, want_grad=False)
            fm, _ = O.log_marginal_likelihood(X, Y[:, m], h - e, want_grad=False)
            fd = (fp - fm) / 2e-5
            assert g[j] == pytest.approx(fd, rel=1e-6, abs=1e-7 * np.abs(g).max())


def test_zero_targets_push_signal_variance_down():
    """y = 0 -> d/dlog s = -tr(Khat^-1 K)/2 < 0."""
    X, _, ell, s, noise = small_gp_data(N=30, d=2, p=1, seed=2)
    _, g = O.log_marginal_likelihood(X, np.zeros(30), np.log(np.r_[ell[0], s[0], noise[0]]))
    assert g[2] < 0 and g[3] < 0


# ------------------------------------------------------------------ BBMM estimate (NEXT-1 at large N, R39)
def _khat(X, ell, s, sn2):
    K = O.kernel_matrix(X, X, ell, s)
    return K + sn2 * np.eye(len(X))


def _dK(X, ell, s, sn2, j):
    d = X.shape[1]
    K = O.kernel_matrix(X, X, ell, s)
    if j < d:
        diff = X[:, None, j] - X[None, :, j]
        return K * diff ** 2 / ell[j] ** 2
    if j == d:
        return K
    return sn2 * np.eye(len(X))


def test_bbmm_probes_are_rademacher_from_philox():
    """z_i[n] = -1 iff the sign bit of Philox4x32-10(key = seed, ctr = (i, n >> 2, 0x4242424D, 4)) word
    n & 3 is set (the convention the GPU reproduces)."""
    Z = O.bbmm_probes(0x1234, 3, 9)
    for i in range(3):
        for n in range(9):
            o = O.philox4x32_10(np.array([i, n >> 2, 0x4242424D, 4], dtype=np.uint32), [0x1234, 0])
            assert Z[i, n] == (-1.0 if o[n & 3] >> 31 else 1.0)
    assert set(np.unique(Z)) <= {-1.0, 1.0}


def test_bbmm_full_krylov_is_exact_per_probe():
    """With J = N CG iterations (the Krylov space is the whole space) each probe's quadrature is exact:
    ||z||^2 e_1^T log(T) e_1 = z^T log(Khat) z, so the SLQ estimate equals (1/t) sum_i z_i^T log(Khat) z_i
    computed by numpy's eigh; y^T u_0 = y^T Khat^-1 y; the Hutchinson term equals (1/t) sum_i
    z_i^T Khat^-1 dK z_i (numpy solve) -- deterministic identities for the same probes."""
    X, Y, ell, s, noise = small_gp_data(N=24, d=3, p=1, seed=5)
    y = Y[:, 0]
    s, sn2 = float(s[0]), 0.3 * float(s[0])  # well conditioned: full CG converges to rounding
    t, seed = 5, 77
    h = np.log(np.r_[ell[0], s, sn2])
    mll, g, logdet, quad = O.log_marginal_likelihood_bbmm(X, y, h, t, len(y), seed)
    Kh = _khat(X, ell[0], s, sn2)
    lam, V = np.linalg.eigh(Kh)
    logK = (V * np.log(lam)) @ V.T
    Z = O.bbmm_probes(seed, t, len(y))
    ref_logdet = np.mean([z @ logK @ z for z in Z])
    assert logdet == pytest.approx(ref_logdet, rel=1e-9)
    assert quad == pytest.approx(y @ np.linalg.solve(Kh, y), rel=1e-9)
    assert mll == pytest.approx(-0.5 * quad - 0.5 * logdet - 0.5 * len(y) * LOG2PI, rel=1e-14)
    a = np.linalg.solve(Kh, y)
    for j in range(X.shape[1] + 2):
        D = _dK(X, ell[0], s, sn2, j)
        tr = np.mean([z @ np.linalg.solve(Kh, D @ z) for z in Z])
        assert g[j] == pytest.approx(0.5 * a @ D @ a - 0.5 * tr, rel=1e-8, abs=1e-10 * np.abs(g).max())


def test_bbmm_is_an_unbiased_estimate_of_the_exact_mll():
    """Many probes: the SLQ log-det and the Hutchinson gradient converge to the exact (Cholesky) values
    of orc_mll within a few standard errors (Rademacher probes: E[z^T A z] = tr A)."""
    X, Y, ell, s, noise = small_gp_data(N=40, d=2, p=1, seed=6)
    y = Y[:, 0]
    h = np.log(np.r_[ell[0], float(s[0]), float(noise[0]) * 10])
    exact, g_exact = O.log_marginal_likelihood(X, y, h)
    t = 600
    mll, g, logdet, quad = O.log_marginal_likelihood_bbmm(X, y, h, t, 40, 11)
    Kh = _khat(X, ell[0], np.exp(h[2]), np.exp(h[3]))
    lam, V = np.linalg.eigh(Kh)
    L = (V * np.log(lam)) @ V.T
    # Var(z^T L z) = 4 sum_{i<j} L_ij^2 for Rademacher z; the mll carries half the log-det
    sd_logdet = np.sqrt(4 * np.sum(np.triu(L, 1) ** 2) / t)
    assert abs(mll - exact) <= 4 * 0.5 * sd_logdet + 1e-9
    assert np.linalg.norm(g - g_exact) <= 0.1 * np.linalg.norm(g_exact)


def test_bbmm_fixed_iterations_and_thread_count_independent():
    X, Y, ell, s, noise = small_gp_data(N=50, d=3, p=1, seed=8)
    h = np.log(np.r_[ell[0], float(s[0]), float(noise[0])])
    n0 = O.num_threads()
    try:
        O.set_num_threads(1)
        r1 = O.log_marginal_likelihood_bbmm(X, Y[:, 0], h, 4, 20, 5)
        O.set_num_threads(max(2, n0))
        r2 = O.log_marginal_likelihood_bbmm(X, Y[:, 0], h, 4, 20, 5)
    finally:
        O.set_num_threads(n0)
    assert r1[0] == r2[0] and np.array_equal(r1[1], r2[1])


# ------------------------------------------------------------ preconditioned BBMM (reading R40)
def test_pivoted_cholesky_nystrom_properties():
    """Greedy pivoted Cholesky (Harbrecht et al.; GPyTorch's preconditioner): with equal diagonals the
    first pivot is index 0 and L[:, 0] = K[:, 0] / sqrt(K_00); L L^T reproduces K exactly on the
    pivot columns (the Nystrom interpolation property); the residual diagonal is >= 0 and its trace
    decreases with the rank; at the numerical rank of a smooth kernel L L^T = K."""
    X, Y, ell, s, noise = small_gp_data(N=40, d=2, p=1, seed=12)
    Kf = _khat(X, ell[0], float(s[0]), 0.0)
    L, piv = O.pivoted_cholesky(Kf, 6)
    assert piv[0] == 0 and len(set(piv)) == len(piv)
    np.testing.assert_allclose(L[:, 0], Kf[:, 0] / np.sqrt(Kf[0, 0]), rtol=1e-15)
    np.testing.assert_allclose((L @ L.T)[:, piv], Kf[:, piv], rtol=0, atol=1e-12 * Kf.max())
    traces = []
    for k in (1, 3, 6, 12, 24):
        Lk, _ = O.pivoted_cholesky(Kf, k)
        res = np.diag(Kf - Lk @ Lk.T)
        assert res.min() >= -1e-12 * Kf.max()
        traces.append(res.sum())
    assert all(a >= b for a, b in zip(traces, traces[1:]))
    Lf, _ = O.pivoted_cholesky(Kf, 40)
    assert np.abs(Kf - Lf @ Lf.T).max() <= 1e-8 * Kf.max()


def test_bbmm_gauss_is_box_muller_of_philox():
    """g_i[j] = Box-Muller word j & 3 of Philox4x32-10(key = seed, ctr = (i, j >> 2, 0x4242424E, 5)),
    uniforms ((o >> 9) + 0.5) 2^-23 (R29)."""
    for i, j in [(0, 0), (0, 1), (1, 2), (3, 7), (2, 13)]:
        o = O.philox4x32_10(np.array([i, j >> 2, 0x4242424E, 5], dtype=np.uint32), [0xBEEF, 0])
        u = ((o >> 9).astype(np.float64) + 0.5) * 2.0 ** -23
        r0, r1 = np.sqrt(-2 * np.log(u[0])), np.sqrt(-2 * np.log(u[2]))
        e = [r0 * np.cos(2 * np.pi * u[1]), r0 * np.sin(2 * np.pi * u[1]),
             r1 * np.cos(2 * np.pi * u[3]), r1 * np.sin(2 * np.pi * u[3])]
        assert O.bbmm_gauss(0xBEEF, i, j) == pytest.approx(e[j & 3], rel=1e-14, abs=1e-15)


def test_bbmm_pc_rank_zero_is_plain_bbmm():
    X, Y, ell, s, noise = small_gp_data(N=50, d=3, p=1, seed=9)
    h = np.log(np.r_[ell[0], float(s[0]), float(noise[0])])
    a = O.log_marginal_likelihood_bbmm(X, Y[:, 0], h, 4, 20, 5)
    b = O.log_marginal_likelihood_bbmm_pc(X, Y[:, 0], h, 4, 20, 0, 5)
    assert a[0] == b[0] and np.array_equal(a[1], b[1]) and a[2] == b[2] and b[4] == 0


def test_bbmm_pc_full_krylov_is_exact_per_probe():
    """J = N preconditioned CG: each probe's quadrature is exact for M = P^-1/2 Khat P^-1/2, so
    logdet = log|P| + (1/t) sum_i w_i^T log(M) w_i with w_i = P^-1/2 z_i, z_i = L g_i[:k] + sn g_i[k:]
    (numpy eigh of P and M); y^T u_0 = y^T Khat^-1 y; the Hutchinson term = (1/t) sum_i
    (Khat^-1 z_i)^T dK (P^-1 z_i)."""
    X, Y, ell, s, noise = small_gp_data(N=24, d=3, p=1, seed=5)
    y = Y[:, 0]
    s, sn2 = float(s[0]), 0.05 * float(s[0])
    t, seed, k = 4, 91, 5
    h = np.log(np.r_[ell[0], s, sn2])
    N = len(y)
    mll, g, logdet, quad, rank = O.log_marginal_likelihood_bbmm_pc(X, y, h, t, N, k, seed)
    assert rank == k
    Kh = _khat(X, ell[0], s, sn2)
    L, _ = O.pivoted_cholesky(Kh - sn2 * np.eye(N), k)
    P = L @ L.T + sn2 * np.eye(N)
    lp, Vp = np.linalg.eigh(P)
    Pm12 = (Vp / np.sqrt(lp)) @ Vp.T
    lm, Vm = np.linalg.eigh(Pm12 @ Kh @ Pm12)
    logM = (Vm * np.log(lm)) @ Vm.T
    Z = np.array([[O.bbmm_gauss(seed, i, j) for j in range(k + N)] for i in range(t)])
    Zs = np.array([L @ z[:k] + np.sqrt(sn2) * z[k:] for z in Z])
    ref = np.sum(np.log(lp)) + np.mean([(Pm12 @ z) @ logM @ (Pm12 @ z) for z in Zs])
    assert logdet == pytest.approx(ref, rel=1e-9)
    assert quad == pytest.approx(y @ np.linalg.solve(Kh, y), rel=1e-9)
    a = np.linalg.solve(Kh, y)
    for j in range(X.shape[1] + 2):
        D = _dK(X, ell[0], s, sn2, j)
        tr = np.mean([np.linalg.solve(Kh, z) @ D @ np.linalg.solve(P, z) for z in Zs])
        assert g[j] == pytest.approx(0.5 * a @ D @ a - 0.5 * tr, rel=1e-8, abs=1e-10 * np.abs(g).max())


def test_bbmm_pc_is_unbiased_and_preconditioning_helps():
    """(a) Many Gaussian probes: the log-det estimate is within 4 s.e. of the exact log|Khat| (Var of
    w^T A w for w ~ N(0, I) is 2 ||A||_F^2, A = log M); (b) at a short CG run (J = 8) on an
    ill-conditioned Khat the preconditioned estimate of log p is closer to the exact value than the
    unpreconditioned one, for each of 3 probe seeds."""
    X, Y, ell, s, noise = small_gp_data(N=40, d=2, p=1, seed=6)
    y = Y[:, 0]
    h = np.log(np.r_[ell[0], float(s[0]), float(noise[0]) * 10])
    exact_ld = np.linalg.slogdet(_khat(X, ell[0], np.exp(h[2]), np.exp(h[3])))[1]
    t, k = 400, 4
    _, _, logdet, _, _ = O.log_marginal_likelihood_bbmm_pc(X, y, h, t, 40, k, 13, want_grad=False)
    Kh = _khat(X, ell[0], np.exp(h[2]), np.exp(h[3]))
    L, _ = O.pivoted_cholesky(Kh - np.exp(h[3]) * np.eye(40), k)
    P = L @ L.T + np.exp(h[3]) * np.eye(40)
    lp, Vp = np.linalg.eigh(P)
    Pm12 = (Vp / np.sqrt(lp)) @ Vp.T
    lm = np.linalg.eigvalsh(Pm12 @ Kh @ Pm12)
    sd = np.sqrt(2 * np.sum(np.log(lm) ** 2) / t)
    assert abs(logdet - exact_ld) <= 4 * sd + 1e-9
    X2, Y2, ell2, s2, noise2 = small_gp_data(N=300, d=2, p=1, seed=14)
    h2 = np.log(np.r_[ell2[0], float(s2[0]), float(noise2[0])])
    exact, _ = O.log_marginal_likelihood(X2, Y2[:, 0], h2, want_grad=False)
    for seed in (1, 2, 3):
        plain = O.log_marginal_likelihood_bbmm(X2, Y2[:, 0], h2, 4, 8, seed, want_grad=False)[0]
        pc = O.log_marginal_likelihood_bbmm_pc(X2, Y2[:, 0], h2, 4, 8, 30, seed, want_grad=False)[0]
        assert abs(pc - exact) < abs(plain - exact), (seed, pc, plain, exact)
