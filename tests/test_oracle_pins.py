"""Pins for the float64 oracle (no GPU).  Each test ties the oracle to something
other than itself: known-answer vectors, printed worked values, closed forms,
brute-force inverses, theorems (LOVE rank N = exact, Galerkin monotonicity),
limits, and finite differences."""
import math

import numpy as np
import pytest

import oracle as O
from conftest import read_golden, small_gp_data, spec_examples


# ------------------------------------------------------------------ Philox
def test_philox_kat():
    rows = read_golden("philox_kat.txt")
    assert len(rows) == 3
    for row in rows:
        v = [int(x, 16) for x in row.split()]
        out = O.philox4x32_10(v[0:4], v[4:6])
        assert list(out) == v[6:10], row


def test_box_muller_convention_and_statistics():
    # u = ((o >> 9) + 0.5) 2^-23 lies strictly in (0,1) for the extreme words.
    e = O.box_muller4([0, 0xFFFFFFFF, 0xFFFFFFFF, 0])
    assert np.all(np.isfinite(e))
    bound = math.sqrt(-2.0 * math.log(0.5 * 2.0 ** -23))  # max |eps| ~ 5.77
    assert np.all(np.abs(e) <= bound + 1e-12)
    # u0 = (0 + .5) 2^-23, u1 = (2^23 - .5) 2^-23: eps0 = r cos(2 pi u1) ~ r, eps1 ~ 0-
    assert e[0] == pytest.approx(bound * math.cos(2 * math.pi * (2 ** 23 - 0.5) / 2 ** 23), rel=1e-12)
    # moments of 4 * 50_000 draws (3-sigma bounds)
    n = 50_000
    draws = np.array([O.rollout_eps(1234, b, 0, m) for b in range(n // 4) for m in range(4)])
    assert abs(draws.mean()) < 3 / math.sqrt(draws.size) * 1.0 + 1e-12
    assert abs(draws.var() - 1.0) < 3 * math.sqrt(2.0 / draws.size)


def test_rollout_eps_counter_layout():
    # eps_{b,t,m} = BoxMuller(Philox(key=(seed lo, seed hi), ctr=(b, t, m>>2, 0)))[m & 3]
    seed = (7 << 32) | 0x5EED0003
    o = O.philox4x32_10([11, 5, 0, 0], [seed & 0xFFFFFFFF, seed >> 32])
    e = O.box_muller4(o)
    for m in range(4):
        assert O.rollout_eps(seed, 11, 5, m) == e[m]
    o2 = O.philox4x32_10([11, 5, 1, 0], [seed & 0xFFFFFFFF, seed >> 32])
    assert O.rollout_eps(seed, 11, 5, 5) == O.box_muller4(o2)[1]


# ------------------------------------------------------------------ kernel (Eq.4)
def test_kernel_special_values():
    ex = spec_examples()
    # unit hyperparameters, squared distance 2 -> exp(-1)
    K = O.kernel_matrix([[0.0, 0.0]], [[1.0, 1.0]], [1.0, 1.0], 1.0)
    assert K[0, 0] == pytest.approx(float(ex["kernel_unit_dist2"]), abs=5e-7)
    assert K[0, 0] == pytest.approx(math.exp(-1.0), rel=1e-15)
    # k(x,x) = s
    x = np.array([[0.3, -1.2, 2.0]])
    assert O.kernel_matrix(x, x, [0.5, 2.0, 3.0], 2.5)[0, 0] == 2.5
    # ARD: displacement of exactly l_c along one axis gives s e^{-1/2}, whatever the other l's
    ell = np.array([0.3, 1.7, 4.0])
    for c in range(3):
        b = x.copy()
        b[0, c] += ell[c]
        assert O.kernel_matrix(x, b, ell, 1.5)[0, 0] == pytest.approx(1.5 * math.exp(-0.5), rel=1e-14)


def test_kernel_matrix_symmetry():
    X, _, ell, s, _ = small_gp_data(N=12)
    K = O.kernel_matrix(X, X, ell[0], s[0])
    assert np.array_equal(K, K.T)
    assert np.all(np.linalg.eigvalsh(K) > -1e-12)


# ------------------------------------------------------------------ Cholesky / exact GP (Eq.2-3)
def test_cholesky_worked_example_and_failure():
    ex = [float(v) for v in spec_examples()["cholesky_4223"].split(",")]
    L, rc = O.cholesky([[4.0, 2.0], [2.0, 3.0]])
    assert rc == 0
    assert np.allclose(L, np.array(ex).reshape(2, 2), atol=1e-8)
    assert L[1, 1] == pytest.approx(math.sqrt(2.0), rel=1e-15)
    A = np.array([[1.0, 2.0, 0.0], [2.0, 1.0, 0.0], [0.0, 0.0, 1.0]])  # indefinite at pivot 1
    _, rc = O.cholesky(A)
    assert rc == 2  # pivot index 1, reported + 1


@pytest.mark.parametrize("N", [1, 2, 5, 8])
def test_exact_alpha_vs_gauss_jordan(N):
    X, Y, ell, s, noise = small_gp_data(N=N, seed=N)
    Kh = O.kernel_matrix(X, X, ell[0], s[0]) + noise[0] * np.eye(N)
    alpha, L = O.exact_fit(X, Y[:, 0], ell[0], s[0], noise[0])
    inv = _gauss_jordan_inverse(Kh)
    assert np.allclose(alpha, inv @ Y[:, 0], rtol=1e-11, atol=1e-13 * np.abs(inv @ Y[:, 0]).max())
    assert np.linalg.norm(Kh @ alpha - Y[:, 0]) <= 1e-12 * np.linalg.norm(Y[:, 0])
    assert np.allclose(L @ L.T, Kh, rtol=0, atol=1e-14 * np.abs(Kh).max())
    # exact variance vs explicit inverse: s - k^T Khat^-1 k
    xs = np.random.default_rng(1).uniform(-2, 2, size=(6, X.shape[1]))
    mean, var = O.exact_predict(X, ell[0], s[0], L, alpha, xs)
    kx = O.kernel_matrix(xs, X, ell[0], s[0])
    assert np.allclose(mean, kx @ (inv @ Y[:, 0]), rtol=1e-10, atol=1e-14)
    assert np.allclose(var, s[0] - np.einsum("in,nm,im->i", kx, inv, kx), rtol=1e-9, atol=1e-14)


def _gauss_jordan_inverse(A):
    """Brute-force explicit inverse (partial pivoting Gauss-Jordan), independent of Cholesky."""
    n = A.shape[0]
    M = np.concatenate([A.astype(float).copy(), np.eye(n)], axis=1)
    for c in range(n):
        piv = c + int(np.argmax(np.abs(M[c:, c])))
        M[[c, piv]] = M[[piv, c]]
        M[c] /= M[c, c]
        for r in range(n):
            if r != c:
                M[r] -= M[r, c] * M[c]
    return M[:, n:]


def test_exact_n1_closed_form():
    X = np.array([[0.2, -0.4]])
    y = np.array([0.7])
    ell, s, noise = np.array([0.9, 1.3]), 0.8, 0.05
    alpha, L = O.exact_fit(X, y, ell, s, noise)
    assert alpha[0] == pytest.approx(0.7 / (s + noise), rel=1e-15)
    xs = np.array([[1.0, 0.5]])
    k = s * math.exp(-0.5 * ((0.8 / 0.9) ** 2 + (0.9 / 1.3) ** 2))
    mean, var = O.exact_predict(X, ell, s, L, alpha, xs)
    assert mean[0] == pytest.approx(k * 0.7 / (s + noise), rel=1e-14)
    assert var[0] == pytest.approx(s - k * k / (s + noise), rel=1e-14)


def test_exact_n2_closed_form_variance():
    X = np.array([[0.0], [1.0]])
    y = np.array([1.0, -0.5])
    ell, s, noise = np.array([1.0]), 1.0, 0.1
    k12 = math.exp(-0.5)
    a, b, c = s + noise, k12, s + noise
    det = a * c - b * b
    inv = np.array([[c, -b], [-b, a]]) / det
    alpha, L = O.exact_fit(X, y, ell, s, noise)
    assert np.allclose(alpha, inv @ y, rtol=1e-14)
    xs = np.array([[0.3]])
    kx = np.array([math.exp(-0.5 * 0.09), math.exp(-0.5 * 0.49)])
    mean, var = O.exact_predict(X, ell, s, L, alpha, xs)
    assert mean[0] == pytest.approx(kx @ inv @ y, rel=1e-13)
    assert var[0] == pytest.approx(1.0 - kx @ inv @ kx, rel=1e-12)


def test_interpolation_and_far_field_limits():
    X, Y, ell, s, _ = small_gp_data(N=30, seed=3)
    # noise -> 1e-8: mean at a training input -> y (1e-3), var < 1e-4
    alpha, L = O.exact_fit(X, Y[:, 0], ell[0], s[0], 1e-8)
    mean, var = O.exact_predict(X, ell[0], s[0], L, alpha, X[:5])
    assert np.all(np.abs(mean - Y[:5, 0]) < 1e-3)
    assert np.all(var < 1e-4)
    # far field -> mean 0, var s
    far = np.full((2, X.shape[1]), 1e3)
    mean, var = O.exact_predict(X, ell[0], s[0], L, alpha, far)
    assert np.all(np.abs(mean) < 1e-12)
    assert np.allclose(var, s[0], rtol=1e-14)


def test_mean_linear_in_y():
    X, Y, ell, s, noise = small_gp_data(N=20, seed=4)
    a1, L = O.exact_fit(X, Y[:, 0], ell[0], s[0], noise[0])
    a2, _ = O.exact_fit(X, 2.0 * Y[:, 0], ell[0], s[0], noise[0])
    assert np.allclose(a2, 2.0 * a1, rtol=1e-14, atol=0)


# ------------------------------------------------------------------ LOVE
def _love_model(X, Y, ell, s, noise, k):
    return O.Model.build(X, Y, ell, s, noise, k)


def test_love_full_rank_equals_exact():
    X, Y, ell, s, noise = small_gp_data(N=60, p=2, seed=5)
    mdl = _love_model(X, Y, ell, s, noise, k=60)
    xs = np.random.default_rng(2).uniform(-2.5, 2.5, size=(25, X.shape[1]))
    mean, var, *_ = mdl.predict(xs)
    for m in range(2):
        alpha, L = O.exact_fit(X, Y[:, m], ell[m], s[m], noise[m])
        em, ev = O.exact_predict(X, ell[m], s[m], L, alpha, xs)
        assert np.allclose(mean[:, m], em, rtol=1e-12, atol=1e-15)
        assert np.max(np.abs(var[:, m] - ev)) < 1e-10 * s[m]


def test_love_restart_path_full_rank_equals_exact():
    """An eigenvector probe makes the Krylov space invariant after one step: the
    breakdown test fires and the Philox restart must still reach the exact variance."""
    X, Y, ell, s, noise = small_gp_data(N=24, p=1, seed=6)
    Kh = O.kernel_matrix(X, X, ell[0], s[0]) + noise[0] * np.eye(24)
    w, V = np.linalg.eigh(Kh)
    probe = V[:, -1].copy()
    R, a, b, restarts = O.love_build(X, probe, ell[0], s[0], noise[0], 24)
    assert restarts >= 1
    assert b[0] == 0.0
    alpha, L = O.exact_fit(X, probe, ell[0], s[0], noise[0])
    xs = np.random.default_rng(3).uniform(-2, 2, size=(10, X.shape[1]))
    kx = O.kernel_matrix(xs, X, ell[0], s[0])
    _, ev = O.exact_predict(X, ell[0], s[0], L, alpha, xs)
    vl = s[0] - np.sum((kx @ R.T) ** 2, axis=1)
    assert np.max(np.abs(vl - ev)) < 1e-10 * s[0]


def test_love_galerkin_monotone_in_rank():
    """v_exact <= v_love(k) <= v_love(k-1) <= s: Q (Q^T Khat Q)^-1 Q^T <= Khat^-1 on nested subspaces."""
    X, Y, ell, s, noise = small_gp_data(N=80, p=1, seed=7)
    xs = np.random.default_rng(4).uniform(-2, 2, size=(40, X.shape[1]))
    kx = O.kernel_matrix(xs, X, ell[0], s[0])
    alpha, L = O.exact_fit(X, Y[:, 0], ell[0], s[0], noise[0])
    _, ev = O.exact_predict(X, ell[0], s[0], L, alpha, xs)
    prev = np.full(xs.shape[0], s[0])
    tol = 1e-12 * s[0]
    for k in (1, 2, 4, 8, 16, 32, 64, 80):
        R, a, b, _ = O.love_build(X, Y[:, 0], ell[0], s[0], noise[0], k)
        v = s[0] - np.sum((kx @ R.T) ** 2, axis=1)
        assert np.all(v <= prev + tol), k
        assert np.all(v >= ev - 1e-10 * s[0]), k
        prev = v
    assert np.max(np.abs(prev - ev)) < 1e-10 * s[0]


def test_love_tridiagonal_is_projection():
    """T = Q^T Khat Q: the Lanczos coefficients reproduce R^T R ~ Q T^-1 Q^T, checked as
    R Khat R^T = I (R = L_T^-1 Q^T, T = L_T L_T^T)."""
    X, Y, ell, s, noise = small_gp_data(N=50, p=1, seed=8)
    Kh = O.kernel_matrix(X, X, ell[0], s[0]) + noise[0] * np.eye(50)
    R, a, b, _ = O.love_build(X, Y[:, 0], ell[0], s[0], noise[0], 20)
    assert np.allclose(R @ Kh @ R.T, np.eye(20), atol=1e-9)


def test_constant_kernel_closed_form():
    """l = 1e7: K -> s 11^T, mu = s sum(y)/(N s + sigma^2), v = s sigma^2/(N s + sigma^2);
    1 is in span{y, Khat y} so LOVE rank >= 2 is exact."""
    rng = np.random.default_rng(9)
    N = 300
    X = rng.uniform(-2, 2, size=(N, 3))
    Y = rng.normal(size=(N, 1)) * 0.3 + 0.1
    ell = np.full((1, 3), 1e7)
    s, noise = np.array([0.5]), np.array([0.01])
    xs = rng.uniform(-2, 2, size=(5, 3))
    mu_cf = s[0] * Y[:, 0].sum() / (N * s[0] + noise[0])
    v_cf = s[0] * noise[0] / (N * s[0] + noise[0])
    for k in (2, 3, 8):
        mdl = O.Model.build(X, Y, ell, s, noise, k)
        mean, var, jmu, jv, _, _ = mdl.predict(xs)
        assert np.allclose(mean[:, 0], mu_cf, rtol=1e-6)
        assert np.allclose(var[:, 0], v_cf, rtol=1e-3, atol=1e-9 * s[0])
        assert np.all(np.abs(jmu) < 1e-9) and np.all(np.abs(jv) < 1e-9)
    mdl1 = O.Model.build(X, Y, ell, s, noise, 1)
    _, var1, *_ = mdl1.predict(xs)
    assert np.all(var1[:, 0] > 10 * v_cf)  # rank 1 is not exact


def test_love_jacobians_match_central_differences():
    X, Y, ell, s, noise = small_gp_data(N=50, p=2, seed=10)
    mdl = _love_model(X, Y, ell, s, noise, k=20)
    xs = np.random.default_rng(5).uniform(-1.5, 1.5, size=(4, 3))
    mean, var, jmu, jv, _, _ = mdl.predict(xs)
    h = 1e-6
    for c in range(3):
        e = np.zeros(3)
        e[c] = h
        mp, vp, *_ = mdl.predict(xs + e)
        mm, vm, *_ = mdl.predict(xs - e)
        fd_m = (mp - mm) / (2 * h)
        fd_v = (vp - vm) / (2 * h)
        assert np.allclose(jmu[:, :, c], fd_m, rtol=1e-6, atol=1e-9 * np.abs(fd_m).max())
        assert np.allclose(jv[:, :, c], fd_v, rtol=1e-5, atol=1e-9 * np.abs(fd_v).max() + 1e-14)


def test_variance_bounds_nonneg_and_at_most_s():
    X, Y, ell, s, noise = small_gp_data(N=70, p=2, seed=11)
    mdl = _love_model(X, Y, ell, s, noise, k=30)
    xs = np.random.default_rng(6).uniform(-4, 4, size=(200, 3))
    _, var, *_ = mdl.predict(xs)
    assert np.all(var >= 0.0)
    assert np.all(var <= s[None, :] + 1e-12)


# ------------------------------------------------------------------ reward (Eq.8)
def test_reward_worked_values():
    ex = spec_examples()
    assert O.reward([10.0, 0.1], 1.0, [0.1, 0.0], [0.0, 0.0]) == pytest.approx(float(ex["reward_q10_err01"]), abs=5e-7)
    assert O.reward([10.0, 0.1], 1.0, [0.1, 0.0], [0.0, 0.0]) == pytest.approx(math.exp(-0.05), rel=1e-15)
    assert O.reward([10.0, 0.1], 1.0, [0.4, -2.0], [0.4, -2.0]) == 1.0
    # sigma_r halves the exponent scale twice: r(sigma_r=2) = r(sigma_r=1)^(1/4)
    r1 = O.reward([10.0, 0.1], 1.0, [0.3, 0.2], [0.0, 0.0])
    r2 = O.reward([10.0, 0.1], 2.0, [0.3, 0.2], [0.0, 0.0])
    assert r2 == pytest.approx(r1 ** 0.25, rel=1e-14)
