"""GPU parity of the log marginal likelihood and its gradient (Eq.5-6; SURVEY.md §8(f)
NEXT-1) through the C ABI against the float64 oracle, plus the hyperparameter fit.

Tolerances (both sides float64, different summation orders): log p relative 1e-10; gradient
|d g| <= 1e-7 ||g||_inf + 1e-9 |log p| (the trace term cancels against the quadratic term)."""
import numpy as np
import pytest
import torch

import oracle as O
import workloads as W
from conftest import small_gp_data

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bagel():
    from paper_2202_13638_b200 import bagel as b

    assert torch.cuda.is_available()
    b.lib()
    return b


def _ctx(bagel, X, Y, ell, s, noise):
    ctx = bagel.Context(0)
    ctx.gp_load(X.astype(np.float32), Y.astype(np.float32), ell.astype(np.float32), s.astype(np.float32),
                noise.astype(np.float32))
    return ctx


@pytest.mark.parametrize("N", [1, 2, 63, 64, 65, 700])
def test_mll_and_gradient_match_oracle(bagel, N):
    X, Y, ell, s, noise = small_gp_data(N=N, d=3, p=2, seed=N)
    ctx = _ctx(bagel, X, Y, ell, s, noise)
    Xf, Yf = X.astype(np.float32).astype(np.float64), Y.astype(np.float32).astype(np.float64)
    rng = np.random.default_rng(N)
    for m in range(2):
        for h in (ctx.loaded_log_hyp(m), ctx.loaded_log_hyp(m) + rng.normal(0, 0.3, 5)):
            v, g = ctx.log_marginal_likelihood(m, h)
            vo, go = O.log_marginal_likelihood(Xf, Yf[:, m], h)
            assert v == pytest.approx(vo, rel=1e-10, abs=1e-10)
            assert np.all(np.abs(g - go) <= 1e-7 * np.abs(go).max() + 1e-9 * abs(vo)), (g, go)
    v0, g0 = ctx.log_marginal_likelihood(0, None, want_grad=False)
    assert g0 is None and v0 == pytest.approx(ctx.log_marginal_likelihood(0)[0], rel=0, abs=0)
    ctx.close()


def test_c2_size_gradient_matches_central_differences(bagel):
    """N = 5000 (the C2 dataset): the oracle is too slow here, so the GPU gradient is checked against
    central differences of the GPU's own log p (a property that holds at any size)."""
    wl = W.config("C2")
    ctx = bagel.Context(0)
    ctx.gp_load(wl.X, wl.Y, wl.ell, wl.s, wl.noise)
    h = ctx.loaded_log_hyp(1)
    _, g = ctx.log_marginal_likelihood(1, h)
    for j in range(len(h)):
        e = np.zeros_like(h)
        e[j] = 1e-4
        fp, _ = ctx.log_marginal_likelihood(1, h + e, want_grad=False)
        fm, _ = ctx.log_marginal_likelihood(1, h - e, want_grad=False)
        fd = (fp - fm) / 2e-4
        assert abs(g[j] - fd) <= 1e-4 * np.abs(g).max(), (j, g[j], fd)
    ctx.close()


def test_non_spd_is_reported(bagel):
    from paper_2202_13638_b200.bagel import BagelError, E_NUMERIC

    X = np.zeros((5, 2), dtype=np.float32)  # five identical inputs
    Y = np.ones((5, 1), dtype=np.float32)
    ctx = _ctx(bagel, X, Y, np.ones((1, 2)), np.ones(1), np.full(1, 1e-8))
    with pytest.raises(BagelError) as ei:
        # s = e^30 swamps sn2 = 2e-8 in float64: the second pivot is exactly 0
        ctx.log_marginal_likelihood(0, np.array([0.0, 0.0, 30.0, np.log(2e-8)]))
    assert ei.value.code == E_NUMERIC and "pivot" in str(ei.value)
    ctx.close()


def test_fit_recovers_prior_hyperparameters(bagel):
    """targets drawn from a GP prior with known phi (n = 200, d = 2): the fit raises log p
    monotonically (up to Adam's noise) and recovers the log-lengthscales within 0.3 nats."""
    from paper_2202_13638_b200.fit import fit_hyperparameters

    rng = np.random.default_rng(7)
    N = 200
    X = rng.uniform(-2, 2, (N, 2))
    ell_t, s_t, sn_t = np.array([0.6, 1.4]), 0.8, 0.01
    D = ((X[:, None, :] - X[None, :, :]) / ell_t) ** 2
    K = s_t * np.exp(-0.5 * D.sum(-1)) + sn_t * np.eye(N)
    y = np.linalg.cholesky(K) @ rng.standard_normal(N)
    ctx = _ctx(bagel, X, y[:, None], np.ones((1, 2)), np.ones(1), np.full(1, 0.1))
    phi, log = fit_hyperparameters(ctx, 0, iters=500, lr=0.05)
    assert log.mll[-1] > log.mll[0] + 10
    assert np.all(np.abs(phi[:2] - np.log(ell_t)) < 0.3), phi
    # the fitted phi is (close to) a stationary point of the oracle's objective
    vo, go = O.log_marginal_likelihood(X.astype(np.float32).astype(np.float64),
                                       y.astype(np.float32).astype(np.float64), phi)
    assert np.abs(go).max() < 0.5
    ctx.close()


def test_mll_c4_dims_and_fit_then_rebuild(bagel):
    """d = 5 inputs (the C4 hydraulic plant's shape) at N = 900 against the oracle, then the fitted
    hyperparameters drive a new gp_load + LOVE cache (the Alg.1 order: learn the GP, then roll out)."""
    from paper_2202_13638_b200.fit import fit_hyperparameters

    wl = W.config("C4", N=900, B=8, T=3, rank=64)
    ctx = bagel.setup(wl, device=0)
    Xf, Yf = wl.X.astype(np.float64), wl.Y.astype(np.float64)
    for m in (0, 3):
        h = ctx.loaded_log_hyp(m)
        v, g = ctx.log_marginal_likelihood(m, h)
        vo, go = O.log_marginal_likelihood(Xf, Yf[:, m], h)
        assert v == pytest.approx(vo, rel=1e-10)
        assert np.all(np.abs(g - go) <= 1e-7 * np.abs(go).max() + 1e-9 * abs(vo))
    phis = [fit_hyperparameters(ctx, m, iters=30, lr=0.05)[0] for m in range(wl.p)]
    ell = np.exp(np.stack([ph[:wl.d] for ph in phis])).astype(np.float32)
    s = np.exp([ph[wl.d] for ph in phis]).astype(np.float32)
    sn = np.exp([ph[wl.d + 1] for ph in phis]).astype(np.float32)
    for m in range(wl.p):  # the fit improved every output's likelihood
        assert ctx.log_marginal_likelihood(m, phis[m], want_grad=False)[0] > ctx.log_marginal_likelihood(m)[0]
    ctx.gp_load(wl.X, wl.Y, ell, s, sn)
    ctx.love_cache_build(64)
    ctx.policy_configure(wl.sizes)
    ctx.reward_configure(wl.Q, wl.sigma_r)
    cost, grad = ctx.rollout_cost_and_grad(wl.theta, wl.x0, wl.goals, wl.T, W.rollout_seed(0))
    mdl = O.Model.build(wl.X, wl.Y, ell, s, sn, 64)
    ref = O.rollout(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0, wl.goals, wl.T, W.rollout_seed(0))
    assert abs(cost - ref["cost"]) <= 1e-3 * abs(ref["cost"])
    g = grad.double().cpu().numpy()
    assert np.linalg.norm(g - ref["grad"]) <= 1e-3 * np.linalg.norm(ref["grad"])
    ctx.close()
