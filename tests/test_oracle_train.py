"""Pins of the oracle's Algorithm-1 loop pieces (no GPU): the S_0 / goal sampler (P:101, P:144,
P:180) and Adam, against closed forms, special cases and statistics."""
import math

import numpy as np
import pytest

import oracle as O
import workloads as W


# ---------------------------------------------------------------- sampler
def test_sampler_counter_convention_and_bounds():
    """out[b][m] = lo + (hi - lo) u with u from ctr (traj_offset + b, 0, m >> 2, 2 + which)."""
    lo, hi = np.array([-1.5, -0.25, 0.0]), np.array([0.5, 2.0, 0.0])
    seed, off = 0x5EED0007, 11
    for which in (0, 1):
        s = O.sample_states(seed, off, 5, lo, hi, which)
        assert s.shape == (5, 3)
        assert np.all(s >= lo) and np.all(s <= hi)
        assert np.all(s[:, 2] == 0.0)  # lo == hi: the bound itself
        o = O.philox4x32_10([off + 3, 0, 0, 2 + which], [seed & 0xFFFFFFFF, seed >> 32])
        u = ((int(o[1]) >> 9) + 0.5) * 2.0 ** -23
        assert s[3, 1] == -0.25 + 2.25 * u
    # shards: rows of a traj_offset block equal the same rows of the full batch
    full = O.sample_states(seed, 0, 20, lo, hi, 0)
    assert np.array_equal(O.sample_states(seed, 7, 6, lo, hi, 0), full[7:13])


def test_sampler_statistics_and_stream_independence():
    lo, hi = np.array([-1.0, 2.0]), np.array([3.0, 2.5])
    B = 200_000
    a = O.sample_states(123, 0, B, lo, hi, 0)
    g = O.sample_states(123, 0, B, lo, hi, 1)
    mean, var = (lo + hi) / 2, (hi - lo) ** 2 / 12
    se_mean = np.sqrt(var / B)
    assert np.all(np.abs(a.mean(0) - mean) < 4 * se_mean)
    assert np.all(np.abs(a.var(0) / var - 1) < 0.02)
    # S_0 and G streams are different and uncorrelated
    r = np.corrcoef(a[:, 0], g[:, 0])[0, 1]
    assert abs(r) < 4 / math.sqrt(B)
    assert not np.array_equal(a, g)


# ---------------------------------------------------------------- Adam
def _adam(theta, g, steps, lr=1e-2):
    th = np.array(theta, dtype=np.float64)
    m1, m2 = np.zeros_like(th), np.zeros_like(th)
    for t in range(1, steps + 1):
        gg = np.array(g(th) if callable(g) else g, dtype=np.float64)
        assert not O.adam_step(th, gg, m1, m2, t, lr)
    return th


def test_adam_first_step_is_lr_sign():
    """S:402 example: scalar g = 1, lr = 0.01 -> delta = -0.01 / (1 + 1e-8) (m1hat = g, m2hat = g^2)."""
    th = _adam([0.0], [1.0], 1)
    assert th[0] == pytest.approx(-0.01 / (1.0 + 1e-8), rel=1e-15)
    th = _adam([2.0, -1.0], [-3e-3, 40.0], 1, lr=0.5)
    assert th == pytest.approx([2.0 + 0.5 * 3e-3 / (3e-3 + 1e-8), -1.0 - 0.5 * 40.0 / (40.0 + 1e-8)], rel=1e-14)


def test_adam_constant_gradient_closed_form():
    """With a constant g the bias corrections make m1hat = g and m2hat = g^2 at every t, so
    theta_t = theta_0 - t lr g / (|g| + eps)."""
    g = np.array([0.7, -2e-4, 5.0])
    th = _adam([1.0, 1.0, 1.0], g, 37, lr=3e-3)
    assert th == pytest.approx(1.0 - 37 * 3e-3 * g / (np.abs(g) + 1e-8), rel=1e-12)


def test_adam_zero_gradient_and_nonfinite_skip():
    th = _adam([0.3, -0.4], [0.0, 0.0], 5)
    assert np.array_equal(th, [0.3, -0.4])
    th = np.array([1.0, 2.0])
    m1, m2 = np.array([0.1, 0.2]), np.array([0.3, 0.4])
    assert O.adam_step(th, np.array([np.nan, 1.0]), m1, m2, 3)
    assert O.adam_step(th, np.array([1.0, np.inf]), m1, m2, 3)
    assert np.array_equal(th, [1.0, 2.0]) and np.array_equal(m1, [0.1, 0.2]) and np.array_equal(m2, [0.3, 0.4])


def test_adam_converges_on_quadratic():
    """a 10-d quadratic converges to ||theta|| < 1e-3 within 2000 steps at lr = 0.01."""
    rng = np.random.default_rng(0)
    A = np.diag(np.linspace(0.5, 5.0, 10))
    th = _adam(rng.uniform(-1, 1, 10), lambda x: A @ x, 2000, lr=0.01)
    assert np.linalg.norm(th) < 1e-3


# ---------------------------------------------------------------- loop
def test_train_loop_improves_the_return_on_c1():
    """Algorithm 1 with the Exp. 1 setup (fixed S_0 and goal; goal 0.6 normalised units above
    S_0 so the reward is informative): 60 Adam steps lower L = -mean return by more than a quarter of
    its range [-(T+1), 0]; zero iterations leave theta unchanged.  (lr 5e-2: at the paper's 1e-2,
    P:151, this 20-step toy needs a few hundred iterations.)"""
    wl = W.config("C1")
    wl.goals = (wl.x0 + 0.6).astype(np.float32)
    mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank)
    lo, hi = wl.X[:, :wl.p].min(0), wl.X[:, :wl.p].max(0)
    th0, c0 = O.train(mdl, wl.sizes, "xgd", wl.theta, wl.Q, wl.sigma_r, wl.T, 0, wl.B, lo, hi, 0x5EED0000,
                      x0=wl.x0, goals=wl.goals)
    assert c0 == [] and np.array_equal(th0, wl.theta.astype(np.float64))
    th, costs = O.train(mdl, wl.sizes, "xgd", wl.theta, wl.Q, wl.sigma_r, wl.T, 60, wl.B, lo, hi, 0x5EED0000,
                        lr=5e-2, x0=wl.x0, goals=wl.goals)
    assert np.mean(costs[-10:]) < costs[0] - 0.25 * (wl.T + 1), costs
    assert np.all(np.isfinite(th))
