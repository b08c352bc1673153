"""GPU parity of Algorithm 1's loop pieces through the C ABI against the
float64 oracle: the S_0 / goal sampler, Adam, and whole training runs.

Tolerances: sampler |d| <= 2^-22 (hi - lo) + 2^-23 max(|lo|, |hi|) (fp32 rounding of one
multiply-add); Adam relative 1e-5 per parameter after several steps (fp32 moments vs fp64);
training runs: per-iteration cost 1e-3 relative, final theta 1e-3 relative L2."""
import numpy as np
import pytest
import torch

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bagel():
    from paper_2202_13638_b200 import bagel as b

    assert torch.cuda.is_available()
    b.lib()
    return b


def test_sampler_matches_oracle(bagel):
    ctx = bagel.Context(0)
    lo = np.array([-1.5, -3.1, 0.2, 0.0], dtype=np.float32)
    hi = np.array([2.2, 2.0, 0.2, 1e-3], dtype=np.float32)
    for which in (0, 1):
        for (off, B) in ((0, 1), (5, 1000), (123_457, 333)):
            g = ctx.sample_states(0x5EED0003, off, B, lo, hi, which).cpu().numpy()
            o = O.sample_states(0x5EED0003, off, B, lo, hi, which)
            tol = 2.0 ** -22 * (hi - lo) + 2.0 ** -23 * np.maximum(np.abs(lo), np.abs(hi))
            assert np.all(np.abs(g - o) <= tol), (which, off, B)
            assert np.all(g >= lo) and np.all(g <= hi)
    ctx.close()


def test_adam_matches_oracle_and_skips_nonfinite(bagel):
    ctx = bagel.Context(0)
    rng = np.random.default_rng(0)
    n = 133_121 + 7  # the C3 policy plus a ragged tail
    th64 = rng.normal(0, 0.3, n).astype(np.float32).astype(np.float64)
    m1_64, m2_64 = np.zeros(n), np.zeros(n)
    th = torch.from_numpy(th64.astype(np.float32)).cuda()
    m1, m2 = torch.zeros_like(th), torch.zeros_like(th)
    for t in range(1, 6):
        g32 = (rng.normal(0, 1e-2, n) * rng.choice([1e-4, 1.0, 30.0], n)).astype(np.float32)
        g32[:3] = 0.0
        assert not ctx.adam_step(th, torch.from_numpy(g32).cuda(), m1, m2, t, lr=1e-2, report_skip=True)
        assert not O.adam_step(th64, g32.astype(np.float64), m1_64, m2_64, t, 1e-2)
    got = th.cpu().numpy().astype(np.float64)
    # fp32 moments vs fp64: the 5 updates (each <= lr in size) agree to ~1e-5 of lr, theta to its rounding
    assert np.all(np.abs(got - th64) <= 1e-5 * np.abs(th64) + 1e-5 * 5 * 1e-2)
    assert np.array_equal(got[:3], th64[:3])  # g = 0 at every step: untouched on both sides
    before = th.clone()
    bad = torch.from_numpy(np.where(np.arange(n) == n - 1, np.nan, 1.0).astype(np.float32)).cuda()
    m1b, m2b = m1.clone(), m2.clone()
    assert ctx.adam_step(th, bad, m1, m2, 6, lr=1e-2, report_skip=True)
    assert torch.equal(th, before) and torch.equal(m1, m1b) and torch.equal(m2, m2b)
    ctx.close()


def _c1_goal_problem():
    wl = W.config("C1")
    wl.goals = (wl.x0 + 0.6).astype(np.float32)
    return wl


def test_training_run_matches_oracle_fixed_goal(bagel):
    """Exp. 1 setup (fixed S_0 and goal) on C1: 10 iterations of Algorithm 1 at lr 5e-2."""
    from paper_2202_13638_b200.train import train_policy

    wl = _c1_goal_problem()
    mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank)
    lo, hi = wl.X[:, :wl.p].min(0), wl.X[:, :wl.p].max(0)
    ctx = bagel.setup(wl, device=0)
    for m in range(mdl.p):
        ctx.cache_set(m, mdl.alpha[m], mdl.R[m])
    iters = 10
    th, log = train_policy(ctx, wl.theta, wl.T, iters, wl.B, x0=wl.x0, goals=wl.goals, lr=5e-2)
    th_o, costs_o = O.train(mdl, wl.sizes, "xgd", wl.theta, wl.Q, wl.sigma_r, wl.T, iters, wl.B, lo, hi,
                            0x5EED0000, lr=5e-2, x0=wl.x0, goals=wl.goals)
    np.testing.assert_allclose(log.cost, costs_o, rtol=1e-3)
    t = th.cpu().numpy().astype(np.float64)
    assert np.linalg.norm(t - th_o) <= 1e-3 * np.linalg.norm(th_o)
    assert log.skipped == 0
    # bitwise repeatable
    th2, log2 = train_policy(ctx, wl.theta, wl.T, iters, wl.B, x0=wl.x0, goals=wl.goals, lr=5e-2)
    assert torch.equal(th, th2) and log.cost == log2.cost
    ctx.close()


def test_training_run_matches_oracle_sampled_goals(bagel):
    """Goal-conditioned setup (S_0 and G uniform within the data bounds each iteration, P:144,
    P:180) on a small boom problem: 6 iterations at the paper's lr 1e-2."""
    from paper_2202_13638_b200.train import train_policy

    wl = W.make_workload(plant="boom", N=600, rank=64, hidden=(8, 8), B=48, T=15)
    mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank)
    lo, hi = wl.X[:, :wl.p].min(0), wl.X[:, :wl.p].max(0)
    ctx = bagel.setup(wl, device=0)
    for m in range(mdl.p):
        ctx.cache_set(m, mdl.alpha[m], mdl.R[m])
    th, log = train_policy(ctx, wl.theta, wl.T, 6, wl.B, lo, hi, lr=1e-2, seed0=0x5EED1000)
    th_o, costs_o = O.train(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.T, 6, wl.B, lo, hi, 0x5EED1000,
                            lr=1e-2)
    np.testing.assert_allclose(log.cost, costs_o, rtol=1e-3)
    t = th.cpu().numpy().astype(np.float64)
    assert np.linalg.norm(t - th_o) <= 1e-3 * np.linalg.norm(th_o)
    ctx.close()


def test_training_run_wide_policy_matches_oracle(bagel):
    """Algorithm 1 with a wide policy (the cluster MLP kernels, the tensor-core theta gradient and
    the weight repacking every iteration): 4 iterations at lr 1e-2 with sampled goals."""
    from paper_2202_13638_b200.train import train_policy

    wl = W.make_workload(plant="boom", N=500, rank=64, hidden=(256, 256), B=96, T=6)
    mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank)
    lo, hi = wl.X[:, :wl.p].min(0), wl.X[:, :wl.p].max(0)
    ctx = bagel.setup(wl, device=0)
    for m in range(mdl.p):
        ctx.cache_set(m, mdl.alpha[m], mdl.R[m])
    th, log = train_policy(ctx, wl.theta, wl.T, 4, wl.B, lo, hi, lr=1e-2, seed0=0x5EED2000)
    th_o, costs_o = O.train(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.T, 4, wl.B, lo, hi, 0x5EED2000,
                            lr=1e-2)
    np.testing.assert_allclose(log.cost, costs_o, rtol=1e-3)
    # Adam normalises per coordinate (a step is lr m / sqrt(v)), so a coordinate's step error is lr
    # times the RELATIVE error of its own gradient: tiny on the coordinates that matter, up to 2 lr
    # where a gradient sits below the ~1e-4 (of the norm) gradient error (scripts/diag_train.py: the
    # per-iteration costs agree to 7e-5; 2 of 67,329 first-iteration gradients differ in sign, both
    # at 1.9e-7 of the largest; theta after 4 iterations 2.0e-3 relative L2, 3.7e-4 after 1).
    # Asserted: the costs above, theta within 5e-3 relative L2, no coordinate beyond 2 lr per step.
    t = th.cpu().numpy().astype(np.float64)
    assert np.linalg.norm(t - th_o) <= 5e-3 * np.linalg.norm(th_o)
    assert np.abs(t - th_o).max() <= 2 * 1e-2 * 4
    ctx.close()


def test_exp1_shape_reaches_the_spec_return_bar(bagel):
    """SPEC S:416's end-to-end bar on the Exp. 1 shape (workload E1: n = 2200, b = 100, H = 300,
    policy [8, 8], fixed start and goal, Adam lr 1e-2): the mean return per step
    exceeds 0.85 within 100 iterations.  (A property of the whole loop; the oracle is too slow for
    this shape, its agreement with the GPU loop is checked above on small problems.)"""
    from paper_2202_13638_b200.train import train_policy

    wl = W.config("E1")
    ctx = bagel.setup(wl, device=0)
    th, log = train_policy(ctx, wl.theta, wl.T, 100, wl.B, x0=wl.x0, goals=wl.goals, lr=1e-2)
    per_step = -np.array(log.cost) / (wl.T + 1)
    assert per_step[:5].mean() < 0.2          # starts far from the goal
    assert per_step[-5:].mean() > 0.85, per_step[-10:]
    assert log.skipped == 0 and log.seconds[-1] < 30.0  # the paper's "under 30 seconds", as a sanity bound
    ctx.close()


def test_goal_conditioned_training_improves_the_return(bagel):
    """Exp. 2's mode: S_0 and G drawn uniformly within the data bounds at every
    iteration; a goal-conditioned policy (input [x, g]) on the C2 boom GP improves its mean return
    per step over 80 Adam iterations (fresh samples each iteration, so the comparison is between
    10-iteration averages)."""
    from paper_2202_13638_b200.train import train_policy

    wl = W.config("C2", T=60)
    lo, hi = wl.X[:, :wl.p].min(0), wl.X[:, :wl.p].max(0)
    ctx = bagel.setup(wl, device=0)
    th, log = train_policy(ctx, wl.theta, wl.T, 80, wl.B, lo, hi, lr=1e-2, seed0=0x5EED3000)
    per_step = -np.array(log.cost) / (wl.T + 1)
    assert per_step[-10:].mean() > per_step[:10].mean() + 0.05, (per_step[:10].mean(), per_step[-10:].mean())
    ctx.close()
