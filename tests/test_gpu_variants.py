"""GPU parity of the absolute-target variant ("y = x_{k+1}"): the
GPs model the next state itself, x' = mu + sigma eps, and the reverse pass drops the identity path.
Same tolerances as tests/test_gpu_parity.py (cost 1e-3 relative, gradient 1e-3 relative L2)."""
import os

import numpy as np
import pytest
import torch

import oracle as O
import workloads as W
from conftest import GOLDEN
from test_gpu_parity import _assert_cost_grad, _inject, _rollout_gpu, _rollout_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bagel():
    from paper_2202_13638_b200 import bagel as b

    assert torch.cuda.is_available()
    b.lib()
    return b


def _abs_problem(bagel, wl):
    mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank, abs_target=True)
    ctx = bagel.setup(wl, device=0, build_cache=False)
    ctx.gp_target_mode(True)
    _inject(ctx, mdl)
    return ctx, mdl


@pytest.mark.parametrize("gp_kernel", [1, 0])
def test_absolute_targets_rollout(bagel, gp_kernel):
    wl = W.make_workload(plant="boom", N=700, rank=100, hidden=(32, 32), B=150, T=10, target="abs")
    goals = (wl.x0 + np.array([0.5, -0.3], dtype=np.float32)).astype(np.float32)
    ctx, mdl = _abs_problem(bagel, wl)
    ctx.set_gp_kernel(gp_kernel)
    seed = W.rollout_seed(7)
    cost, grad = _rollout_gpu(ctx, wl, goals, seed)
    _assert_cost_grad(cost, grad, _rollout_oracle(mdl, wl, goals, seed), f"abs targets, kernel {gp_kernel}")
    tr = ctx.rollout_trace(wl.theta, wl.x0, goals, wl.T, seed)
    ref = O.rollout(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0, goals, wl.T, seed, trace=True)
    np.testing.assert_allclose(tr["x"].cpu().numpy(), ref["x"], atol=2e-3)
    # switching back to Delta targets changes the dynamics (and matches the Delta oracle)
    ctx.gp_target_mode(False)
    cost_d, _ = _rollout_gpu(ctx, wl, goals, seed)
    mdl_d = O.Model(mdl.X, mdl.ell, mdl.s, mdl.alpha, mdl.R, abs_target=False)
    assert abs(cost_d - _rollout_oracle(mdl_d, wl, goals, seed)["cost"]) <= 1e-3 * abs(cost_d)
    ctx.close()


@pytest.mark.parametrize("T", [20, 40, 100])
def test_absolute_targets_long_horizon(bagel, T):
    """Absolute targets on C2's data and policy (full N and rank, a 64-trajectory block) up to T = 100
    against the float64 oracle (tests/golden/abs_targets.npz, written by scripts/make_golden_abs.py):
    gradient within 1e-3 relative L2.  The oracle's own fp32 envelope there is 4e-5 / 1.6e-4 / 2.2e-4
    at T = 20 / 40 / 100.  This variant runs on the round-to-nearest CUDA-core GP step
    (gp_target_mode, R38): the tensor-core path's truncating accumulation cannot resolve
    v = s - ||z||^2 when v / s ~ 1e-6 (measured 7.5e-3 at T = 40)."""
    wl = W.config("C2", target="abs", B=64, T=100)
    ctx, mdl = _abs_problem(bagel, wl)
    assert ctx.gp_kernel() == 0
    G = np.load(os.path.join(GOLDEN, "abs_targets.npz"))
    cost, grad = _rollout_gpu(ctx, wl, wl.goals, W.rollout_seed(8), T=T)
    ref = {"cost": float(G[f"cost_T{T}"]), "grad": G[f"grad_T{T}"]}
    print(f"T={T}: oracle fp32 envelope {np.max(G[f'floors_T{T}']):.2e}")
    _assert_cost_grad(cost, grad, ref, f"abs targets T={T}")
    ctx.close()


def test_absolute_targets_wide_policy_subset(bagel):
    """C3's 133k-parameter policy with absolute targets (full N and rank, short horizon)."""
    wl = W.config("C3", target="abs", B=48, T=8)
    ctx, mdl = _abs_problem(bagel, wl)
    seed = W.rollout_seed(8)
    cost, grad = _rollout_gpu(ctx, wl, wl.goals, seed)
    _assert_cost_grad(cost, grad, _rollout_oracle(mdl, wl, wl.goals, seed), "C3 abs targets")
    ctx.close()
