"""GPU parity of the exact-GP variant ("AutoDiff on exact GPs"):
exact_cache_build installs R = L^-1 at rank N, so the hot path's variance is Eq.3 exactly.
Checked against the oracle's exact posterior (Cholesky + triangular solves, orc_exact_predict) and
through a rollout against the oracle run on the same exact cache."""
import numpy as np
import pytest
import torch

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu
U32 = 2.0 ** -24


@pytest.fixture(scope="module")
def bagel():
    from paper_2202_13638_b200 import bagel as b

    assert torch.cuda.is_available()
    b.lib()
    return b


@pytest.mark.parametrize("N", [200, 700])
def test_exact_cache_predict_matches_exact_posterior(bagel, N):
    wl = W.make_workload(plant="boom", N=N, rank=50, hidden=(16,), B=300, T=5)
    ctx = bagel.setup(wl, device=0, build_cache=False)
    ctx.exact_cache_build()
    assert ctx.cache_rank() == N
    rng = np.random.default_rng(N)
    xs = rng.uniform(-1.5, 1.5, (300, wl.d)).astype(np.float32)
    mean, var, _, _ = [t.cpu().numpy() for t in ctx.gp_predict(xs)]
    for m in range(wl.p):
        a_o, L_o = O.exact_fit(wl.X, wl.Y[:, m], wl.ell[m], float(wl.s[m]), float(wl.noise[m]))
        mu_o, v_o = O.exact_predict(wl.X, wl.ell[m], float(wl.s[m]), L_o, a_o, xs)
        # conditioning-aware fp32 bounds (tests/test_gpu_parity.py): sum |k alpha|, 2 sum|z| sum|R k|
        K = O.kernel_matrix(xs, wl.X, wl.ell[m], float(wl.s[m]))
        mb = 1e-4 * np.abs(mu_o) + 32 * U32 * np.abs(K * a_o).sum(1)
        assert np.all(np.abs(mean[:, m] - mu_o) <= mb)
        Li = np.linalg.inv(L_o)
        z = K @ Li.T
        vb = 1e-4 * np.abs(v_o) + 32 * U32 * 2 * (np.abs(z) * (np.abs(K) @ np.abs(Li).T)).sum(1)
        assert np.all(np.abs(var[:, m] - v_o) <= vb)
        assert np.all(var[:, m] <= wl.s[m] * (1 + 1e-5))
    # the cache the GPU built: alpha and L^-1 against the oracle's
    alpha, R = ctx.cache_get(0)
    a_o, L_o = O.exact_fit(wl.X, wl.Y[:, 0], wl.ell[0], float(wl.s[0]), float(wl.noise[0]))
    np.testing.assert_allclose(alpha.cpu().numpy(), a_o, rtol=1e-8, atol=1e-10 * np.abs(a_o).max())
    Li_o = np.linalg.solve(L_o, np.eye(N))
    np.testing.assert_allclose(R.cpu().numpy(), Li_o, rtol=1e-8, atol=1e-10 * np.abs(Li_o).max())
    ctx.close()


def test_exact_cache_rollout_matches_oracle(bagel):
    wl = W.make_workload(plant="boom", N=300, rank=50, hidden=(16, 16), B=64, T=12)
    ctx = bagel.setup(wl, device=0, build_cache=False)
    ctx.exact_cache_build()
    alphas, Rs = [], []
    for m in range(wl.p):
        a, R = ctx.cache_get(m)
        alphas.append(a.cpu().numpy())
        Rs.append(R.cpu().numpy())
    mdl = O.Model(wl.X, wl.ell, wl.s, np.stack(alphas), np.stack(Rs))
    cost, grad = ctx.rollout_cost_and_grad(torch.from_numpy(wl.theta).cuda(), torch.from_numpy(wl.x0).cuda(),
                                           torch.from_numpy(wl.goals).cuda(), wl.T, W.rollout_seed(3))
    ref = O.rollout(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0, wl.goals, wl.T, W.rollout_seed(3))
    assert abs(cost - ref["cost"]) <= 1e-3 * abs(ref["cost"])
    g = grad.double().cpu().numpy()
    assert np.linalg.norm(g - ref["grad"]) <= 1e-3 * np.linalg.norm(ref["grad"])
    ctx.close()


def test_exact_cache_rejects_large_n(bagel):
    from paper_2202_13638_b200.bagel import BagelError, E_ARG

    wl = W.make_workload(plant="boom", N=8200, rank=50, hidden=(16,), B=4, T=2)
    ctx = bagel.setup(wl, device=0, build_cache=False)
    with pytest.raises(BagelError) as ei:
        ctx.exact_cache_build()
    assert ei.value.code == E_ARG
    ctx.close()


@pytest.mark.slow
def test_exact_gp_at_the_paper_baseline_size(bagel):
    """The paper's exact-GP baseline shape (Exp. 1: n = 2200, b = 100, H = 300, [8, 8]; P:149-151,
    P:162 "AutoDiff+ExactGPs"): rank-N cache (nine 256-column z tiles, nine j tiles), predict against
    the oracle's exact posterior, and the full rollout cost and gradient against the oracle run on the
    same exact cache."""
    wl = W.config("E1")
    assert wl.N == 2200
    ctx = bagel.setup(wl, device=0, build_cache=False)
    ctx.exact_cache_build()
    assert ctx.cache_rank() == wl.N
    rng = np.random.default_rng(22)
    xs = np.concatenate([wl.X[rng.integers(0, wl.N, 150)] + rng.normal(0, 0.05, (150, wl.d)),
                         rng.uniform(-1.5, 1.5, (106, wl.d))]).astype(np.float32)
    mean, var, _, _ = [t.cpu().numpy() for t in ctx.gp_predict(xs)]
    alphas, Rs = [], []
    for m in range(wl.p):
        a_o, L_o = O.exact_fit(wl.X, wl.Y[:, m], wl.ell[m], float(wl.s[m]), float(wl.noise[m]))
        mu_o, v_o = O.exact_predict(wl.X, wl.ell[m], float(wl.s[m]), L_o, a_o, xs)
        K = O.kernel_matrix(xs, wl.X, wl.ell[m], float(wl.s[m]))
        mb = 1e-4 * np.abs(mu_o) + 16 * U32 * np.abs(K * a_o).sum(1)
        assert np.all(np.abs(mean[:, m] - mu_o) <= mb)
        Li = np.linalg.solve(L_o, np.eye(wl.N))
        z = K @ Li.T
        vb = 1e-4 * np.abs(v_o) + 16 * U32 * 2 * (np.abs(z) * (np.abs(K) @ np.abs(Li).T)).sum(1)
        assert np.all(np.abs(var[:, m] - v_o) <= vb)
        a, R = ctx.cache_get(m)
        np.testing.assert_allclose(R.cpu().numpy(), Li, rtol=1e-7, atol=1e-9 * np.abs(Li).max())
        alphas.append(a.cpu().numpy())
        Rs.append(R.cpu().numpy())
    mdl = O.Model(wl.X, wl.ell, wl.s, np.stack(alphas), np.stack(Rs))
    seed = W.rollout_seed(7)
    th = torch.from_numpy(wl.theta).cuda()
    # the full b = 100 batch on the GPU: sampled per-trajectory returns vs the oracle one row at a time
    # (a row's arithmetic is batch-invariant, so the subset below replays these rows exactly)
    ret = ctx.rollout_trace(th, wl.x0, wl.goals, wl.T, seed)["ret"].double().cpu().numpy()
    for b in (0, 63, 99):
        r = O.rollout(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0[b:b + 1], wl.goals[b:b + 1], wl.T, seed,
                      traj_offset=b, B_global=1)
        assert abs(ret[b] - r["ret"][0]) <= 1e-3 * abs(r["ret"][0])
    # cost and gradient of a 16-trajectory block (ids 40..55) of the same iteration
    off, n = 40, 16
    cost, grad = ctx.rollout_cost_and_grad(th, torch.from_numpy(wl.x0[off:off + n]).cuda(),
                                           torch.from_numpy(wl.goals[off:off + n]).cuda(), wl.T, seed,
                                           traj_offset=off, B_global=wl.B)
    ref = O.rollout(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0[off:off + n], wl.goals[off:off + n],
                    wl.T, seed, traj_offset=off, B_global=wl.B)
    rel_g = np.linalg.norm(grad.double().cpu().numpy() - ref["grad"]) / np.linalg.norm(ref["grad"])
    print(f"exact GP n=2200: cost rel {abs(cost - ref['cost']) / abs(ref['cost']):.2e}, grad rel L2 {rel_g:.2e}")
    assert abs(cost - ref["cost"]) <= 1e-3 * abs(ref["cost"])
    assert rel_g <= 1e-3
    ctx.close()


def test_exact_cache_with_absolute_targets(bagel):
    """The two variants together: exact variance (R = L^-1) and absolute targets (x' = mu + sigma eps)."""
    wl = W.make_workload(plant="boom", N=400, rank=50, hidden=(16, 16), B=48, T=8, target="abs")
    ctx = bagel.setup(wl, device=0, build_cache=False)
    ctx.gp_target_mode(True)
    ctx.exact_cache_build()
    alphas, Rs = zip(*[(a.cpu().numpy(), r.cpu().numpy()) for a, r in (ctx.cache_get(m) for m in range(wl.p))])
    mdl = O.Model(wl.X, wl.ell, wl.s, np.stack(alphas), np.stack(Rs), abs_target=True)
    cost, grad = ctx.rollout_cost_and_grad(torch.from_numpy(wl.theta).cuda(), torch.from_numpy(wl.x0).cuda(),
                                           torch.from_numpy(wl.goals).cuda(), wl.T, W.rollout_seed(4))
    ref = O.rollout(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0, wl.goals, wl.T, W.rollout_seed(4))
    assert abs(cost - ref["cost"]) <= 1e-3 * abs(ref["cost"])
    g = grad.double().cpu().numpy()
    assert np.linalg.norm(g - ref["grad"]) <= 1e-3 * np.linalg.norm(ref["grad"])
    ctx.close()
