"""Rollout / gradient pins for the oracle (no GPU): closed forms, special
cases, invariants and central finite differences."""
import math

import numpy as np
import pytest

import oracle as O
import workloads as W
from conftest import small_gp_data, spec_examples


def _boom_problem(N, k, hidden, B, T, seed=0):
    wl = W.make_workload(plant="boom", N=N, rank=k, hidden=hidden, B=B, T=T, data_seed=seed)
    mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank)
    return wl, mdl


def _run(wl, mdl, theta=None, **kw):
    kw.setdefault("T", wl.T)
    kw.setdefault("seed", W.rollout_seed(0))
    return O.rollout(mdl, wl.sizes, "xg" if wl.sizes[0] == 2 * wl.p else "xgd",
                     wl.theta if theta is None else theta, wl.Q, wl.sigma_r, kw.pop("x0", wl.x0),
                     kw.pop("goals", wl.goals), **kw)


def test_param_count_formula():
    # SPEC.md S:318 prints 129 for [8,8] with in = 4, q = 1, but its own sum
    # (5*8 + 8 + 9*8 + 8 + 9*1) is garbled; sum_l (in_l + 1) out_l = 121 (R28).
    assert W.n_params((4, 8, 8, 1)) == 4 * 8 + 8 + 8 * 8 + 8 + 8 * 1 + 1 == 121
    assert [W.n_params(W.config(c).sizes) for c in ("C1", "C2", "C4")] == [81, 4545, 4801]


def test_scalar_rollout_closed_form():
    """N=1, p=q=1, zero policy (u = tanh(0) = 0):
    x_{t+1} = x_t + k(x_t) y1/(s+sn2) + sqrt(s - k(x_t)^2/(s+sn2)) eps_t."""
    X = np.array([[0.3, -0.2]])
    y = np.array([[0.05]])
    ell = np.array([[0.8, 0.6]])
    s, sn2 = 0.04, 0.004
    mdl = O.Model.build(X, y, ell, [s], [sn2], 1)
    sizes = (2, 3, 1)
    theta = np.zeros(W.n_params(sizes))
    x0, g = np.array([[-0.5]]), np.array([[0.4]])
    Q, sr = np.array([10.0]), 1.0
    T, seed, b = 12, 0x5EED0042, 7
    out = O.rollout(mdl, sizes, "xg", theta, Q, sr, x0, g, T, seed, traj_offset=b, B_global=1,
                    trace=True)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    x = -0.5
    G = math.exp(-0.5 * 10.0 * (x - 0.4) ** 2)
    for t in range(T):
        o = O.philox4x32_10([b, t, 0, 0], key)
        u0, u1 = [((int(v) >> 9) + 0.5) * 2.0 ** -23 for v in o[:2]]
        eps = math.sqrt(-2.0 * math.log(u0)) * math.cos(2.0 * math.pi * u1)
        k = s * math.exp(-0.5 * (((x - 0.3) / 0.8) ** 2 + ((0.0 + 0.2) / 0.6) ** 2))
        mu = k * 0.05 / (s + sn2)
        v = s - k * k / (s + sn2)
        assert out["mu"][t, 0, 0] == pytest.approx(mu, rel=1e-12)
        assert out["var"][t, 0, 0] == pytest.approx(v, rel=1e-10)
        x = x + mu + math.sqrt(v) * eps
        assert out["x"][t + 1, 0, 0] == pytest.approx(x, rel=1e-11, abs=1e-14)
        G += math.exp(-0.5 * 10.0 * (x - 0.4) ** 2)
    assert out["cost"] == pytest.approx(-G, rel=1e-11)


@pytest.fixture(scope="module")
def boom_small():
    return _boom_problem(N=120, k=40, hidden=(8, 8), B=6, T=12)


def test_horizon_zero(boom_small):
    wl, mdl = boom_small
    out = _run(wl, mdl, T=0)
    r = [O.reward(wl.Q, 1.0, wl.x0[b], wl.goals[b]) for b in range(wl.B)]
    assert out["cost"] == pytest.approx(-np.mean(r), rel=1e-14)
    assert np.all(out["grad"] == 0.0)


def test_zero_noise_is_mean_propagation(boom_small):
    wl, mdl = boom_small
    theta = np.zeros(W.n_params(wl.sizes))  # u = 0 so x* = [x, 0]
    out = _run(wl, mdl, theta=theta, eps_mode=1, trace=True)
    for t in range(wl.T):
        xs = np.concatenate([out["x"][t], np.zeros((wl.B, wl.q))], axis=1)
        mean, var, *_ = mdl.predict(xs)
        assert np.allclose(out["mu"][t], mean, rtol=1e-13, atol=1e-16)
        assert np.allclose(out["x"][t + 1], out["x"][t] + mean, rtol=1e-13, atol=1e-15)


def test_batch_row_equals_single_trajectory_run(boom_small):
    wl, mdl = boom_small
    full = _run(wl, mdl)
    for b in range(wl.B):
        one = _run(wl, mdl, x0=wl.x0[b:b + 1], goals=wl.goals[b:b + 1], traj_offset=b, B_global=1)
        assert one["ret"][0] == full["ret"][b]


def test_returns_bounded(boom_small):
    wl, mdl = boom_small
    out = _run(wl, mdl)
    assert np.all(out["ret"] > 0.0) and np.all(out["ret"] <= wl.T + 1)
    assert -(wl.T + 1) <= out["cost"] < 0.0


def test_shards_sum_to_full_batch(boom_small):
    wl, mdl = boom_small
    full = _run(wl, mdl)
    cost, grad = 0.0, np.zeros_like(full["grad"])
    for off in (0, 2, 4):
        sh = _run(wl, mdl, x0=wl.x0[off:off + 2], goals=wl.goals[off:off + 2], traj_offset=off,
                  B_global=wl.B)
        cost += sh["cost"]
        grad += sh["grad"]
    assert cost == pytest.approx(full["cost"], rel=1e-13)
    assert np.allclose(grad, full["grad"], rtol=1e-12, atol=1e-15 * np.abs(full["grad"]).max())


def test_gradient_central_fd_spec_instance():
    """n = 50, b = 4, H = 10, [4] hidden -> relative error < 1e-4 (frozen eps = same seed)."""
    wl, mdl = _boom_problem(N=50, k=50, hidden=(4,), B=4, T=10, seed=1)
    # goals near the states so rewards (and gradients) are not vanishingly small
    goals = (wl.x0 + 0.3).astype(np.float32)
    base = _run(wl, mdl, goals=goals)
    g = base["grad"]
    th = wl.theta.astype(np.float64)
    fd = np.zeros_like(th)
    for i in range(th.size):
        h = 1e-6 * max(1.0, abs(th[i]))
        tp, tm = th.copy(), th.copy()
        tp[i] += h
        tm[i] -= h
        fp = _run(wl, mdl, theta=tp, goals=goals, want_grad=False)["cost"]
        fm = _run(wl, mdl, theta=tm, goals=goals, want_grad=False)["cost"]
        fd[i] = (fp - fm) / (2 * h)
    err = np.abs(g - fd) / np.maximum(1.0, np.abs(fd))
    assert err.max() < 1e-4
    assert np.linalg.norm(g - fd) / np.linalg.norm(fd) < 1e-4


def test_gradient_directional_fd_deeper_policy():
    wl, mdl = _boom_problem(N=150, k=48, hidden=(16, 16), B=8, T=15, seed=2)
    goals = (wl.x0 + np.array([0.4, -0.2], dtype=np.float32)).astype(np.float32)
    base = _run(wl, mdl, goals=goals)
    th = wl.theta.astype(np.float64)
    rng = np.random.default_rng(0)
    for _ in range(3):
        dirv = rng.normal(size=th.size)
        dirv /= np.linalg.norm(dirv)
        h = 1e-5
        fp = _run(wl, mdl, theta=th + h * dirv, goals=goals, want_grad=False)["cost"]
        fm = _run(wl, mdl, theta=th - h * dirv, goals=goals, want_grad=False)["cost"]
        fd = (fp - fm) / (2 * h)
        an = float(base["grad"] @ dirv)
        assert abs(an - fd) <= 1e-6 * max(abs(fd), 1e-3 * np.linalg.norm(base["grad"]))


def test_goal_difference_input_mode_gradient():
    """C1-style policy input [x, g, g - x] (in = 3p): gradient through the g - x block."""
    wl = W.config("C1", B=4, T=8)
    mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank)
    goals = (wl.x0 + 0.5).astype(np.float32)
    base = _run(wl, mdl, goals=goals)
    th = wl.theta.astype(np.float64)
    rng = np.random.default_rng(1)
    dirv = rng.normal(size=th.size)
    h = 1e-5
    fp = _run(wl, mdl, theta=th + h * dirv, goals=goals, want_grad=False)["cost"]
    fm = _run(wl, mdl, theta=th - h * dirv, goals=goals, want_grad=False)["cost"]
    fd = (fp - fm) / (2 * h)
    assert float(base["grad"] @ dirv) == pytest.approx(fd, rel=1e-6)


def test_determinism(boom_small):
    wl, mdl = boom_small
    a, b = _run(wl, mdl), _run(wl, mdl)
    assert a["cost"] == b["cost"] and np.array_equal(a["grad"], b["grad"])


def test_thread_count_independence(boom_small):
    wl, mdl = boom_small
    n0 = O.num_threads()
    try:
        O.set_num_threads(1)
        a = _run(wl, mdl)
        O.set_num_threads(max(2, n0))
        b = _run(wl, mdl)
    finally:
        O.set_num_threads(n0)
    assert a["cost"] == b["cost"] and np.array_equal(a["grad"], b["grad"])


def test_scalar_rollout_closed_form_absolute_targets():
    """Absolute targets (y = x_{k+1}; NEXT-4): N=1, p=q=1, zero policy:
    x_{t+1} = k(x_t) y1/(s+sn2) + sqrt(s - k(x_t)^2/(s+sn2)) eps_t (no x_t carried)."""
    X = np.array([[0.3, -0.2]])
    y = np.array([[0.05]])
    ell = np.array([[0.8, 0.6]])
    s, sn2 = 0.04, 0.004
    mdl = O.Model.build(X, y, ell, [s], [sn2], 1, abs_target=True)
    sizes = (2, 3, 1)
    out = O.rollout(mdl, sizes, "xg", np.zeros(W.n_params(sizes)), np.array([10.0]), 1.0, np.array([[-0.5]]),
                    np.array([[0.4]]), 9, 0x5EED0043, traj_offset=3, B_global=1, trace=True)
    key = [0x5EED0043, 0]
    x = -0.5
    G = math.exp(-5.0 * (x - 0.4) ** 2)
    for t in range(9):
        o = O.philox4x32_10([3, t, 0, 0], key)
        u0, u1 = [((int(v) >> 9) + 0.5) * 2.0 ** -23 for v in o[:2]]
        eps = math.sqrt(-2.0 * math.log(u0)) * math.cos(2.0 * math.pi * u1)
        k = s * math.exp(-0.5 * (((x - 0.3) / 0.8) ** 2 + ((0.0 + 0.2) / 0.6) ** 2))
        x = k * 0.05 / (s + sn2) + math.sqrt(s - k * k / (s + sn2)) * eps
        assert out["x"][t + 1, 0, 0] == pytest.approx(x, rel=1e-11, abs=1e-14)
        G += math.exp(-5.0 * (x - 0.4) ** 2)
    assert out["cost"] == pytest.approx(-G, rel=1e-11)


def test_gradient_directional_fd_absolute_targets():
    wl = W.make_workload(plant="boom", N=150, rank=48, hidden=(16, 16), B=8, T=15, data_seed=2, target="abs")
    mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank, abs_target=True)
    goals = (wl.x0 + np.array([0.4, -0.2], dtype=np.float32)).astype(np.float32)
    base = _run(wl, mdl, goals=goals)
    th = wl.theta.astype(np.float64)
    rng = np.random.default_rng(5)
    for _ in range(3):
        dirv = rng.normal(size=th.size)
        dirv /= np.linalg.norm(dirv)
        h = 1e-5
        fp = _run(wl, mdl, theta=th + h * dirv, goals=goals, want_grad=False)["cost"]
        fm = _run(wl, mdl, theta=th - h * dirv, goals=goals, want_grad=False)["cost"]
        fd = (fp - fm) / (2 * h)
        an = float(base["grad"] @ dirv)
        assert abs(an - fd) <= 1e-6 * max(abs(fd), 1e-3 * np.linalg.norm(base["grad"]))
    # and it is a different dynamics from the Delta form on the same data
    mdl_d = O.Model(mdl.X, mdl.ell, mdl.s, mdl.alpha, mdl.R, abs_target=False)
    assert abs(_run(wl, mdl_d, goals=goals)["cost"] - base["cost"]) > 1e-3


@pytest.mark.parametrize("phi_mode", ["xg", "xgd"])
@pytest.mark.parametrize("hidden", [(16,), (64, 64), (8, 8, 5)])
def test_policy_forward_matches_torch_sequential(phi_mode, hidden):
    """The oracle's policy (P:129 pi(x, x_g), "bounded in [-1, 1] using a saturating function";
    readings R13/R14) against torch.nn.Sequential(Linear, Tanh, ..., Linear, Tanh) in float64 with
    NONZERO weights.  theta is torch's own flattening of the module's parameters
    (parameters_to_vector: W_l [out x in] row-major, then b_l, layer by layer), so a transposed W,
    a swapped bias or a permuted phi block fails here.  phi = [x, g] (in = 2p) or [x, g, g - x]
    (in = 3p)."""
    import torch

    p, q = 2, 1
    n_in = (2 if phi_mode == "xg" else 3) * p
    sizes = (n_in,) + tuple(hidden) + (q,)
    torch.manual_seed(7)
    layers = []
    for a, b in zip(sizes[:-1], sizes[1:]):
        layers += [torch.nn.Linear(a, b, dtype=torch.float64), torch.nn.Tanh()]
    net = torch.nn.Sequential(*layers)
    with torch.no_grad():
        for prm in net.parameters():   # nonzero biases too (default init leaves them small)
            prm.uniform_(-1.5, 1.5)
    theta = torch.nn.utils.parameters_to_vector(net.parameters()).detach().numpy()
    assert theta.shape[0] == W.n_params(sizes)
    rng = np.random.default_rng(3)
    x = rng.uniform(-1.5, 1.5, (40, p))
    g = rng.uniform(-1.5, 1.5, (40, p))
    xt, gt = torch.from_numpy(x), torch.from_numpy(g)
    phi = torch.cat([xt, gt] if phi_mode == "xg" else [xt, gt, gt - xt], dim=1)
    with torch.no_grad():
        ref = net(phi).numpy()
    u = O.policy_act(sizes, phi_mode, theta, x, g)
    assert np.max(np.abs(u - ref)) <= 1e-14
    assert np.std(ref) > 0.1  # the check is not vacuous (saturated or constant outputs)
