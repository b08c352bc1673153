"""Seeded synthetic inputs for BAGEL's hot path (shared by tests, smoke() and bench.py).

This module holds NONE of the method's arithmetic: no kernel, no GP prediction,
no policy, no reward, no rollout.  It only simulates the stand-in plants that
produce the training transitions, standardises them (caller-side data prep,
PAPER.md P:149 "normalized according to the mean mu_X and standard deviation
sigma_X"), fixes the documented hyperparameters, and draws x0 / goals / theta.
Both the CUDA path and the oracle consume exactly the float32 arrays returned
here (the oracle widens them to float64 exactly).

Recipe:
  * boom plant (C2, C3, C5): phi'' = 2.0*dead(u) - 1.5*phi' - 0.5*cos(phi),
    semi-implicit Euler at dt = 0.05, hard stops [-1.2, 0.9] rad (rate zeroed),
    observation noise (0.002 rad, 0.01 rad/s)  (SPEC.md S:497 defaults);
  * 1-D actuator (C1): phi_{k+1} = phi_k + dt*(1.0*dead(u) - 0.2*cos(phi_k)) + 0.002*xi;
  * 4-state hydraulic actuator (C4): see ``_simulate_hydraulic4``;
  * excitation: an emulated operator "manually lowering and raising the boom"
     "at two speeds": phi_ref ~ U(-1.1, 0.8) redrawn every 100
    steps, n_{k+1} = 0.9 n_k + 0.3 xi, u = clip(1.5 (phi_ref - phi) + n, -1, 1);
  * GP inputs standardised; targets are Delta x in normalised state units;
  * hyperparameters fixed: s_m = Var(Delta_m), sigma_n^2 = 1e-2 s_m,
    l = 1.0 (state dims), 0.7 (action dims), times (1 + 0.1 m);
  * x0, goals ~ U(per-column [min, max] of the normalised state columns of X)
    (P:180), C1 uses the fixed single goal of Exp. 1;
  * theta: He init W ~ N(0, 2/fan_in), b = 0.
Seeds: data 0, x0 1, goals 2, theta 3 (numpy default_rng); rollout seed of
iteration i is 0x5EED0000 + i.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

DT = 0.05
DEADBAND = 0.1
STOPS = (-1.2, 0.9)
ROLLOUT_SEED0 = 0x5EED0000


def dead(u: float, db: float = DEADBAND) -> float:
    """Actuator deadband: 0 inside |u| < db, linear ramp to +-1 outside."""
    a = abs(u)
    if a <= db:
        return 0.0
    return math.copysign((a - db) / (1.0 - db), u)


class _Operator:
    """Emulated human operator raising/lowering the boom."""

    def __init__(self, rng: np.random.Generator):
        self.rng = rng
        self.ref = 0.0
        self.n = 0.0
        self.k = 0

    def action(self, phi: float) -> float:
        if self.k % 100 == 0:
            self.ref = float(self.rng.uniform(-1.1, 0.8))
        self.k += 1
        self.n = 0.9 * self.n + 0.3 * float(self.rng.standard_normal())
        return min(1.0, max(-1.0, 1.5 * (self.ref - phi) + self.n))


def _simulate_boom(n: int, rng: np.random.Generator):
    phi, dphi = -0.5, 0.0
    op = _Operator(rng)
    obs = np.empty((n + 1, 2))
    act = np.empty((n, 1))
    noise = (0.002, 0.01)
    for k in range(n + 1):
        obs[k, 0] = phi + noise[0] * rng.standard_normal()
        obs[k, 1] = dphi + noise[1] * rng.standard_normal()
        if k == n:
            break
        u = op.action(obs[k, 0])
        act[k, 0] = u
        acc = 2.0 * dead(u) - 1.5 * dphi - 0.5 * math.cos(phi)
        dphi = dphi + DT * acc
        phi = phi + DT * dphi
        if phi < STOPS[0]:
            phi, dphi = STOPS[0], 0.0
        elif phi > STOPS[1]:
            phi, dphi = STOPS[1], 0.0
    return obs, act


def _simulate_actuator1(n: int, rng: np.random.Generator):
    phi = -0.5
    op = _Operator(rng)
    obs = np.empty((n + 1, 1))
    act = np.empty((n, 1))
    for k in range(n + 1):
        obs[k, 0] = phi
        if k == n:
            break
        u = op.action(phi)
        act[k, 0] = u
        phi = phi + DT * (1.0 * dead(u) - 0.2 * math.cos(phi)) + 0.002 * rng.standard_normal()
        phi = min(STOPS[1], max(STOPS[0], phi))
    return obs, act


def _simulate_hydraulic4(n: int, rng: np.random.Generator):
    """Position, velocity, chamber pressures p_A, p_B; one valve."""
    x1, x2, x3, x4 = -0.5, 0.0, 0.0, 0.0
    op = _Operator(rng)
    obs = np.empty((n + 1, 4))
    act = np.empty((n, 1))
    for k in range(n + 1):
        obs[k] = (x1, x2, x3, x4) + 0.01 * rng.standard_normal(4)
        if k == n:
            break
        u = op.action(obs[k, 0])
        act[k, 0] = u
        du = dead(u)
        x3 = x3 + DT * (5.0 * (du - x2) - 0.3 * x3)
        x4 = x4 + DT * (4.0 * (-du + 0.8 * x2) - 0.5 * x4)
        x2 = x2 + DT * (2.0 * (x3 - x4) - 1.5 * x2 - 0.5 * math.cos(x1))
        x1 = x1 + DT * x2
        if x1 < STOPS[0]:
            x1, x2 = STOPS[0], 0.0
        elif x1 > STOPS[1]:
            x1, x2 = STOPS[1], 0.0
    return obs, act


PLANTS = {"boom": _simulate_boom, "actuator1": _simulate_actuator1, "hydraulic4": _simulate_hydraulic4}
Q_DIAG = {"boom": (10.0, 0.1), "actuator1": (10.0,), "hydraulic4": (10.0, 0.1, 1.0, 1.0)}


@dataclass
class Workload:
    """One hot-path problem instance; every array is float32 (what the GPU sees)."""

    name: str
    plant: str
    N: int
    p: int
    q: int
    rank: int                 # LOVE rank k
    sizes: tuple              # MLP layer sizes (in, h1, ..., q)
    B: int
    T: int
    X: np.ndarray = field(repr=False)        # N x d standardised (x, u)
    Y: np.ndarray = field(repr=False)        # N x p Delta-x targets (normalised state units)
    ell: np.ndarray = field(repr=False)      # p x d lengthscales
    s: np.ndarray = field(repr=False)        # p outputscale (signal variance)
    noise: np.ndarray = field(repr=False)    # p noise variance sigma_n^2
    Q: np.ndarray = field(repr=False)        # p reward weights
    sigma_r: float = 1.0
    x0: np.ndarray = field(default=None, repr=False)     # B x p
    goals: np.ndarray = field(default=None, repr=False)  # B x p
    theta: np.ndarray = field(default=None, repr=False)  # |theta|

    @property
    def d(self) -> int:
        return self.p + self.q

    @property
    def n_params(self) -> int:
        return n_params(self.sizes)


def n_params(sizes) -> int:
    return int(sum((sizes[i] + 1) * sizes[i + 1] for i in range(len(sizes) - 1)))


def he_init(sizes, seed: int = 3) -> np.ndarray:
    """theta in nn.Sequential(Linear, Tanh, ...) order: W_l [out x in] row-major, then b_l."""
    rng = np.random.default_rng(seed)
    parts = []
    for i in range(len(sizes) - 1):
        fin, fout = sizes[i], sizes[i + 1]
        parts.append(rng.normal(0.0, math.sqrt(2.0 / fin), size=fout * fin))
        parts.append(np.zeros(fout))
    return np.concatenate(parts).astype(np.float32)


def make_dataset(plant: str, N: int, seed: int = 0, target: str = "delta"):
    """Simulate, standardise and build (X, Y, hyperparameters).  Returns float32 arrays.
    target "delta": y = Delta x (reading R6); "abs": y = x_{k+1}, both in normalised units."""
    rng = np.random.default_rng(seed)
    obs, act = PLANTS[plant](N, rng)
    states, nxt = obs[:-1], obs[1:]
    raw = np.concatenate([states, act], axis=1)
    mu = raw.mean(axis=0)
    sd = raw.std(axis=0)
    sd[sd < 1e-8] = 1.0
    X = (raw - mu) / sd
    p = states.shape[1]
    Y = (nxt - states) / sd[:p] if target == "delta" else (nxt - mu[:p]) / sd[:p]
    q = act.shape[1]
    s = Y.var(axis=0)
    noise = 1e-2 * s
    ell = np.empty((p, p + q))
    for m in range(p):
        ell[m, :p] = 1.0 * (1.0 + 0.1 * m)
        ell[m, p:] = 0.7 * (1.0 + 0.1 * m)
    norm = {"mu": mu, "sd": sd}
    return (X.astype(np.float32), Y.astype(np.float32), ell.astype(np.float32),
            s.astype(np.float32), noise.astype(np.float32), norm)


def make_workload(name: str = "custom", plant: str = "boom", N: int = 5000, rank: int = 256,
                  hidden=(64, 64), B: int = 1024, T: int = 100, phi_mode: str = "xg",
                  data_seed: int = 0, fixed_start: bool = False, target: str = "delta") -> Workload:
    """Build a workload.  phi_mode 'xg' -> policy input [x, g] (in = 2p);
    'xgd' -> [x, g, g - x] (in = 3p, C1)."""
    X, Y, ell, s, noise, norm = make_dataset(plant, N, data_seed, target)
    p = Y.shape[1]
    q = X.shape[1] - p
    n_in = 2 * p if phi_mode == "xg" else 3 * p
    sizes = (n_in,) + tuple(hidden) + (q,)
    wl = Workload(name=name, plant=plant, N=N, p=p, q=q, rank=rank, sizes=sizes, B=B, T=T,
                  X=X, Y=Y, ell=ell, s=s, noise=noise,
                  Q=np.asarray(Q_DIAG[plant], dtype=np.float32))
    if fixed_start or name == "C1":
        # Exp. 1: all rows start at the same state ("a low angle": -0.8 rad, at rest), single
        # fixed goal r(., -mu_X / sigma_X), i.e. 0 rad (and 0 rad/s) in normalised units.
        x0 = ((np.array([-0.8, 0.0, 0.0, 0.0])[:p] - norm["mu"][:p]) / norm["sd"][:p]).astype(np.float32)
        g = ((0.0 - norm["mu"][:p]) / norm["sd"][:p]).astype(np.float32)
        wl.x0 = np.tile(x0, (B, 1)).astype(np.float32)
        wl.goals = np.tile(g, (B, 1)).astype(np.float32)
    else:
        wl.x0, wl.goals = sample_states_goals(X, p, B)
    wl.theta = he_init(sizes, 3)
    return wl


def sample_states_goals(X: np.ndarray, p: int, B: int, seed_x0: int = 1, seed_g: int = 2):
    """Uniform within the per-column bounds of the normalised state columns."""
    lo = X[:, :p].min(axis=0).astype(np.float64)
    hi = X[:, :p].max(axis=0).astype(np.float64)
    x0 = np.random.default_rng(seed_x0).uniform(lo, hi, size=(B, p))
    g = np.random.default_rng(seed_g).uniform(lo, hi, size=(B, p))
    return x0.astype(np.float32), g.astype(np.float32)


# BASELINE.json configs; SURVEY.md §0 table with the §8(c) #15 readings for unstated fields.
CONFIGS = {
    "C1": dict(plant="actuator1", N=200, rank=50, hidden=(16,), B=16, T=20, phi_mode="xgd"),
    "C2": dict(plant="boom", N=5000, rank=256, hidden=(64, 64), B=1024, T=100, phi_mode="xg"),
    "C3": dict(plant="boom", N=5000, rank=256, hidden=(256, 256, 256), B=4096, T=500, phi_mode="xg"),
    "C4": dict(plant="hydraulic4", N=20000, rank=512, hidden=(64, 64), B=8192, T=200, phi_mode="xg"),
    "C5": dict(plant="boom", N=50000, rank=512, hidden=(64, 64), B=65536, T=200, phi_mode="xg"),
    # the paper's Exp. 1 shape: n = 2200, b = 100, H = 300, policy [8, 8], fixed start and
    # goal; LOVE rank unstated -> 100 (GPyTorch's default root-decomposition size, reading R32)
    "E1": dict(plant="boom", N=2200, rank=100, hidden=(8, 8), B=100, T=300, phi_mode="xg", fixed_start=True),
}


def config(name: str, **overrides) -> Workload:
    kw = dict(CONFIGS[name])
    kw.update(overrides)
    return make_workload(name=name, **kw)


def rollout_seed(iteration: int) -> int:
    return ROLLOUT_SEED0 + int(iteration)


def with_batch(wl: Workload, B: int) -> Workload:
    """Same problem, first B rows of x0/goals (trajectory subset; ids stay global)."""
    return replace(wl, B=B, x0=wl.x0[:B].copy(), goals=wl.goals[:B].copy())
