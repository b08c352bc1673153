"""BAGEL's policy-optimisation loop (Algorithm 1) around the hot path.

One iteration, all on the GPU:
  1. sample S_0 and G (Alg.1; fixed "repeating entries" as in Exp. 1, or uniform
     within the data bounds as in Exp. 2) -- ``Context.sample_states``;
  2. L and dL/dtheta by ``rollout_cost_and_grad``;
  3. one all_reduce(SUM) of [dL/dtheta | L] over the data-parallel group (``dist``);
  4. Adam (lr 1e-2) -- ``Context.adam_step``.
Iteration i uses the Philox seed ``seed0 + i`` for its noise and its samples (fresh eps per
iteration, reading R17).  Argument marshalling only: every step runs in libbagel.so.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import dist


@dataclass
class TrainLog:
    cost: list = field(default_factory=list)     # L_i (= -mean return) per iteration
    seconds: list = field(default_factory=list)  # wall time since the start, per iteration
    skipped: int = 0                             # updates skipped on a non-finite gradient


def train_policy(ctx, theta0, T: int, iters: int, B_global: int, lo=None, hi=None, *, x0=None, goals=None,
                 lr: float = 1e-2, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 seed0: int = 0x5EED0000, group=None, max_consecutive_skips: int = 10):
    """Runs `iters` iterations of Algorithm 1's inner loop on this rank's trajectory block and returns
    (theta [device tensor], TrainLog).  x0 / goals (B_global x p) fix S_0 / G for every iteration
    (Exp. 1); otherwise they are drawn uniformly in [lo, hi] per state column each iteration (Exp. 2).
    With a torch.distributed group of size G, rank r owns trajectories [r B/G, (r+1) B/G) and the
    gradient is all-reduced before the (replicated, identical) Adam update."""
    world = dist.tdist.get_world_size(group) if dist.tdist.is_initialized() else 1
    rank = dist.tdist.get_rank(group) if dist.tdist.is_initialized() else 0
    off, bl = dist.shard(int(B_global), world, rank)
    dev = ctx.dev
    theta = torch.as_tensor(np.asarray(theta0, dtype=np.float32) if not isinstance(theta0, torch.Tensor) else theta0,
                            dtype=torch.float32).to(dev).clone().contiguous()
    m1 = torch.zeros_like(theta)
    m2 = torch.zeros_like(theta)
    grad = torch.empty_like(theta)

    def fixed(a):
        return None if a is None else torch.as_tensor(np.asarray(a, dtype=np.float32))[off:off + bl].to(dev).contiguous()

    x0_fixed, g_fixed = fixed(x0), fixed(goals)
    if (x0_fixed is None or g_fixed is None) and (lo is None or hi is None):
        raise ValueError("train_policy: give lo/hi bounds for the sampled S_0 / G")
    xs = x0_fixed if x0_fixed is not None else torch.empty(bl, len(lo), device=dev)
    gs = g_fixed if g_fixed is not None else torch.empty(bl, len(lo), device=dev)
    log = TrainLog()
    t_adam, consecutive = 0, 0
    t0 = time.perf_counter()
    for i in range(int(iters)):
        seed = int(seed0) + i
        if x0_fixed is None:
            ctx.sample_states(seed, off, bl, lo, hi, which=0, out=xs)
        if g_fixed is None:
            ctx.sample_states(seed, off, bl, lo, hi, which=1, out=gs)
        cost, grad = ctx.rollout_cost_and_grad(theta, xs, gs, T, seed, traj_offset=off, B_global=B_global, grad=grad)
        cost, grad = dist.allreduce_cost_grad(cost, grad, group)
        skipped = ctx.adam_step(theta, grad, m1, m2, t_adam + 1, lr, beta1, beta2, eps, report_skip=True)
        if skipped:
            log.skipped += 1
            consecutive += 1
            if consecutive >= max_consecutive_skips:
                raise FloatingPointError(f"train_policy: {consecutive} consecutive non-finite gradients (S:403)")
        else:
            t_adam += 1
            consecutive = 0
        log.cost.append(cost)
        log.seconds.append(time.perf_counter() - t0)
    return theta, log
