"""BAGEL (arXiv 2202.13638) hot path on B200: batched LOVE-GP policy rollouts
and their reverse pass as sm_100a CUDA kernels behind a C ABI (include/bagel.h).

    from paper_2202_13638_b200 import bagel, dist
    ctx = bagel.Context()
    ctx.gp_load(X, Y, lengthscales, outputscale, noise)
    ctx.love_cache_build(rank)
    ctx.policy_configure(sizes); ctx.reward_configure(Q, sigma_r)
    cost, grad = ctx.rollout_cost_and_grad(theta, x0, goals, T, seed)
"""
from .build import LIB  # noqa: F401
