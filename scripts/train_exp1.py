"""Time to train a policy at the paper's Exp. 1 shape: boom GP on n = 2200 synthetic
transitions, b = 100 trajectories, H = 300, policy [8, 8], fixed start and goal, Adam lr 1e-2 --
Algorithm 1's inner loop run entirely through libbagel.so (train.train_policy).  The paper's figure
for this task is "under 30 seconds" on a laptop T2000: context, not a target.

Prints one JSON line: seconds per iteration (median), iterations/s, the cost curve in blocks of
10 iterations, and the mean return per step at the start and the end."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402
from paper_2202_13638_b200.train import train_policy  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
lr = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-2
wl = W.config("E1")
t0 = time.perf_counter()
ctx = bagel.setup(wl, device=0)
setup_s = time.perf_counter() - t0
train_policy(ctx, wl.theta, wl.T, 2, wl.B, x0=wl.x0, goals=wl.goals, lr=lr)  # warm-up (workspace allocation)
torch.cuda.synchronize()
th, log = train_policy(ctx, wl.theta, wl.T, iters, wl.B, x0=wl.x0, goals=wl.goals, lr=lr)
sec = np.diff([0.0] + log.seconds)
c = np.array(log.cost)
blocks = [float(x) for x in c[: len(c) // 10 * 10].reshape(-1, 10).mean(1)]
print(json.dumps({
    "workload": "E1: boom GP N=2200 d=3 p=2, LOVE rank 100, MLP 4-8-8-1, B=100, T=300, fixed start/goal (Exp. 1)",
    "iters": iters, "lr": lr, "setup_s (gp_load + cache build + config)": setup_s,
    "cache_build_s": ctx.cache_seconds,
    "train_s": log.seconds[-1], "s_per_iter_median": float(np.median(sec)), "iters_per_s": iters / log.seconds[-1],
    "traj_steps_per_s": iters * wl.B * wl.T / log.seconds[-1],
    "mean_return_per_step_first10": float(-c[:10].mean() / (wl.T + 1)),
    "mean_return_per_step_last10": float(-c[-10:].mean() / (wl.T + 1)),
    "cost_blocks_of_10": blocks, "skipped": log.skipped,
    "paper_context": "BAGEL-GPU: under 30 s to train this task's policy on an i7-10750H + Quadro T2000 (P:20, P:156)",
}))
