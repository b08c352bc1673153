"""Fig. 5-style scalability sweep: time per policy-gradient
iteration (rollout_cost_and_grad, CUDA events, median of 5 after 2 warm-ups) and device memory of
the library's workspace, versus batch size (up to 10K), horizon (up to 1K) and policy size, on the
C2 boom dataset (N = 5000, LOVE rank 256).  The paper's V100 curves are images (no numbers in the
text); it reports near-linear growth in H, sublinear in BS and policy size, and OOM for plain
GPyTorch at large BS."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

base = W.config("C2", B=1)
ctx = bagel.Context(0)
ctx.gp_load(base.X, base.Y, base.ell, base.s, base.noise)
ctx.love_cache_build(base.rank)
ctx.reward_configure(base.Q, base.sigma_r)
free0 = torch.cuda.mem_get_info()[0]


def run(B, T, hidden):
    sizes = (2 * base.p,) + tuple(hidden) + (base.q,)
    ctx.policy_configure(sizes)
    theta = torch.from_numpy(W.he_init(sizes)).cuda()
    x0, g = (torch.from_numpy(a).cuda() for a in W.sample_states_goals(base.X, base.p, B))
    grad = torch.empty(W.n_params(sizes), device="cuda")
    for i in range(2):
        ctx.rollout_cost_and_grad(theta, x0, g, T, W.rollout_seed(i), grad=grad)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for i in range(5):
        e0.record()
        ctx.rollout_cost_and_grad(theta, x0, g, T, W.rollout_seed(10 + i), grad=grad)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    used = (free0 - torch.cuda.mem_get_info()[0]) / 2 ** 20
    m = float(np.median(ms))
    rec = {"B": B, "T": T, "policy": list(hidden), "n_params": W.n_params(sizes), "ms_per_iter": m,
           "traj_steps_per_s": B * T / m * 1e3, "device_MiB_used_by_library_and_inputs": round(used, 1)}
    print(json.dumps(rec), flush=True)


for B in (10, 100, 1000, 10000):
    run(B, 100, (64, 64))
for T in (300, 1000):
    run(1000, T, (64, 64))
for hidden in ((8, 8), (256, 256), (256, 256, 256)):
    run(1000, 100, hidden)
