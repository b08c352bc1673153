"""Per-phase timing of one step (t = T/2) of the reverse recursion (block 0, warp 0)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

wl = W.config(sys.argv[1] if len(sys.argv) > 1 else "C2")
ctx = bagel.setup(wl, device=0)
theta = torch.from_numpy(wl.theta).cuda()
x0 = torch.from_numpy(wl.x0).cuda()
goals = torch.from_numpy(wl.goals).cuda()
grad = torch.empty(ctx.n_params, device="cuda")
for i in range(3):
    ctx.rollout_cost_and_grad(theta, x0, goals, wl.T, W.rollout_seed(i), traj_offset=0, B_global=wl.B, grad=grad)
ctx.debug_trace(True)
ctx.rollout_cost_and_grad(theta, x0, goals, wl.T, W.rollout_seed(9), traj_offset=0, B_global=wl.B, grad=grad)
torch.cuda.synchronize()
st = ctx.debug_stamps(6).astype(np.int64)[0]
names = ["start", "tape row landed", "xs, delta_L", "layer L-1", "layer L-2", "layer L-3", "-", "-", "end of step"]
for k in range(9):
    if st[k] > 0:
        print(f"{names[k]:18s} {(st[k] - st[0]) / 1e3:7.3f} us")
