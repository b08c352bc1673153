"""Profiling driver (run under ncu on the GPU box): one workload's cache build, then R rollouts of
T steps (fwd + reverse) at the bench launch shape.  Launch-list / --set full captures select the
kernels by name; nothing here is timed.
    python scripts/prof_kernels.py CONFIG T [R]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

name, T = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
wl = W.config(name, T=T)
ctx = bagel.setup(wl, device=0)
th = torch.from_numpy(wl.theta).cuda()
x0 = torch.from_numpy(wl.x0).cuda()
g = torch.from_numpy(wl.goals).cuda()
for i in range(reps):
    cost, grad = ctx.rollout_cost_and_grad(th, x0, g, T, W.rollout_seed(i))
torch.cuda.synchronize()
print(name, "T", T, "cost", cost, "launches", ctx.last_launch_count())
