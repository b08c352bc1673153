import sys, os
sys.path.insert(0, '.')
import numpy as np, torch
import workloads as W
from paper_2202_13638_b200 import bagel
wl = W.config("C3", T=20)
ctx = bagel.setup(wl, device=0)
th = torch.from_numpy(wl.theta).cuda(); x0 = torch.from_numpy(wl.x0).cuda(); g = torch.from_numpy(wl.goals).cuda()
ctx.rollout_cost_and_grad(th, x0, g, 20, 1)
ctx.debug_trace(True)
ctx.rollout_cost_and_grad(th, x0, g, 20, 1)
torch.cuda.synchronize()
st = ctx.debug_stamps(5).reshape(-1)
st = st[60000:60100]
t0 = st[0]
for i in range(100):
    if st[i]: print(i, (int(st[i]) - int(t0)) / 1000.0, "us")
